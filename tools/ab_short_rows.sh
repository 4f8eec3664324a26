# bf16 V=32000 (short 64 KB rows): loss pass per layout/mix (bench_update two-pass loss_ms).
set -u
for r in 1 2; do
  for v in "7 0" "6 0" "6 4" "6 1"; do
    set -- $v
    echo "== math=$1 ldg=$2"
    RLO_VOCAB_MATH=$1 RLO_VOCAB_LDG=$2 timeout 600 python tools/bench_update.py --forms two_pass --cases bf16_32k,cfg3 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['case'], 'loss', round(d['loss_ms'], 3), 'ms', round(d['loss_gbs']), 'GB/s')"
  done
done
