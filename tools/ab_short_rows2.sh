# bf16 V=32000 (short rows), sustained (300 iterations): loss pass per layout/mix.
set -u
for r in 1 2; do
  for v in "7 1" "6 0" "6 4" "6 1"; do
    set -- $v
    RLO_VOCAB_MATH=$1 RLO_VOCAB_LDG=$2 timeout 600 python tools/bench_update.py --forms two_pass --cases bf16_32k --iters 300 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('math=$1 ldg=$2', d['case'], 'loss', round(d['loss_ms'], 3), 'ms', round(d['loss_gbs']), 'GB/s')"
  done
done
