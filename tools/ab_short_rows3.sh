# bf16 short rows, V-dependent default (auto) vs forced mixes; P=3 and P=1 loss passes, V=32000 and 50264 (stride), cfg3.
set -u
RLO_VOCAB_MATH= timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  for v in "auto" "7" "6"; do
    for P in 3 1; do
      if [ $v = auto ]; then unset RLO_VOCAB_MATH; else export RLO_VOCAB_MATH=$v; fi
      timeout 600 python tools/bench_update.py --forms two_pass --cases bf16_32k,cfg3 --P $P --iters 200 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('math=$v P=$P', d['case'], 'loss', round(d['loss_ms'], 3), 'ms', round(d['loss_gbs']), 'GB/s')"
    done
  done
done
