#!/bin/bash
# Round-2 multi-GPU call (one 4-GPU box): dp2 / dp4 parity (tests/test_gpu_multi.py: global whitening,
# rank-ordered merge, fused pass, bit-identical bucketed broadcast) and bench lines at N = 1 / 2 / 4:
# cfg3 (default, weak scaling), cfg2 (weak), cfg5 (one global batch sharded: strong).
cd "$(dirname "$0")/.."
O=gpurun_out; P=${P:-r2m}
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -rf -s > $O/${P}_multi_tests.log 2>&1; echo "multi tests rc=$?" >> $O/${P}_multi_tests.log; tail -3 $O/${P}_multi_tests.log
run() {  # cfg n steps
  if [ $2 = 1 ]; then
    timeout 900 python bench.py --config $1 --steps $3 --warmup 3 --no-cpu-baseline > $O/${P}_cfg$1_n$2.json 2> $O/${P}_cfg$1_n$2.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 295$1$2 \
      bench.py --config $1 --gpus $2 --steps $3 --warmup 3 > $O/${P}_cfg$1_n$2.json 2> $O/${P}_cfg$1_n$2.err
  fi
  echo "cfg$1 n$2 rc=$?"
}
for n in 1 2 4; do run 3 $n 5; done
for n in 1 2 4; do run 2 $n 20; done
for n in 1 2 4; do run 5 $n 2; done
grep -h "nRanks\|nranks" $O/${P}_cfg3_n4.err | head -4
for f in $O/${P}_cfg*_n*.json; do python3 -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d['roofline']
print('$f', d['n_gpus'], round(d['value']), 'tok/s', round(r['achieved']), round(r['frac'],3), 'e2e', round(d['e2e']['value']), 'p1', round(d['p1']['value']), d['clocks']['sm_mhz'])" 2>/dev/null || echo "$f failed"; done
