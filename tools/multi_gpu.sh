# 4-GPU round: multi-GPU tests (dp2/dp4 parity incl. the fused pass, broadcast), weak-scaling bench lines.
timeout 900 python -m pytest tests/test_gpu_multi.py -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/m_cfg2_n1.json 2> gpurun_out/m_cfg2_n1.err; echo n1 rc=$?
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/m_cfg2_n$n.json 2> gpurun_out/m_cfg2_n$n.err; echo n$n rc=$?
done
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m_cfg3_n1.json 2> gpurun_out/m_cfg3_n1.err; echo cfg3 n1 rc=$?
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --config 3 --gpus $n --steps 2 --warmup 3 > gpurun_out/m_cfg3_n$n.json 2> gpurun_out/m_cfg3_n$n.err; echo cfg3 n$n rc=$?
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/bench_next.py --only broadcast 2>&1 | grep "^{"
for f in gpurun_out/m_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]);r=d['roofline']
print('$f', d['n_gpus'], round(d['value']), 'tok/s', round(r['achieved']), round(r['frac'],3), 'e2e', round(d['e2e']['value']), 'p1', round(d['p1']['value']), d['clocks']['sm_mhz'])"; done
