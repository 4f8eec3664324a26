# 4-GPU round: full GPU suite (incl. dp2/dp4 parity), integration binary, weak-scaling bench lines.
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
./build/integration_test | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/m_cfg2_n1.json 2> gpurun_out/m_cfg2_n1.err; echo n1 rc=$?
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/m_cfg2_n$n.json 2> gpurun_out/m_cfg2_n$n.err; echo n$n rc=$?
done
for n in 1 4; do
  if [ $n -eq 1 ]; then timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m_cfg3_n1.json 2> gpurun_out/m_cfg3_n1.err;
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --config 3 --gpus 4 --steps 2 --warmup 3 > gpurun_out/m_cfg3_n4.json 2> gpurun_out/m_cfg3_n4.err; fi; echo cfg3 n$n rc=$?
done
for f in gpurun_out/m_*.json; do python -c "
import json,sys
d=json.load(open('$f'));r=d['roofline']
print('$f', d['n_gpus'], round(d['value']), 'tok/s', round(r['achieved']), round(r['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"; done
