# cfg5 (batch-sharded global batch, strong scaling) at 1/2/4 GPUs.
timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.err; echo n1 rc=$?
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --config 5 --gpus $n --steps 2 --warmup 3 > gpurun_out/c5_n$n.json 2> gpurun_out/c5_n$n.err; echo n$n rc=$?
done
for n in 1 2 4; do python -c "
import json
d=json.loads(open('gpurun_out/c5_n$n.json').read().strip().splitlines()[-1]);r=d['roofline']
print('cfg5 n=$n', d['scaling'], round(d['value']), 'tok/s', round(d['ms_per_step']), 'ms/step', round(r['achieved']), 'GB/s', 'e2e', round(d['e2e']['value']), 'p1', round(d['p1']['value']), d['config']['B_per_rank'], d['clocks']['sm_mhz'])"; done
