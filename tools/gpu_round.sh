# Full GPU check on a 2-GPU box: suite (incl. dp2 + broadcast), integration, default bench lines.
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
./build/integration_test | tail -1
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/r_cfg2.json 2> gpurun_out/r_cfg2.err; echo cfg2 rc=$?
timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r_cfg3.json 2> gpurun_out/r_cfg3.err; echo cfg3 rc=$?
for f in gpurun_out/r_cfg2.json gpurun_out/r_cfg3.json; do python -c "
import json
l=open('$f').read().strip().splitlines(); print(len(l),'stdout line(s)'); d=json.loads(l[-1]); r=d['roofline']
print('$f', round(d['value']), 'tok/s', round(r['achieved']), round(r['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks'], d['gpu_launches'])"; done
