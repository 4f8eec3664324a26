# Round-end measurement on one B200: GPU suite, integration, bench lines for every
# config (+ the reference arm), the ncu launch list of the default bench command.
set -u
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
./build/integration_test | tail -1
for c in 1 2 3 4 5; do
  st=20; [ $c -ge 3 ] && st=3; [ $c -eq 5 ] && st=2
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/e_cfg$c.json 2> gpurun_out/e_cfg$c.err; echo cfg$c rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/e_ref_cfg2.json 2> gpurun_out/e_ref_cfg2.err; echo ref rc=$?
timeout 600 python bench.py --impl reference --config 3 --steps 3 --warmup 1 > gpurun_out/e_ref_cfg3.json 2> gpurun_out/e_ref_cfg3.err; echo ref3 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/e_ncu.log 2>&1; echo ncu rc=$?
for c in 1 2 3 4 5; do python -c "
import json
d=json.loads(open('gpurun_out/e_cfg$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cfg$c', round(d['value']), 'tok/s', round(r['achieved']), round(r['frac'],3), 'e2e', round(d['e2e']['value']), 'p1', round(d['p1']['value']), 'cpu', round(d['cpu_baseline']['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['gpu_launches'])"; done
cat gpurun_out/e_ref_cfg2.json gpurun_out/e_ref_cfg3.json
