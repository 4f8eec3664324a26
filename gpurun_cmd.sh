bash tools/probes/power_probe.sh 2>&1 | tee gpurun_out/r2_power_probe.txt
python bench.py --steps 15 --warmup 3 --no-cpu-baseline --no-e2e --no-p1 > gpurun_out/r2_power_bench3.json 2>/dev/null
python bench.py --config 2 --steps 400 --warmup 3 --no-cpu-baseline --no-e2e --no-p1 > gpurun_out/r2_power_bench2.json 2>/dev/null
python3 -c "
import json
for f in ['gpurun_out/r2_power_bench3.json','gpurun_out/r2_power_bench2.json']:
    d=json.load(open(f)); print(f, round(d['roofline']['achieved']), d['clocks'], d['ms_per_step']*d['steps'], 'ms timed')
" | tee -a gpurun_out/r2_power_probe.txt
