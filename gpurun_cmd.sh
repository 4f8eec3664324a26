timeout 600 python -m pytest tests/test_gpu_production.py -m gpu -q -p no:cacheprovider -rf -k "alignments" 2>&1 | tail -3
for c in 1 4; do timeout 900 python bench.py --config $c > gpurun_out/r2k_bench_cfg$c.json 2> gpurun_out/r2k_bench_cfg$c.err; echo "cfg$c rc=$?"; done
python3 -c "
import json
for c in (1,4):
    d=json.load(open(f'gpurun_out/r2k_bench_cfg{c}.json')); r=d['roofline']
    print(c, round(d['value']), round(r['achieved']), round(r['frac'],4), d['clocks']['sm_mhz'], round(d['e2e']['value']), d['cpu_baseline']['value'], d['cpu_baseline']['gpu_oracle_check']['max_scaled_err'])
"
