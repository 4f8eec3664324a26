timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2k_bench_cfg3.json 2> gpurun_out/r2k_bench_cfg3.err; python3 -c "
import json; d=json.loads(open('gpurun_out/r2k_bench_cfg3.json').read().strip().splitlines()[0]); r=d['roofline']; p=d['p1']
print(round(d['value']/1e6,3), round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'], round(p['value']/1e6,2), round(p['achieved_gbs']), r['traffic'])"
