timeout 300 python -m pytest tests/test_gpu_edges.py -q 2>&1 | grep -E "^E |assert|passed|failed" | head -40
# A/B: __launch_bounds__(256, 4) (in-tree) vs (256) (variants/librlo_lb1.so) on the fp32 and bf16 vocab pass
for lib in "" "paper_2506_06122_b200/lib/variants/librlo_lb1.so" "" "paper_2506_06122_b200/lib/variants/librlo_lb1.so"; do
  RLO_LIB=$lib timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab2.json 2>/dev/null
  RLO_LIB=$lib timeout 200 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab3.json 2>/dev/null
  python -c "
import json
for f in ['gpurun_out/ab2.json','gpurun_out/ab3.json']:
  d=json.load(open(f)); r=d['roofline']; print('lib=${lib:-default}', f, round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'])"
done
