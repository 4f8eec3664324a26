timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
RLO_VOCAB_IMPL=ldg RLO_VOCAB_MATH=3 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or full_size or synthetic" 2>&1 | tail -2
for impl in ldg tma; do for m in 0 1 2 3; do
  RLO_VOCAB_IMPL=$impl RLO_VOCAB_MATH=$m timeout 200 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw3_${impl}_$m.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw3_${impl}_$m.json'));r=d['roofline'];print('cfg3 $impl math=$m', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'])"
done; done
for impl in ldg tma; do for m in 0 1; do
  RLO_VOCAB_IMPL=$impl RLO_VOCAB_MATH=$m timeout 200 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw2_${impl}_$m.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sw2_${impl}_$m.json'));r=d['roofline'];print('cfg2 $impl math=$m', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'])"
done; done
