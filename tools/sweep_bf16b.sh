# bf16 sweep round 2: MATH 4 now also offloads 25% of the actor row's exponentials.
RLO_VOCAB_MATH=4 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -q -x 2>&1 | tail -2
for m in 2 4 1 4 2; do
  RLO_VOCAB_MATH=$m timeout 200 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sc_$m.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sc_$m.json'));r=d['roofline'];print('cfg3 math=$m', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'], round(r['achieved']/d['clocks']['sm_mhz'],3), 'GB/s per MHz')"
done
