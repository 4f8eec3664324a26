# bf16 vocab-pass tuning sweep (cfg3 shape): LDG layout x instruction mix.
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
RLO_VOCAB_MATH=5 RLO_VOCAB_LDG=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for L in 0 1 2 3; do for m in 1 2 4 5; do
  RLO_VOCAB_LDG=$L RLO_VOCAB_MATH=$m timeout 200 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sb_${L}_$m.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/sb_${L}_$m.json'));r=d['roofline'];print('cfg3 ldg_layout=$L math=$m', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
