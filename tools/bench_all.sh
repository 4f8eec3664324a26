# Round-1 bench lines for every BASELINE.json config on one B200 (defaults).
for c in 1 2 3 4 5; do
  steps=10; [ $c -ge 3 ] && steps=3; [ $c -eq 5 ] && steps=2
  timeout 900 python bench.py --config $c --steps $steps --warmup 3 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c rc=$?"; tail -2 gpurun_out/bench_cfg$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_cfg$c.json'));r=d['roofline'];print('cfg$c', round(d['value']), 'tok/s', round(r['achieved']), 'GB/s', round(r['frac'],3), 'e2e', round(d['e2e']['value']), 'cpu', round(d['cpu_baseline']['value']), d['clocks'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref_cfg2.err; echo ref rc=$?; cat gpurun_out/bench_ref_cfg2.json
