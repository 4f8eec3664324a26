# bf16 cfg3: sequential streams (RLO_VOCAB_LDG=0) vs lockstep streams with a shared max (=4), alternating.
for r in 1 2; do for l in 0 4; do
  RLO_VOCAB_LDG=$l timeout 300 python bench.py --config 3 --steps 2 --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ldg=$l', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz', d['clocks'].get('power_w'), 'W')"
done; done
