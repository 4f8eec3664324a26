# LDG (default) vs TMA ring producer under the bench's power-capped conditions, cfg3 bf16 and cfg2 fp32.
for r in 1 2; do for impl in ldg tma; do for c in 3 2; do
  st=10; [ $c = 3 ] && st=2
  RLO_VOCAB_IMPL=$impl timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$impl cfg$c', round(r['achieved']), 'GB/s  p1', round(d['p1']['achieved_gbs']), d['clocks']['sm_mhz'], 'MHz', round(d['clocks'].get('power_w') or 0), 'W')"
done; done; done
