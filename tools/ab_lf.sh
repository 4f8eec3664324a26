# default vocab kernel vs the barrier-free variant (RLO_VOCAB_LF=1), cfg2 fp32 and cfg3 bf16, alternating.
for r in 1 2; do for e in 0 1; do for c in 2 3; do
  st=10; [ $c = 3 ] && st=2
  RLO_VOCAB_LF=$e timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('lf=$e cfg$c', round(r['achieved']), 'GB/s  p1', round(d['p1']['achieved_gbs']), d['clocks']['sm_mhz'], 'MHz')"
done; done; done
