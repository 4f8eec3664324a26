# bf16 instruction mix (RLO_VOCAB_MATH) on cfg3, P=3 and the P=1 leg, under bench conditions.
for m in 4 6 2 4 6; do
  RLO_VOCAB_MATH=$m timeout 300 python bench.py --config 3 --steps 2 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; p=d['p1']; print('math=$m P3', round(r['achieved']), 'GB/s  P1', round(p['achieved_gbs']), 'GB/s', d['clocks']['sm_mhz'], 'MHz')"
done
