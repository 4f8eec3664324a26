# A/B of library builds (RLO_LIB) on the box probe and short bench lines; args: variant names under lib/variants
for lib in "" "$@"; do
  p=""; [ -n "$lib" ] && p=paper_2506_06122_b200/lib/variants/librlo_$lib.so
  echo "== ${lib:-current}"; RLO_LIB=$p python tools/probes/box_probe.py 2>&1 | grep -E "forward"
  for c in 2 3; do
    st=10; [ $c = 3 ] && st=2
    RLO_LIB=$p timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  cfg$c', round(d['value']), 'tok/s', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz')"
  done
done
