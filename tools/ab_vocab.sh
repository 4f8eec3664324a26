# A/B of the vocab pass across library builds (RLO_LIB), same box, interleaved.
for round in 1 2; do
  for lib in "" paper_2506_06122_b200/lib/variants/librlo_a3f4.so paper_2506_06122_b200/lib/variants/librlo_f337.so; do
    for c in 2 3; do
      st=10; [ $c = 3 ] && st=2
      RLO_LIB=$lib timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('lib=${lib:-cur}'.split('/')[-1], 'cfg$c', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz')"
    done
  done
done
