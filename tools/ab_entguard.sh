# fp32 entropy row: always guarded (current) vs unguarded + guarded redo (librlo_prev.so), cfg1/cfg2 fp32, interleaved.
for round in 1 2 3; do
  for lib in "" paper_2506_06122_b200/lib/variants/librlo_prev.so; do
    for c in 1 2; do
      RLO_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('lib=${lib:-cur}'.split('/')[-1], 'cfg$c', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz')"
    done
  done
done
