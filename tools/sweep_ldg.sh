# bf16 fused-loss pass (cfg3): register cap (launch bounds 4 = in-tree, 3 = variants/librlo_lb3.so) x LDG layout
for lib in "" lb3; do
  p=""; [ -n "$lib" ] && p=paper_2506_06122_b200/lib/variants/librlo_$lib.so
  for ldg in 0 1 2; do
    RLO_LIB=$p RLO_VOCAB_LDG=$ldg timeout 300 python bench.py --config 3 --steps 2 --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('lib=${lib:-lb4} ldg=$ldg', round(d['value']), 'tok/s', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz')"
  done
done
