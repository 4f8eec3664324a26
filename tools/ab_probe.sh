for lib in "" r0l4 r0l1 r1l1 4b0; do
  p=""; [ -n "$lib" ] && p=paper_2506_06122_b200/lib/variants/librlo_$lib.so
  echo "== ${lib:-current(r1l4)}"; RLO_LIB=$p python tools/probes/box_probe.py 2>&1 | grep -E "forward"
done
