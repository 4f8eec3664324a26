# fused update pass: 2 vs 3 actor slices in flight (RLO_FUSED_NB), cfg2 shape; 32 and 24 KB slices for NB=3
for r in 1 2; do
  for cfg in "2 32" "3 32" "3 24"; do set -- $cfg
    RLO_FUSED_DEBUG=1 RLO_FUSED_NB=$1 RLO_FUSED_SLICE_KB=$2 timeout 300 python tools/bench_update.py --cases cfg2 --forms fused --iters 5 2>&1 | \
      grep -E "^\{|fused pass" | sort | uniq | cut -c1-110 | sed "s/^/NB=$1 kb=$2 /"
  done
done
