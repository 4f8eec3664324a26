# Backward epilogue: 4 loads in flight per thread (default) vs 1 (librlo_bw1.so); two-pass update step.
set -u
timeout 900 python -m pytest tests -m gpu -q -x -k "backward or fused or update or next" 2>&1 | tail -1
for r in 1 2; do
  for lib in "" paper_2506_06122_b200/lib/variants/librlo_bw1.so; do
    echo "== lib=${lib:-default(U4)}"
    RLO_LIB=$lib timeout 600 python tools/bench_update.py --forms two_pass --cases cfg2,cfg3,bf16_32k 2>&1 | grep '^{'
  done
done
