./build/ffma2_probe
timeout 300 python -m pytest tests/test_gpu_edges.py -q -x 2>&1 | grep -E "^E |assert |passed|failed" | head -20
RLO_VOCAB_MATH=0 timeout 300 python -m pytest tests/test_gpu_edges.py -q -x -k extremes 2>&1 | tail -2
