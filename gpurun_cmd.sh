timeout 1200 python -m pytest tests/test_gpu_production.py tests/test_gpu_guards.py tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2q_tests.txt; cat gpurun_out/r2q_tests.txt
bash tools/ab_bench.sh q 2 head cur ls3b3 | tee gpurun_out/r2q_ab.txt
