timeout 600 python -m pytest tests/test_gpu_production.py tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2c_tests.log 2>&1; tail -3 gpurun_out/r2c_tests.log
bash tools/ab_bench.sh c 2 head reload m9 m8 r1 | tee gpurun_out/r2c_ab.txt
