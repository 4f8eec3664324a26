timeout 900 python -m pytest tests/test_gpu_guards.py tests/test_gpu_integration.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2d_tests.log 2>&1; tail -15 gpurun_out/r2d_tests.log
