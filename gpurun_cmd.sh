RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_rpf.so timeout 900 python -m pytest tests/test_gpu_production.py tests/test_gpu_guards.py tests/test_gpu_packed.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
AB_P1=1 bash tools/ab_bench.sh k 2 head rpf | tee gpurun_out/r2n_ab.txt
AB_ARGS="--config 2" bash tools/ab_bench.sh k2 2 head rpf | tee -a gpurun_out/r2n_ab.txt
