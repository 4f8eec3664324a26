RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_w256.so timeout 900 python -m pytest tests/test_gpu_production.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_guards.py -m gpu -q -p no:cacheprovider -x -rf 2>&1 | tail -3
bash tools/ab_bench.sh g 2 head w256 | tee gpurun_out/r2h_ab.txt
AB_ARGS="--config 2" bash tools/ab_bench.sh g2 2 head w256 | tee -a gpurun_out/r2h_ab.txt
