RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_bc.so timeout 900 python -m pytest tests/test_gpu_production.py tests/test_gpu_guards.py tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
bash tools/ab_bench.sh s 3 cur bc bcb3 | tee gpurun_out/r2s_ab.txt
