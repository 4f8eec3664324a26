RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_p1df.so timeout 900 python -m pytest tests/test_gpu_production.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
AB_P1=1 bash tools/ab_bench.sh ak 3 cur p1df | tee gpurun_out/r2ak_ab.txt
