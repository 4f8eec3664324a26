for L in t128 t512; do RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 900 python -m pytest tests/test_gpu_production.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1; done
AB_P1=1 bash tools/ab_bench.sh ae 2 cur t128 t512 | tee gpurun_out/r2ae_ab.txt
