RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_pls1.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
bash tools/ab_bench.sh ba 2 cur pls1 pls2 | tee gpurun_out/r2ba_ab.txt
