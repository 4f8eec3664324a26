RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_f1t128.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
AB_P1=1 AB_ARGS="--config 2" bash tools/ab_bench.sh an 3 cur f1t128 f1t64 | tee gpurun_out/r2an_ab.txt
