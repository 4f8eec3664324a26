RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_u4t640.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
bash tools/ab_bench.sh av 3 cur u4t640 u4t704 u5t576 | tee gpurun_out/r2av_ab.txt
