bash tools/ab_bench.sh e 2 head un8 un8m9 un4 | tee gpurun_out/r2f_ab.txt
