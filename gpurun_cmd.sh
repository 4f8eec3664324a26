AB_P1=1 AB_ARGS="--config 2" bash tools/ab_bench.sh am 3 cur f128 f512 | tee gpurun_out/r2am_ab.txt
