AB_P1=1 bash tools/ab_bench.sh al 2 cur p1m4 m5 m9 | tee gpurun_out/r2al_ab.txt
