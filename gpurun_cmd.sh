AB_P1=1 bash tools/ab_bench.sh ai 2 cur u2 u4 p1u8 | tee gpurun_out/r2ai_ab.txt
