AB_P1=1 bash tools/ab_bench.sh j 2 head p1m4 p1m8 | tee gpurun_out/r2m_ab.txt
