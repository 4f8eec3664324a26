bash tools/ab_bench.sh i 2 head h1 h2 h3 | tee gpurun_out/r2l_ab.txt
