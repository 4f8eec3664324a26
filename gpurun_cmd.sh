bash tools/ab_bench.sh as 3 cur l704 l832 | tee gpurun_out/r2as_ab.txt
