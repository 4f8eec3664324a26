./build/trainer_step 2>&1 | tail -5
./build/integration_test | tail -2
bash tools/ab_bench.sh h 2 head nopf5 nopf6 | tee gpurun_out/r2j_ab.txt
