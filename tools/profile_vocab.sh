# ncu evidence for the default vocab kernels (one GPU; plain run first, exit 0, then ncu).
./build/integration_test | tail -1
C2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C2 > gpurun_out/plain2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_v2.csv $C2 > gpurun_out/ncu_l2.log 2>&1; echo l2=$?
ncu --set full --clock-control none --import-source on -k regex:vocab_ -s 3 -c 1 -o gpurun_out/prof_cfg2_v2 $C2 > gpurun_out/ncu_f2.log 2>&1; echo f2=$?
$C3 > gpurun_out/plain3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_cfg3_v2.csv $C3 > gpurun_out/ncu_l3.log 2>&1; echo l3=$?
ncu --set full --clock-control none --import-source on -k regex:vocab_ -s 40 -c 1 -o gpurun_out/prof_cfg3_v2 $C3 > gpurun_out/ncu_f3.log 2>&1; echo f3=$?
