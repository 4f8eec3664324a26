#!/bin/bash
# Round-2 GPU call b: integration binary, bench cfg3 (default) + cfg2, then the
# ncu launch list and one --set full capture of the cfg3 vocab kernel (the
# plain command exits 0 first).
cd "$(dirname "$0")/.."
O=gpurun_out
./build/integration_test > $O/r2b_integration.log 2>&1; echo "rc=$?" >> $O/r2b_integration.log
timeout 900 python bench.py > $O/r2b_bench_cfg3.json 2> $O/r2b_bench_cfg3.err; echo "rc=$?" >> $O/r2b_bench_cfg3.err
timeout 600 python bench.py --config 2 > $O/r2b_bench_cfg2.json 2> $O/r2b_bench_cfg2.err
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-p1"
$C3 > $O/r2b_plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r2b_launches_cfg3.csv $C3 > $O/r2b_ncu_l3.log 2>&1; echo l3=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:vocab_ -s 40 -c 1 -o $O/r2b_prof_cfg3 $C3 > $O/r2b_ncu_f3.log 2>&1; echo f3=$?
tail -2 $O/r2b_integration.log; head -c 400 $O/r2b_bench_cfg3.json
