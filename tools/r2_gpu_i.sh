#!/bin/bash
# Round-2 GPU call i (the final round-2 library: lockstep kernel at 768 threads per SM): smoke, full -m gpu suite, bench cfg3 / cfg2 /
# reference arm, ncu launch list + --set full captures of the cfg3 and cfg2 vocab kernels (plain runs exit 0 first).
cd "$(dirname "$0")/.."
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2i_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r2i_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 900 > $O/r2i_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r2i_gputest.log
timeout 900 python bench.py > $O/r2i_bench_cfg3.json 2> $O/r2i_bench_cfg3.err
timeout 600 python bench.py --config 2 > $O/r2i_bench_cfg2.json 2> $O/r2i_bench_cfg2.err
timeout 900 python bench.py --config 4 > $O/r2i_bench_cfg4.json 2> $O/r2i_bench_cfg4.err
timeout 900 python bench.py --config 5 > $O/r2i_bench_cfg5.json 2> $O/r2i_bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/r2i_ref_cfg3.json 2> $O/r2i_ref_cfg3.err
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-p1"
$C3 > $O/r2i_plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r2i_launches_cfg3.csv $C3 > $O/r2i_ncu_l3.log 2>&1; echo l3=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:vocab_ -s 40 -c 1 -o $O/r2i_prof_cfg3 $C3 > $O/r2i_ncu_f3.log 2>&1; echo f3=$?
C2="python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-p1"
$C2 > $O/r2i_plain2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:vocab_ -s 3 -c 1 -o $O/r2i_prof_cfg2 $C2 > $O/r2i_ncu_f2.log 2>&1; echo f2=$?
tail -2 $O/r2i_smoke.log; tail -3 $O/r2i_gputest.log
