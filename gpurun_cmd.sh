RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_bc.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -2
bash tools/ab_bench.sh aw 3 cur bc | tee gpurun_out/r2aw_ab.txt
C3="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-p1"
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_bc.so timeout 1200 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:vocab_ -s 40 -c 1 --csv $C3 2>/dev/null | grep -E "inst_executed|duration" | tail -2
