# ncu metrics of the bf16 fused-loss kernel for the three LDG layouts (U4, U4+prefetch, U8)
for l in 0 1 2; do
  RLO_VOCAB_LDG=$l timeout 300 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_selected,launch__registers_per_thread,sm__cycles_elapsed.avg.per_second,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum.per_second \
    --clock-control none -k regex:vocab_ldg -s 3 -c 1 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-p1 2>&1 | grep -E "vocab_ldg|duration|dram__|issue_active|warps_active|stalled|registers|cycles_elapsed|l1tex" | sed "s/^/layout=$l /"
done
