# Round-end measurement (v7 code): round_end.sh, then ncu --set full of the default bf16 vocab
# kernel (cfg3) and of the decode screen kernel.  Plain runs exit 0 before any ncu run.
set -u
bash tools/round_end.sh
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vocab_ -s 40 -c 1 -o gpurun_out/prof_cfg3_v7 $C3 > gpurun_out/ncu_f3_v7.log 2>&1; echo f3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_screen -s 2 -c 1 -o gpurun_out/prof_decode_v7 python tools/probes/decode_probe.py > gpurun_out/ncu_dec_v7.log 2>&1; echo dec=$?
