MODES="0:1,4:1,0:1,4:1" bash tools/probes/power_probe.sh 2>&1 | tee gpurun_out/r2_power_probe3.txt
