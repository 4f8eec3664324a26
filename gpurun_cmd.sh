MODES="2:1,5:1,6:1,2:1,5:1,6:1" bash tools/probes/power_probe.sh 2>&1 | tee gpurun_out/r2_power_probe4.txt
