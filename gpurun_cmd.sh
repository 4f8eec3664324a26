bash tools/probes/power_probe.sh 2>&1 | tee gpurun_out/r2_power_probe2.txt
