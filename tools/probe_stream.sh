# Memory ceiling of the vocab pass's access pattern (tools/probes/stream_probe.cu) next to the pass itself.
set -u
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 200 > gpurun_out/probe_clk.csv &
SMI=$!
for u in 4 8 2; do ./build/stream_probe 32768 304128 $u; done
for u in 4 8; do ./build/stream_probe 65536 128000 $u; done
./build/stream_probe 32768 64000 4
kill $SMI
sort -n gpurun_out/probe_clk.csv | awk -F, '{print $1}' | uniq -c | sort -rn | head -5
