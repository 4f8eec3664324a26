# L2-residency probe for re-reading the actor row in a fused update pass.
for cfg in "32768 304128 1 512 1" "32768 304128 1 512 0" "32768 304128 2 256 1" "131072 128000 2 256 1" "131072 128000 2 256 0" "131072 128000 4 256 1"; do
  ./build/l2_probe $cfg | tail -2 | head -1
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -c 1 ./build/l2_probe 32768 304128 1 512 1 2>&1 | grep -E "dram__|duration"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -c 1 ./build/l2_probe 32768 304128 1 512 0 2>&1 | grep -E "dram__|duration"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -c 1 ./build/l2_probe 131072 128000 2 256 1 2>&1 | grep -E "dram__|duration"
