#!/bin/bash
# Sustained power / clock / bandwidth per work mode of tools/probes/power_probe.cu (one GPU).
cd "$(dirname "$0")/../.."
mkdir -p build gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/power_probe tools/probes/power_probe.cu || exit 1
# MODES: comma-separated mode:data pairs (data 0 = constant bytes, 1 = random bf16)
for md in $(echo "${MODES:-0:0,0:1,1:1,2:1,3:1,2:0}" | tr ',' ' '); do
  m=${md%:*}; d=${md#*:}
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > /tmp/pw_$m.csv &
  P=$!
  r=$(./build/power_probe $m 8 $d)
  kill $P; wait $P 2>/dev/null
  python3 - "$m" "$r" <<'PY'
import sys, statistics
m, r = sys.argv[1], sys.argv[2]
rows = [l.split(',') for l in open(f'/tmp/pw_{m}.csv') if l.strip()]
rows = rows[len(rows)//4: -2]  # steady part
mhz = statistics.median(float(x[0]) for x in rows); w = statistics.median(float(x[1]) for x in rows)
print(f"{r.strip()}  | median SM {mhz:.0f} MHz, {w:.0f} W, cap active {sum('Active' in x[2] for x in rows)}/{len(rows)}")
PY
done
