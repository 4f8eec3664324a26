#!/bin/bash
# Round-2 GPU check: smoke, the full -m gpu suite, the spike tests against the
# round-1 library (expected to FAIL there), bench cfg3 (default) / cfg2 / reference arm.
cd "$(dirname "$0")/.."
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/r2a_nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r2a_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 900 > $O/r2a_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r2a_gputest.log
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_r1.so timeout 600 python -m pytest tests/test_gpu_production.py -m gpu -q -p no:cacheprovider -k spike -rf > $O/r2a_spike_r1lib.log 2>&1; echo "rc=$?" >> $O/r2a_spike_r1lib.log
timeout 900 python bench.py > $O/r2a_bench_cfg3.json 2> $O/r2a_bench_cfg3.err; echo "rc=$?" >> $O/r2a_bench_cfg3.err
timeout 600 python bench.py --config 2 > $O/r2a_bench_cfg2.json 2> $O/r2a_bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/r2a_ref_cfg3.json 2> $O/r2a_ref_cfg3.err
tail -3 $O/r2a_gputest.log; tail -2 $O/r2a_spike_r1lib.log; cat $O/r2a_bench_cfg3.json | head -c 600
