AB_P1=1 bash tools/ab_bench.sh at 2 cur o768 | tee gpurun_out/r2at_ab.txt
AB_P1=1 AB_ARGS="--config 2" bash tools/ab_bench.sh at2 2 cur o768 | tee -a gpurun_out/r2at_ab.txt
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_dm3.so timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -q -p no:cacheprovider -k decode 2>&1 | tail -1
for r in 1 2; do for L in cur dm3; do
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 600 python tools/bench_next.py --only decode 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['path']=='screened' and d['V']==152064: print('$L r$r', d['rows'], d['V'], d['temperature'], round(d['rows_per_s']/1e6,3))"
done; done | tee -a gpurun_out/r2at_ab.txt
