for L in dw4 dw16 bw32; do RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_production.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1; done
for r in 1 2; do for L in cur dw4 dw16; do
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 600 python tools/bench_next.py --only decode 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['path']=='screened': print('$L r$r', d['rows'], d['V'], d['stride'], d['dtype'], d['temperature'], round(d['rows_per_s']/1e6,3))"
done; done | tee gpurun_out/r2aj_dec.txt
for r in 1 2; do for L in cur bw32 bw64; do
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 300 python tools/bench_update.py --cases cfg3,bf16_32k --forms two_pass --iters 200 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$L r$r', d['case'], 'backward_ms', round(d['backward_ms'],3), 'loss_ms', round(d['loss_ms'],3))"
done; done | tee gpurun_out/r2aj_bw.txt
