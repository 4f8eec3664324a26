for L in pfb3 pfu2 pfu3; do RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_production.py -k "decode" -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -1; done
for r in 1 2; do for L in dec1 pf pfb3 pfu2 pfu3; do
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 600 python tools/bench_next.py --only decode 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['path']=='screened': print('$L r$r', d['rows'], d['V'], d['stride'], d['dtype'], d['temperature'], round(d['rows_per_s']/1e6,3))"
done; done | tee gpurun_out/r2aa_dec.txt
