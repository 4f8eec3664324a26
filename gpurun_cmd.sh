RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_ls768.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
AB_P1=1 bash tools/ab_bench.sh ar 3 cur ls768 tps768u4 | tee gpurun_out/r2ar_ab.txt
for r in 1 2; do for L in cur ls768; do
RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 300 python tools/bench_update.py --cases bf16_32k --P 3 --forms two_pass --iters 200 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$L r$r', d['case'], 'loss_ms', round(d['loss_ms'],3), 'loss_gbs', round(d['loss_gbs']))"
done; done | tee -a gpurun_out/r2ar_ab.txt
