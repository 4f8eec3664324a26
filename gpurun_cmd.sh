RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_pfwd.so timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -2
for r in 1 2 3; do for L in cur pfwd; do RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$L.so timeout 300 python tools/bench_fwd.py 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$L r$r', 'entropy', d['entropy'], round(d['ms'],3), 'ms', round(d['gbs']), 'GB/s')"; done; done | tee gpurun_out/r2az_fwd.txt
