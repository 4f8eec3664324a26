# Decode screen at T != 1: share of the untempered exponentials on the FMA pipe
# (RLO_SCREEN_POLY 0 / 1 = default half / 2), rows/s by RLO_LIB A/B, two repeats.
set -u
for rep in 1 2; do
for lib in "" paper_2506_06122_b200/lib/variants/librlo_poly0.so paper_2506_06122_b200/lib/variants/librlo_poly2.so; do
  echo "== rep $rep lib=${lib:-poly1(default)}"
  RLO_LIB=$lib timeout 300 python tools/bench_next.py --only decode 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    if d['path'] == 'screened' and d['temperature'] != 1.0:
        print(d['rows'], d['V'], d['stride'], d['dtype'], d['temperature'], round(d['ms'], 3), 'ms', round(d['rows_per_s']/1e6, 2), 'M rows/s')"
done
done
RLO_LIB=paper_2506_06122_b200/lib/variants/librlo_poly2.so timeout 600 python -m pytest tests/test_gpu_next.py -q -x -k decode 2>&1 | tail -1
