# Decode screen: a-posteriori argument-error bound (sum w|t| of the row) vs the
# worst case total*log2(V): parity, screen fail rates, rows/s (RLO_LIB A/B).
set -u
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_edges.py -q -x 2>&1 | tail -1
for lib in "" paper_2506_06122_b200/lib/variants/librlo_oldscreen.so; do
  echo "== lib=${lib:-new(apost)}"
  for v in 152064 32000; do RLO_LIB=$lib V=$v ROWS=8192 timeout 300 python tools/probes/decode_probe.py 2>&1 | grep -v "^$"; done
  for rep in 1 2; do
  RLO_LIB=$lib timeout 300 python tools/bench_next.py --only decode 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['rows'], d['V'], d['stride'], d['dtype'], d['temperature'], d['path'], round(d['ms'], 3), 'ms', round(d['rows_per_s']/1e6, 2), 'M rows/s', round(d['gbs_one_pass']), 'GB/s')"
  done
done
