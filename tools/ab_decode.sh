# Screened fp32 decode: parity (decode tests), then rows/s for build variants (RLO_LIB).
set -u
timeout 600 python -m pytest tests/test_gpu_next.py -q -x -k decode 2>&1 | tail -1
for lib in "" paper_2506_06122_b200/lib/variants/librlo_u4b3.so paper_2506_06122_b200/lib/variants/librlo_u2b4.so paper_2506_06122_b200/lib/variants/librlo_u3b4.so; do
  echo "== lib=${lib:-default(u4b4)}"
  RLO_LIB=$lib timeout 300 python tools/bench_next.py --only decode 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['rows'], d['V'], d['dtype'], d['temperature'], d['path'], round(d['ms'], 3), 'ms', round(d['rows_per_s']/1e6, 2), 'M rows/s', round(d['gbs_one_pass']), 'GB/s')"
done
