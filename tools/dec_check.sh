set -u
timeout 600 python -m pytest tests/test_gpu_next.py -q -x -k decode 2>&1 | tail -1
for v in 152064 32000; do V=$v ROWS=8192 python tools/probes/decode_probe.py 2>&1 | grep -v "^$"; done
timeout 300 python tools/bench_next.py --only decode 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['rows'], d['V'], d['stride'], d['dtype'], d['temperature'], d['path'], round(d['ms'], 3), 'ms', round(d['rows_per_s']/1e6, 2), 'M rows/s', round(d['gbs_one_pass']), 'GB/s')"
