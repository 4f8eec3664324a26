# Warp reduction of the online state: max-first (default) vs pairwise combine per level (librlo_pairwise.so).
set -u
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do
  for lib in "" paper_2506_06122_b200/lib/variants/librlo_pairwise.so; do
    for P in 3 1; do
      RLO_LIB=$lib timeout 600 python tools/bench_update.py --forms two_pass --cases bf16_32k,cfg2 --P $P --iters 200 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('lib=${lib##*/} P=$P', d['case'], 'loss', round(d['loss_ms'], 3), 'ms', round(d['loss_gbs']), 'GB/s')"
    done
    RLO_LIB=$lib timeout 600 python bench.py --config 3 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; p=d['p1']; print('lib=${lib##*/} cfg3 P3', round(r['achieved']), 'GB/s | P1', round(p['achieved_gbs']), 'GB/s |', d['clocks']['sm_mhz'], 'MHz')"
  done
done
