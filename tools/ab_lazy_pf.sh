# bf16: mix 6 (U4) vs mix 7 (lazy max + U4 prefetch), P=3 pass and the P=1 (actor-only) leg; suite under mix 7 first.
set -u
RLO_VOCAB_MATH=7 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
one() {  # $1 math $2 config
  RLO_VOCAB_MATH=$1 timeout 600 python bench.py --config $2 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; p=d['p1']; print('math=$1 cfg$2 P3', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s | P1', round(p['avg_launch_ms'],3), 'ms', round(p['achieved_gbs']), 'GB/s |', d['clocks']['sm_mhz'], 'MHz')"
}
for round in 1 2 3; do for m in 6 7; do one $m 3; done; done
for m in 6 7; do one $m 4; done
