# bf16 cfg3 with the copy-forward prefetch layout: mix 7 (25% FMA-pipe exp2 on old/ref) vs mix 8 (all MUFU).
set -u
one() {  # $1 math $2 config
  RLO_VOCAB_MATH=$1 timeout 600 python bench.py --config $2 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; p=d['p1']; print('math=$1 cfg$2 P3', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s | P1', round(p['avg_launch_ms'],3), 'ms', round(p['achieved_gbs']), 'GB/s |', d['clocks']['sm_mhz'], 'MHz')"
}
for round in 1 2 3; do one 7 3; one 9 3; one 10 3; done
