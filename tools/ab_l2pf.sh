# L2 bulk prefetch ahead of the LDG stream (RLO_VOCAB_L2PF = batches ahead; 0 = off).
set -u
RLO_VOCAB_L2PF=2 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
one() {  # $1 l2pf $2 config $3 steps $4 math
  RLO_VOCAB_MATH=$4 RLO_VOCAB_L2PF=$1 timeout 600 python bench.py --config $2 --steps $3 --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('l2pf=$1 math=$4 cfg$2', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz', d['clocks'].get('power_w'), 'W')"
}
for round in 1 2; do
  for p in 0 1 2 4 8; do one $p 3 3 6; done
  one 2 3 3 7
  for p in 0 2 4; do one $p 2 10 1; done
done
