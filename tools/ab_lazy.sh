# Lazy running max (kMathLazy): bf16 mix 6 vs 7 (6 + lazy) vs 8 (1 + lazy); fp32 mix 1 vs 2 (1 + lazy).
# GPU suite under each lazy mix first (parity), then interleaved bench A/B.
set -u
RLO_VOCAB_MATH=7 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
RLO_VOCAB_MATH=2 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
one() {  # $1 math $2 config $3 steps
  RLO_VOCAB_MATH=$1 timeout 600 python bench.py --config $2 --steps $3 --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('math=$1 cfg$2', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz', d['clocks'].get('power_w'), 'W')"
}
for round in 1 2; do
  for m in 6 7 8; do one $m 3 3; done
  for m in 1 2; do one $m 2 10; done
done
