# bf16 cfg3: instruction mix (6 default, 7 = 6 + lazy max) x LDG layout (0 = U4, 1 = U4 + prefetch, 2 = U8).
set -u
one() {  # $1 math $2 ldg
  RLO_VOCAB_MATH=$1 RLO_VOCAB_LDG=$2 timeout 600 python bench.py --config 3 --steps 3 --no-cpu-baseline --no-e2e --no-p1 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('math=$1 ldg=$2', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], 'MHz', d['clocks'].get('power_w'), 'W')"
}
for round in 1 2; do
  for m in 6 7; do for l in 0 1 2; do one $m $l; done; done
done
