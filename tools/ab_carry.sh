# Next-tensor batch carried across the streams of a row (default) vs none (librlo_nocarry.so); cfg3/cfg4 bench.
set -u
RLO_VOCAB_MATH= timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
one() {  # $1 lib $2 config
  RLO_LIB=$1 timeout 600 python bench.py --config $2 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; p=d['p1']; print('lib=${1##*/} cfg$2 P3', round(r['avg_launch_ms'],3), 'ms', round(r['achieved']), 'GB/s | P1', round(p['avg_launch_ms'],3), 'ms', round(p['achieved_gbs']), 'GB/s |', d['clocks']['sm_mhz'], 'MHz')"
}
for round in 1 2 3; do one "" 3; one paper_2506_06122_b200/lib/variants/librlo_nocarry.so 3; done
