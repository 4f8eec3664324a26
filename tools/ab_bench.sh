#!/bin/bash
# A/B of librlo builds on the cfg3 bench (P = 3 vocab pass), alternating rounds.
# usage: tools/ab_bench.sh TAG ROUNDS lib1 lib2 ...   (names under paper_2506_06122_b200/lib/variants/librlo_<name>.so)
cd "$(dirname "$0")/.."
TAG=$1; R=$2; shift 2
O=gpurun_out/ab_$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  for n in "$@"; do
    RLO_LIB=$PWD/paper_2506_06122_b200/lib/variants/librlo_$n.so timeout 300 python bench.py --steps 5 --warmup 3 \
      --no-cpu-baseline --no-e2e $([ -n "$AB_P1" ] || echo --no-p1) ${AB_ARGS} > $O/${n}_$r.json 2> $O/${n}_$r.err
    python3 -c "
import json,sys
d=json.load(open('$O/${n}_$r.json')); c=d['clocks']; r=d['roofline']
p1=d.get('p1') or {}
print('$n r$r', round(r['achieved']), round(r['frac'],4), c['sm_mhz'], c.get('power_w'), round(r['avg_launch_ms'],3),
      'p1', round(p1.get('achieved_gbs', 0)))" 2>/dev/null || echo "$n r$r FAILED"
  done
done
