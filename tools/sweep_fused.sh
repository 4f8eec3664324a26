# Fused update pass sweep over the per-CTA slice budget (RLO_FUSED_SLICE_KB -> cluster size K).
for kb in 16 32 48 64 80; do
  RLO_FUSED_DEBUG=1 RLO_FUSED_SLICE_KB=$kb timeout 200 python tools/bench_update.py --iters 3 --forms fused > gpurun_out/sf.txt 2> gpurun_out/sf.err
  python -c "import sys,json
for l in open('gpurun_out/sf.txt'):
    d=json.loads(l); print('kb=$kb', d['case'], round(d['ms'],3), 'ms', round(d['gbs']), 'GB/s')"
  grep "fused pass" gpurun_out/sf.err | sort | uniq -c
done
