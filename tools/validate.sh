set -u
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/val_cfg2.json 2> gpurun_out/val_cfg2.err; echo cfg2 rc=$?
tail -c 600 gpurun_out/val_cfg2.json
