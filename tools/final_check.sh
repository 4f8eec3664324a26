# Final round-1 check with the shipped build on a 2-GPU box: the whole GPU suite
# (multi-GPU tests included), smoke, the default bench line at N=1 and N=2.
set -u
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 300 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo n1 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 > gpurun_out/final_n2.json 2> gpurun_out/final_n2.err; echo n2 rc=$?
