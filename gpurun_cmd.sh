timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2ad_n2.out 2> gpurun_out/r2ad_n2.err; echo rc=$?
wc -l gpurun_out/r2ad_n2.out; head -c 300 gpurun_out/r2ad_n2.out; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/r2ad_ref_n2.out 2> gpurun_out/r2ad_ref_n2.err; echo rc=$?
wc -l gpurun_out/r2ad_ref_n2.out; head -c 300 gpurun_out/r2ad_ref_n2.out; echo
