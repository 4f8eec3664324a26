timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2j_bench_cfg3.json 2> gpurun_out/r2j_bench_cfg3.err; head -c 400 gpurun_out/r2j_bench_cfg3.json
