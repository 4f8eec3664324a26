timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -8
bash tools/ab_bench.sh w 2 cur new | tee gpurun_out/r2w_ab.txt
