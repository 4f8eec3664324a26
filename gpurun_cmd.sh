timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python tools/bench_fwd.py 2>/dev/null
