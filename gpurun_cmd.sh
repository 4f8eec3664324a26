timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -3
