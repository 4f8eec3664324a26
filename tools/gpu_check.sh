# Round-1 GPU check: parity suite under the default kernels and each vocab variant.
timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for v in "ldg 0" "ldg 3" "tma 1" "tma 2"; do set -- $v
  echo "== RLO_VOCAB_IMPL=$1 RLO_VOCAB_MATH=$2"
  RLO_VOCAB_IMPL=$1 RLO_VOCAB_MATH=$2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | grep -E "passed|failed|Error|assert" | head -8
done
./build/integration_test | tail -12
