# The single-GPU suite under every selectable vocab-pass variant (each must pass like the default).
for v in "" "RLO_VOCAB_IMPL=tma" "RLO_VOCAB_EPI=1" "RLO_VOCAB_LF=1" "RLO_VOCAB_LDG=1" "RLO_VOCAB_LDG=2" "RLO_VOCAB_LDG=4" "RLO_VOCAB_MATH=1" "RLO_VOCAB_MATH=4" "RLO_FUSED_NB=3"; do
  echo "== ${v:-default}"; env $v timeout 500 python -m pytest tests -m gpu -q -x -k "not multi and not integration" 2>&1 | tail -1
done
