for v in "SPG_DBG_NO_TALLSPLIT=1" "SPG_CHOL_REFERENCE_ORDER=1" "SPG_CHOL_REFERENCE_ORDER=1 SPG_DBG_NO_TALLSPLIT=1"; do
  echo "== $v"; env $v python tools_gpu/determinism.py smallgap 30 2>&1 | tail -2
done
