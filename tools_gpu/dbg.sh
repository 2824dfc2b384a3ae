mkdir -p gpurun_out
for v in "" "SPG_DBG_LR_OLD=1" "SPG_DBG_NO_EARLY=1" "SPG_FIRST_ITERATE=cholesky"; do
  echo "== $v"; env $v python -m pytest tests/test_gpu_parity.py -x -q -k "smallgap_config" 2>&1 | tail -2
done
