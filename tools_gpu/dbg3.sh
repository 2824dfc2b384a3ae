for v in "SPG_X=1" "SPG_DBG_FULL_Z=1" "SPG_DBG_LR_OLD=1"; do
  echo "== $v"; env $v python tools_gpu/determinism.py smallgap 30 2>&1 | tail -4
done
python tools_gpu/determinism.py sweep0.999 8 2>&1 | tail -4
