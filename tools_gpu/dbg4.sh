for v in "SPG_DBG_LR_SCALAR=1" "SPG_NO_GRAPH=1" "SPG_NO_GRAPH=1 SPG_SYNC_LAUNCH=1"; do
  echo "== $v"; env $v python tools_gpu/determinism.py smallgap 20 2>&1 | tail -3
done
echo "== old sweep"; SPG_DBG_LR_OLD=1 python tools_gpu/determinism.py sweep0.999 6 2>&1 | tail -3
