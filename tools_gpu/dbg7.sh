export SPG_DBG_NO_TALLSPLIT=1
for v in "SPG_DBG_TV_OFF=1" "SPG_DBG_W12_SYNC=1" "SPG_DBG_CASC_SYNC=1" "SPG_DBG_TV_OFF=1 SPG_DBG_W12_SYNC=1 SPG_DBG_CASC_SYNC=1"; do
  echo "== $v"; env $v python tools_gpu/determinism.py smallgap 30 2>&1 | tail -2
done
