export SPG_DBG_DUMP=1
for v in "SPG_X=1" "SPG_CHOL_REFERENCE_ORDER=1 SPG_DBG_NO_TALLSPLIT=1" "SPG_DBG_TV_OFF=1 SPG_DBG_W12_SYNC=1 SPG_DBG_CASC_SYNC=1 SPG_DBG_NO_TALLSPLIT=1" "SPG_NO_GRAPH=1 SPG_DBG_NO_TALLSPLIT=1"; do
  echo "== $v"; env $v timeout 400 python tools_gpu/determinism3.py smallgap 250 4 2>&1 | grep "DUMP W" | sort | uniq -c | sort -k1,1nr | head -3
done
