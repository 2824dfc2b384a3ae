export SPG_DBG_DUMP=1 SPG_DBG_NO_TALLSPLIT=1
for v in "SPG_DBG_TV_OFF=1 SPG_DBG_W12_SYNC=1 SPG_DBG_CASC_SYNC=1" "SPG_CHOL_REFERENCE_ORDER=1" "SPG_NO_GRAPH=1"; do
  echo "== $v"; env $v python tools_gpu/determinism3.py smallgap 40 4 2>&1 | grep DUMP | sort | uniq -c | sort -k3,3 -k1,1nr | awk '$1>0'
done
