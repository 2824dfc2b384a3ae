export SPG_DBG_DUMP=1 SPG_DBG_NO_TALLSPLIT=1 SPG_CHOL_REFERENCE_ORDER=1
for v in "SPG_DBG_LR_SCALAR=2" "SPG_DBG_LR_OLD=1" "SPG_X=1"; do
  echo "== $v"; env $v python tools_gpu/determinism3.py smallgap 60 4 2>&1 | grep "DUMP W" | sort | uniq -c | sort -k1,1nr
done
