export SPG_DBG_DUMP=1 SPG_DBG_NO_TALLSPLIT=1 SPG_CHOL_REFERENCE_ORDER=1
for v in "SPG_DBG_BLOCKS_AFTER_LEAF=1" "SPG_DBG_LEAF_AFTER_BLOCKS=1" "SPG_X=1"; do
  echo "== $v"; env $v python tools_gpu/determinism3.py smallgap 50 4 2>&1 | grep "DUMP W" | sort | uniq -c | sort -k1,1nr
done
