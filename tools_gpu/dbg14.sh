export SPG_DBG_DUMP=1
for v in "SPG_X=1" "SPG_DBG_NO_TALLSPLIT=1"; do
  echo "== $v"; env $v python tools_gpu/determinism3.py smallgap 60 4 2>&1 | grep "DUMP W" | sort | uniq -c | sort -k1,1nr
done
unset SPG_DBG_DUMP
python tools_gpu/determinism.py smallgap 30 2>&1 | tail -2
python tools_gpu/determinism.py sweep0.999 10 2>&1 | tail -2
