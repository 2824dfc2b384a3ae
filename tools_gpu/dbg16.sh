export SPG_DBG_DUMP=1
for c in none leaf block wtr tv split; do
  echo "== delay $c"; SPG_DBG_DELAY=$c SPG_DBG_DELAY_US=300 timeout 300 python tools_gpu/determinism3.py smallgap 8 4 2>&1 | grep "DUMP W" | sort | uniq -c | sort -k1,1nr | head -4
done
