SPG_DBG_DUMP=1 SPG_DBG_NO_TALLSPLIT=1 python tools_gpu/determinism3.py smallgap 30 4 2>&1 | grep DUMP | sort | uniq -c | sort -k3,3 -k1,1nr
