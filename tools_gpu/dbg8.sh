SPG_DBG_NO_TALLSPLIT=1 python tools_gpu/determinism2.py smallgap 25
