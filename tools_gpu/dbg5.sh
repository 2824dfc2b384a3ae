python tools_gpu/determinism.py smallgap 40 2>&1 | tail -3
python tools_gpu/determinism.py sweep0.999 10 2>&1 | tail -3
python tools_gpu/determinism.py banded 6 2>&1 | tail -3
