mkdir -p gpurun_out
python tools_gpu/determinism.py smallgap 60 2>&1 | tail -2
python tools_gpu/determinism.py sweep0.999 8 2>&1 | tail -2
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools_gpu/timeline.py sweep0.999 gpurun_out/timeline_sweep0.999.csv.gz > gpurun_out/timeline.log 2>&1; tail -1 gpurun_out/timeline.log
