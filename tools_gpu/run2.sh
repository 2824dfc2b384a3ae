mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -18 gpurun_out/pytest_gpu.log
python tools_gpu/timeline.py sweep0.999 gpurun_out/timeline_sweep0.999.csv.gz > gpurun_out/timeline.log 2>&1; tail -1 gpurun_out/timeline.log
