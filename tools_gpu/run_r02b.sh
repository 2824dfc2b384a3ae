mkdir -p gpurun_out
./tools_gpu/ubench_lat > gpurun_out/ubench_lat.txt 2>&1; cat gpurun_out/ubench_lat.txt
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools_gpu/timeline.py sweep0.999 gpurun_out/timeline_sweep0.999.csv.gz > gpurun_out/timeline.log 2>&1; tail -1 gpurun_out/timeline.log
