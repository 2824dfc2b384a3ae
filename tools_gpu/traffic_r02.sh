# GPU box: DRAM traffic of the recompression kernels over one headline projector (ncu replays each
# kernel for the three metrics; the kernels are filtered by name so the capture fits its window)
mkdir -p gpurun_out
SPG_ONE_REPS=1 timeout 3000 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none -k regex:'k_tsqr|k_core_any|k_apply' --csv --log-file gpurun_out/ncu_trunc_traffic.csv \
   python tools_gpu/one.py sweep0.999 > gpurun_out/ncu_trunc_traffic.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_trunc_traffic.log; wc -l gpurun_out/ncu_trunc_traffic.csv
