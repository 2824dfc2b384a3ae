# GPU box: DRAM traffic of the recompression kernels over one headline projector WITHOUT ncu's cache
# flush between kernels (--cache-control none): what the L2 keeps between k_tsqr and k_apply stays
mkdir -p gpurun_out
SPG_ONE_REPS=1 timeout 3000 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
   --clock-control none --cache-control none -k regex:'k_tsqr|k_core_any|k_apply' --csv --log-file gpurun_out/ncu_trunc_traffic_nc.csv \
   python tools_gpu/one.py sweep0.999 > gpurun_out/ncu_trunc_traffic_nc.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_trunc_traffic_nc.log; wc -l gpurun_out/ncu_trunc_traffic_nc.csv
