# GPU box: CUPTI kernel timeline of one headline projector + ncu --set full of the main kernels
mkdir -p gpurun_out
python tools_gpu/timeline.py sweep0.999 gpurun_out/timeline_sweep0.999.csv.gz > gpurun_out/timeline.log 2>&1; tail -2 gpurun_out/timeline.log
python tools_gpu/timeline.py banded gpurun_out/timeline_banded.csv.gz >> gpurun_out/timeline.log 2>&1; tail -1 gpurun_out/timeline.log
for k in k_leaf_chol4:300 k_core_any:2000 k_tsqr:2000 k_apply:2000 k_hsolve2:300 k_gemm:3000 k_leaf_trsm_rows:50 k_lowrank_update:300; do
  name=${k%%:*}; skip=${k#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${name}\$" --launch-skip $skip -c 1 \
      -o gpurun_out/ncu_full_$name -f python tools_gpu/one.py sweep0.999 > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
ls -la gpurun_out
