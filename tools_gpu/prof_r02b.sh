# GPU box: (1) complete ncu launch list of one headline projector of the current build,
# (2) ncu --set full of one mid-run launch of the main kernels
mkdir -p gpurun_out
SPG_ONE_REPS=1 timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/ncu_launches_r02.csv python tools_gpu/one.py sweep0.999 > gpurun_out/ncu_launches_r02.log 2>&1
echo "launch list rc=$?"; wc -l gpurun_out/ncu_launches_r02.csv
for k in k_core_any:1500 k_tsqr:2500 k_apply:2500 k_gemm:3000 k_leaf_chol4:600 k_hsolve2:900; do
  name=${k%%:*}; skip=${k#*:}
  SPG_ONE_REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${name}\$" --launch-skip $skip -c 1 \
      -o gpurun_out/ncu_full_r02b_$name -f python tools_gpu/one.py sweep0.999 > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
ls -la gpurun_out | tail -12
