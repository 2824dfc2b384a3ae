set -x
nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
python tests/parity_big.py --configs pr1,smallgap,stress0.9999,banded,sweep0.5,sweep0.9,sweep0.99,sweep0.999 --run-ref --patched-above 40000 --tag r02_chol > gpurun_out/parity_chol.log 2>&1
SPG_FIRST_GIVENS=1 python tests/parity_big.py --configs pr1,smallgap,stress0.9999,banded,sweep0.5,sweep0.9,sweep0.99,sweep0.999 --tag r02_givens > gpurun_out/parity_givens.log 2>&1
cp /tmp/parity_ref/*.json gpurun_out/ 2>/dev/null; mkdir -p gpurun_out/probes; cp /tmp/parity_ref/*_probe.npz gpurun_out/probes/
tail -5 gpurun_out/parity_chol.log gpurun_out/parity_givens.log
