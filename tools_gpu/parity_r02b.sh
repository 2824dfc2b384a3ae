# GPU box: parity of the final build at BASELINE sizes against the reference run on the host cores
mkdir -p gpurun_out
python tests/parity_big.py --configs pr1,smallgap,stress0.9999,banded,sweep0.5,sweep0.9,sweep0.99,sweep0.999 --run-ref --patched-above 40000 --tag r02b > gpurun_out/parity_r02b.log 2>&1
tail -5 gpurun_out/parity_r02b.log; ls gpurun_out | grep parity
