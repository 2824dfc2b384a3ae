"""Run-to-run determinism of the projector (races show up as differing bits):
python tools_gpu/determinism.py config reps"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
c = CONFIGS[name]
A = make_input(c)
ref = None
bad = 0
for i in range(reps):
    r = S.hqdwh(A, c["nmin"], c["eps"])
    rk, d = r.P.to_flat()
    d = d.copy()
    if ref is None:
        ref = (rk.copy(), d)
    else:
        same_r = np.array_equal(rk, ref[0])
        diff = np.abs(d - ref[1]).max() if same_r and d.shape == ref[1].shape else float("inf")
        if diff != 0.0:
            bad += 1
            print(f"rep {i}: ranks equal {same_r}, max |dP| {diff:.3e}", flush=True)
    r.close()
print(f"{name}: {reps} reps, {bad} differing from the first")
