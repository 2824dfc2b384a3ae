"""Determinism per iteration count: python tools_gpu/determinism2.py config reps"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
c = CONFIGS[name]
A = make_input(c)
r0 = S.hqdwh(A, c["nmin"], c["eps"])
ls = [min(r0.l0, 1 - 1e-12)] + [d.l for d in r0.per_iteration]
r0.close()
for it in range(1, len(ls)):
    delta = 0.5 * (abs(1 - ls[it - 1]) + abs(1 - ls[it]))
    ref, bad = None, 0
    for i in range(reps):
        r = S.hqdwh(A, c["nmin"], c["eps"], delta)
        assert r.iterations == it
        rk, d = r.U.to_flat()
        d = d.copy()
        if ref is None:
            ref = (rk.copy(), d)
        elif not (np.array_equal(rk, ref[0]) and np.array_equal(d, ref[1])):
            bad += 1
        r.close()
    print(f"{name} iterations={it}: {bad}/{reps - 1} differ", flush=True)
