"""Which matrix of iteration `it` diverges first: python tools_gpu/determinism3.py config reps it"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name, reps, it = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = CONFIGS[name]
A = make_input(c)
r0 = S.hqdwh(A, c["nmin"], c["eps"])
ls = [min(r0.l0, 1 - 1e-12)] + [d.l for d in r0.per_iteration]
r0.close()
delta = 0.5 * (abs(1 - ls[it - 1]) + abs(1 - ls[it]))
for i in range(reps):
    r = S.hqdwh(A, c["nmin"], c["eps"], delta)
    r.close()
