"""Size of the run-to-run differences in P (probe vectors) over many runs of a config."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
c = CONFIGS[sys.argv[1]]
A = make_input(c)
X = np.random.default_rng(0).standard_normal((c["n"], 8))
ref = None
nd = 0
worst = 0.0
for i in range(int(sys.argv[2])):
    if i % 3 == 0:
        S.load_library().spg_release_plan_cache()
    r = S.hqdwh(A, c["nmin"], c["eps"])
    rk, d = r.P.to_flat()
    Y = r.apply(X)
    if ref is None:
        ref = (rk.copy(), d.copy(), Y.copy())
    elif not (np.array_equal(rk, ref[0]) and np.array_equal(d, ref[1])):
        nd += 1
        e = float(np.abs(Y - ref[2]).max())
        worst = max(worst, e)
        print("rep", i, "ranks equal", np.array_equal(rk, ref[0]), "max |P X - P_ref X| %.3e" % e, flush=True)
    r.close()
print(sys.argv[1], "runs", sys.argv[2], "differing", nd, "worst %.3e" % worst)
