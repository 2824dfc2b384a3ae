"""Size of the run-to-run differences in P (dense) for the small-gap config."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
c = CONFIGS["smallgap"]
A = make_input(c)
X = np.random.default_rng(0).standard_normal((c["n"], 8))
ref = None
for i in range(int(sys.argv[1])):
    if i % 3 == 0:
        S.load_library().spg_release_plan_cache()
    r = S.hqdwh(A, c["nmin"], c["eps"])
    rk, d = r.P.to_flat()
    Y = r.apply(X)
    if ref is None:
        ref = (rk.copy(), d.copy(), Y.copy())
    elif not np.array_equal(d, ref[1]):
        print("rep", i, "ranks equal", np.array_equal(rk, ref[0]), "max|d flat|", np.abs(d - ref[1]).max() if d.shape == ref[1].shape else None,
              "max |P X - P_ref X|", np.abs(Y - ref[2]).max(), flush=True)
    r.close()
print("done")
