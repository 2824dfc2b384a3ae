"""Per-node localisation of the Cholesky nondeterminism on the smallgap iteration-4 input:
python tools_gpu/chol_race.py reps"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

reps = int(sys.argv[1])
c = CONFIGS["smallgap"]
A = make_input(c)
r0 = S.hqdwh(A, c["nmin"], c["eps"])
ls = [min(r0.l0, 1 - 1e-12)] + [d.l for d in r0.per_iteration]
cs = [d.c for d in r0.per_iteration]
r0.close()
delta = 0.5 * (abs(1 - ls[2]) + abs(1 - ls[3]))
r = S.hqdwh(A, c["nmin"], c["eps"], delta)
assert r.iterations == 3
X3 = r.U
n, nmin = c["n"], c["nmin"]
ctx = S.HodlrContext(n, nmin, c["eps"], 4)
ctx.upload(0, X3)
ctx.op("multiply_upper", 1, 0, 0)
ctx.op("scale_shift", 1, alpha=cs[3], beta=1.0)
T = ctx.tree
depth = np.zeros(len(T), dtype=int)
for i in range(len(T)):
    if not T.leaf(i):
        depth[T.left[i]] = depth[T.right[i]] = depth[i] + 1
ref = None
for k in range(reps):
    ctx.op(os.environ.get("CHOL_OP", "cholesky_deferred"), 2, 1)
    W = ctx.download(2)
    if ref is None:
        ref = W
        continue
    bad = []
    for i in range(len(T)):
        if T.leaf(i):
            if not np.array_equal(W.dense[i], ref.dense[i]):
                bad.append(("leaf", i, int(T.begin[i]), float(np.abs(W.dense[i] - ref.dense[i]).max())))
        else:
            U1, V1 = W.upper[i]
            U0, V0 = ref.upper[i]
            if U1.shape != U0.shape or not (np.array_equal(U1, U0) and np.array_equal(V1, V0)):
                d = float(np.abs(U1 @ V1.T - U0 @ V0.T).max()) if U1.shape[1] and U0.shape[1] else -1
                bad.append(("W12", i, int(depth[i]), int(T.begin[i]), U1.shape[1], U0.shape[1], d))
    if bad:
        print(f"rep {k}: {len(bad)} nodes differ; first (preorder): {bad[:6]}", flush=True)
print("done")
