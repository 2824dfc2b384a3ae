"""Magnitude and place of the first difference between two variants of the deferred Cholesky factor."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
c = CONFIGS["smallgap"]
A = make_input(c)
for dl in (0.3, 0.1, 3e-2, 1e-2, 3e-3, 1e-3, 1e-4, 1e-6, 1e-8):
    r = S.hqdwh(A, c["nmin"], c["eps"], dl)
    if r.iterations >= 3:
        break
    r.close()
X = r.U
r.close()
ctx = S.HodlrContext(c["n"], c["nmin"], c["eps"], 6)
ctx.upload(0, X)
ctx.op("multiply_upper", 1, 0, 0)
ctx.op("scale_shift", 1, alpha=4.175, beta=1.0)
ref = None
for rep in range(int(sys.argv[1])):
    ctx.op("cholesky_deferred", 3, 1)
    W = ctx.download(3)
    rk, d = W.to_flat()
    if ref is None:
        ref = (W, rk.copy(), d.copy())
        continue
    if np.array_equal(rk, ref[1]) and np.array_equal(d, ref[2]):
        continue
    print("rep", rep, "differs; ranks equal:", np.array_equal(rk, ref[1]))
    t = W.tree
    rows = []
    for i in range(len(t)):
        if t.leaf(i):
            D0, D1 = ref[0].dense[i], W.dense[i]
            if not np.array_equal(D0, D1):
                rows.append((t.begin[i], 99, i, "leaf", np.abs(D0 - D1).max(), np.abs(D0).max(), 0, 0))
        else:
            (U0, V0), (U1, V1) = ref[0].upper[i], W.upper[i]
            if U0.shape != U1.shape or not (np.array_equal(U0, U1) and np.array_equal(V0, V1)):
                B0, B1 = U0 @ V0.T, U1 @ V1.T
                rows.append((t.begin[i], -t.size[i], i, "W12", np.linalg.norm(B0 - B1, 2), np.linalg.norm(B0, 2), U0.shape[1], U1.shape[1]))
    rows.sort()
    for b, _, i, kind, dd, nn, k0, k1 in rows[:8]:
        print("   begin %6d node %4d size %5d %-4s |diff| %.3e  |ref| %.3e  ranks %d %d" % (b, i, t.size[i], kind, dd, nn, k0, k1))
    # structure of the largest W12 difference
    big = max((r for r in rows if r[3] == "W12"), key=lambda r: r[4])
    i = big[2]
    (U0, V0), (U1, V1) = ref[0].upper[i], W.upper[i]
    D = U0 @ V0.T - U1 @ V1.T
    sv = np.linalg.svd(D, compute_uv=False)
    print("   origin node", i, "singular values of the difference", sv[:5])
    rn = np.linalg.norm(D, axis=1); cn = np.linalg.norm(D, axis=0)
    print("   row-norm profile (32-row blocks):", np.array2string(np.array([rn[j:j + 32].max() for j in range(0, len(rn), 32)]), precision=2))
    print("   col-norm profile (32-col blocks):", np.array2string(np.array([cn[j:j + 32].max() for j in range(0, len(cn), 32)]), precision=2))
    s0 = np.linalg.svd(U0 @ V0.T, compute_uv=False); s1 = np.linalg.svd(U1 @ V1.T, compute_uv=False)
    print("   sigma tail ref", s0[20:30], "\n   sigma tail alt", s1[20:30])
    break
ctx.close()
