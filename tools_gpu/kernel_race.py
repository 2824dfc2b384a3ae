"""Intra-kernel race hunt: identical component operations run in several host threads at once
(separate engines, separate memory): any run-to-run bit difference of an op's output comes from
inside its kernels (timing under contention), not from cross-stream ordering.
    python tools_gpu/kernel_race.py [threads] [reps]"""
import os, sys, threading, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 3
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 15
g = np.random.default_rng(7)


def lowrank(p, s, k, r):
    Q1 = np.linalg.qr(g.standard_normal((p, r)))[0]; Q2 = np.linalg.qr(g.standard_normal((s, r)))[0]
    sig = np.logspace(0, -12, r)
    M = g.standard_normal((r, k))
    return (Q1 * sig) @ M, Q2 @ np.linalg.pinv(M).T


def h(*arrs):
    m = hashlib.sha1()
    for a in arrs:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:12]


cases = {}
for name, (p, s, k, r) in {"trunc k40 256": (256, 256, 40, 30), "trunc k100 256": (256, 256, 100, 60),
                           "trunc k60 256": (256, 256, 60, 45), "trunc k40 4096": (4096, 4096, 40, 30),
                           "trunc k100 4096": (4096, 4096, 100, 60)}.items():
    U, V = lowrank(p, s, k, r)
    cases[name] = (lambda U=U, V=V: h(*S.truncate(U, V, 1e-10)))

A = S.dimer_chain(4096, 1.0, 0.999, 0.0, 1)


def ctx_ops(which):
    def run():
        ctx = S.HodlrContext(4096, 256, 1e-10, 6)
        ctx.from_banded(0, A)
        ctx.op("scale_shift", 0, alpha=0.5, beta=0.0)
        ctx.op("multiply_upper", 1, 0, 0)
        out = {}
        out["multiply"] = h(*ctx.download(1).to_flat())
        ctx.op("scale_shift", 1, alpha=50.0, beta=1.0)
        for it in range(3):   # a few squarings to raise the ranks
            ctx.op("multiply", 2, 0, 0)
            ctx.op("axpby", 0, 0, 2, 1.5, -0.5)
            ctx.op("symmetrize", 0)
        out["axpby_sym"] = h(*ctx.download(0).to_flat())
        ctx.op("multiply_upper", 1, 0, 0)
        ctx.op("scale_shift", 1, alpha=50.0, beta=1.0)
        ctx.op("cholesky", 3, 1)
        out["cholesky"] = h(*ctx.download(3).to_flat())
        ctx.op("cholesky_deferred", 4, 1)
        out["cholesky_deferred"] = h(*ctx.download(4).to_flat())
        ctx.op("solve_upper_right", 5, 0, 3)
        out["solve"] = h(*ctx.download(5).to_flat())
        ctx.op("solve_upperT_right", 2, 5, 3)
        out["solveT"] = h(*ctx.download(2).to_flat())
        ctx.close()
        return out[which] if which else out
    return run


for w in ("multiply", "axpby_sym", "cholesky", "cholesky_deferred", "solve", "solveT"):
    cases["ctx " + w] = ctx_ops(w)

for name, fn in cases.items():
    res = []
    lock = threading.Lock()

    def worker():
        for _ in range(REPS):
            v = fn()
            with lock:
                res.append(v)
    th = [threading.Thread(target=worker) for _ in range(NT)]
    for t in th: t.start()
    for t in th: t.join()
    print("%-22s runs %3d distinct outputs %d" % (name, len(res), len(set(res))), flush=True)
