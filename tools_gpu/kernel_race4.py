"""Truncation kernels on inputs with singular values clustered at the threshold and far below it
(what the H-Cholesky's cascades produce), concurrently in several threads: bit-stable?"""
import os, sys, threading, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 3
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 40
g = np.random.default_rng(11)


def case(p, s, k, sig):
    r = len(sig)
    Q1 = np.linalg.qr(g.standard_normal((p, r)))[0]; Q2 = np.linalg.qr(g.standard_normal((s, r)))[0]
    M = g.standard_normal((r, k))
    return (Q1 * sig) @ M, Q2 @ np.linalg.pinv(M).T


def h(*arrs):
    m = hashlib.sha1()
    for a in arrs:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:12]


sigs = {
    "cluster at eps": np.concatenate([np.logspace(-3, -8, 22), 1e-10 * (1 + 1e-7 * np.arange(-3, 4)), np.logspace(-12, -17, 10)]),
    "tail to 1e-20": np.concatenate([np.logspace(-3, -8, 26), np.logspace(-11, -20, 14)]),
    "exact rank 26 of 52": np.logspace(-3, -8, 26),
}
cases = {}
for nm, sg in sigs.items():
    for (p, s, k) in ((256, 256, 52), (512, 512, 52), (256, 256, 80)):
        if k < len(sg):
            continue
        U, V = case(p, s, k, sg)
        cases["%s %dx%d k%d" % (nm, p, s, k)] = (lambda U=U, V=V: h(*S.truncate(U, V, 1e-10)))
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
    print("%-36s runs %3d distinct outputs %d" % (name, len(res), len(set(res))), flush=True)
