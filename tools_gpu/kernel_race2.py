"""Intra-kernel race hunt at realistic ranks: the ops of one QDWH iterate on an intermediate iterate
X_k of the small-gap config (ranks ~ 30-40), run concurrently in several threads (separate engines)."""
import os, sys, threading, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
NT = int(sys.argv[1]) if len(sys.argv) > 1 else 3
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 6
c = CONFIGS["smallgap"]
A = make_input(c)
want = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for dl in (0.3, 0.1, 3e-2, 1e-2, 3e-3, 1e-3, 1e-4, 1e-6, 1e-8):
    r = S.hqdwh(A, c["nmin"], c["eps"], dl)
    if r.iterations >= want:
        break
    r.close()
print("intermediate iterate after", r.iterations, "iterations, max rank", max(d.max_rank for d in r.per_iteration), [round(d.c, 2) for d in r.per_iteration])
X = r.U
cnext = 4.175 if want == 3 else 3.0016
r.close()


def h(Hm):
    m = hashlib.sha1()
    for a in Hm.to_flat():
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:12]


def run():
    ctx = S.HodlrContext(c["n"], c["nmin"], c["eps"], 6)
    ctx.upload(0, X)
    out = []
    ctx.op("multiply_upper", 1, 0, 0); out.append(("multiply", h(ctx.download(1))))
    ctx.op("scale_shift", 1, alpha=cnext, beta=1.0)
    if os.environ.get("RACE_ONLY_DEFERRED"):
        for q in range(4):
            ctx.op("cholesky_deferred", 3, 1); out.append(("cholesky_deferred", h(ctx.download(3))))
    else:
        ctx.op("cholesky", 2, 1); out.append(("cholesky", h(ctx.download(2))))
        ctx.op("cholesky_deferred", 3, 1); out.append(("cholesky_deferred", h(ctx.download(3))))
        ctx.op("solve_upper_right", 4, 0, 2); out.append(("solve", h(ctx.download(4))))
        ctx.op("solve_upperT_right", 5, 4, 2); out.append(("solveT", h(ctx.download(5))))
        ctx.op("axpby", 1, 0, 5, 0.3, 0.7); out.append(("axpby", h(ctx.download(1))))
        ctx.op("symmetrize", 1); out.append(("symmetrize", h(ctx.download(1))))
    ctx.close()
    return out


res = []
lock = threading.Lock()


def worker():
    for _ in range(REPS):
        v = run()
        with lock:
            res.append(v)


th = [threading.Thread(target=worker) for _ in range(NT)]
for t in th: t.start()
for t in th: t.join()
import collections
byname = collections.defaultdict(list)
for x in res:
    for name, v in x:
        byname[name].append(v)
for name, vals in byname.items():
    print("%-20s runs %3d distinct %d" % (name, len(vals), len(set(vals))), flush=True)
