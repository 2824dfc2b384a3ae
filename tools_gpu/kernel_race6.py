"""Level-batched ops with the tall / flat truncation split (side stream next to the main stream) on an
intermediate iterate, many repetitions in one engine: bit-stable?  SPG_DBG_SERIAL=1 removes the split."""
import os, sys, hashlib, collections
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
REPS = int(sys.argv[1])
c = CONFIGS["smallgap"]
A = make_input(c)
for dl in (0.3, 0.1, 3e-2, 1e-2, 3e-3, 1e-3, 1e-4, 1e-6, 1e-8):
    r = S.hqdwh(A, c["nmin"], c["eps"], dl)
    if r.iterations >= 3:
        break
    r.close()
X = r.U
r.close()


def h(Hm):
    m = hashlib.sha1()
    for a in Hm.to_flat():
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:12]


ctx = S.HodlrContext(c["n"], c["nmin"], c["eps"], 6)
ctx.upload(0, X)
ctx.op("multiply_upper", 1, 0, 0)
ctx.op("scale_shift", 1, alpha=4.175, beta=1.0)
ctx.op("cholesky", 2, 1)
res = collections.defaultdict(set)
for rep in range(REPS):
    ctx.op("multiply", 3, 0, 0); res["multiply"].add(h(ctx.download(3)))
    ctx.op("multiply_upper", 3, 0, 0); res["multiply_upper"].add(h(ctx.download(3)))
    ctx.op("axpby", 3, 0, 1, 0.3, 0.7); res["axpby"].add(h(ctx.download(3)))
    ctx.op("symmetrize", 3); res["symmetrize(axpby)"].add(h(ctx.download(3)))
    ctx.op("solve_upper_right", 4, 0, 2); res["solve"].add(h(ctx.download(4)))
    ctx.op("solve_upperT_right", 5, 4, 2); res["solveT"].add(h(ctx.download(5)))
for k, v in res.items():
    print("%-20s reps %d distinct %d" % (k, REPS, len(v)), flush=True)
ctx.close()
