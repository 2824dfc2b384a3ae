"""Cold (first call of a shape) vs warm (cached plan, graph replay) projector results, bit for bit."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
c = CONFIGS[sys.argv[1]]
A = make_input(c)
res = []
for i in range(int(sys.argv[2])):
    if len(sys.argv) > 3 and i % int(sys.argv[3]) == 0:
        S.load_library().spg_release_plan_cache()
    r = S.hqdwh(A, c["nmin"], c["eps"])
    rk, d = r.P.to_flat()
    res.append((rk.copy(), d.copy(), r.info["graph_used"]))
    r.close()
groups = []
for i, (rk, d, g) in enumerate(res):
    for grp in groups:
        if np.array_equal(res[grp[0]][0], rk) and np.array_equal(res[grp[0]][1], d):
            grp.append(i)
            break
    else:
        groups.append([i])
print("distinct results:", len(groups), [(g[:8], len(g)) for g in groups], "graph_used", [r[2] for r in res][:12])
