"""Two (or more) identical projectors run concurrently (separate engines), repeated: are the results
bit-identical?  With SPG_DETERMINISTIC=1 each engine is free of the open H-Cholesky item, so any
difference here would come from contention alone (an intra-kernel race)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S
from paper_1608_01164_b200.configs import CONFIGS, make_input
c = CONFIGS["smallgap"]
A = make_input(c)
ref = None
bad = 0
tot = 0
for rep in range(int(sys.argv[1])):
    rs = S.hqdwh_shifts(A, [0.0] * int(sys.argv[2]), c["nmin"], c["eps"], max_concurrent=int(sys.argv[2]))
    for r in rs:
        rk, d = r.P.to_flat()
        if ref is None:
            ref = (rk.copy(), d.copy())
        elif not (np.array_equal(rk, ref[0]) and np.array_equal(d, ref[1])):
            bad += 1
        tot += 1
        r.close()
print("projectors", tot, "differing from the first", bad)
