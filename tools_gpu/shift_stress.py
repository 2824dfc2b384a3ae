"""Stress of the concurrent multi-shift entry points (GPU box): repeated calls, failures counted."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1608_01164_b200 as S
A = S.dimer_chain(1024, 1.0, 0.5, 0.1, 6)
shifts = [0.0, 0.9, -0.9, 0.3]
ref = [S.hqdwh(A.shifted(mu), 64, 1e-10).P.to_flat()[1] for mu in shifts]
for name, call in (("devices", lambda: S.hqdwh_shifts_devices(A, shifts, 64, 1e-10)[0]),
                   ("shifts2", lambda: S.hqdwh_shifts(A, shifts, 64, 1e-10, max_concurrent=2)),
                   ("shifts4", lambda: S.hqdwh_shifts(A, shifts, 64, 1e-10, max_concurrent=4))):
    bad = 0; diff = 0
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
        if it % 3 == 0:
            S.load_library().spg_release_plan_cache()
        try:
            rs = call()
            for r, f in zip(rs, ref):
                if not np.array_equal(r.P.to_flat()[1], f):
                    diff += 1
                r.close()
        except Exception as e:
            bad += 1
            print(name, it, type(e).__name__, str(e)[:100], flush=True)
    print(name, "failures", bad, "mismatches", diff, flush=True)
