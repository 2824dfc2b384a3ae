"""Runs the NPD fixture (debug helper)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402

g = np.load(os.path.join("tests", "golden", "npd_case.npz"))
A = S.BandedSymmetric.from_packed(int(g["n"]), int(g["b"]), g["bands"])
t0 = time.time()
try:
    S.hqdwh(A, int(g["n_min"]), float(g["eps"]))
    print("no error", time.time() - t0)
except Exception as e:  # noqa: BLE001
    print(type(e).__name__, str(e)[:200], time.time() - t0)
