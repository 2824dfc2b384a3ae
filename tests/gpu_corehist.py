"""Diagnostics: histograms of the core SVD (k_in, QRCP rank r', Jacobi sweeps, kept rank) over one projector."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name = sys.argv[1]
c = CONFIGS[name]
L = S.load_library()
out = np.zeros(512)
L.spg_micro_kernel(2, 1, 0, out.ctypes.data_as(C.POINTER(C.c_double)), 0)
S.hqdwh(make_input(name), c["nmin"], c["eps"])
L.spg_micro_kernel(3, 0, 0, out.ctypes.data_as(C.POINTER(C.c_double)), 512)
h = out.reshape(4, 128)
for nm, row in zip(["k_in", "r'", "sweeps", "rank"], h):
    nz = np.nonzero(row)[0]
    print(nm, "total", int(row.sum()), "mean %.1f" % ((row * np.arange(128)).sum() / max(row.sum(), 1)),
          " ".join(f"{i}:{int(row[i])}" for i in nz))
