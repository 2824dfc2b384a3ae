"""e2e breakdown of one headline projector through the public API (diagnostics)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sweep0.999"
c = CONFIGS[name]
A = make_input(name)
packed = A.packed()
for rep in range(3):
    t0 = time.perf_counter()
    r = S.hqdwh(A, c["nmin"], c["eps"], packed=packed)
    t1 = time.perf_counter()
    P = r.P
    t2 = time.perf_counter()
    print(f"call {t1 - t0:.3f} s (device {r.info['ms_total'] / 1e3:.3f} s), fetch P {t2 - t1:.3f} s", flush=True)
    r.close()
    del P
