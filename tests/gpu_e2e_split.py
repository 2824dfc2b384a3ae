"""Diagnostics: where the end-to-end time of one hqdwh call goes (host timers)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sweep0.999"
c = CONFIGS[name]
A = make_input(name)
packed = A.packed()
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t0 = time.perf_counter()
    r = S.hqdwh(A, c["nmin"], c["eps"], packed=packed)
    t1 = time.perf_counter()
    P = r.P
    t2 = time.perf_counter()
    r.close()
    t3 = time.perf_counter()
    print(f"rep {rep}: hqdwh {1e3*(t1-t0):.1f} ms (device {r.info['ms_total']:.1f}), r.P {1e3*(t2-t1):.1f} ms, close {1e3*(t3-t2):.1f} ms", flush=True)
