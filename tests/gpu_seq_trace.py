"""Diagnostics: phase times of the sequential setup kernels (clock64 traces)."""
import sys
sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402
for name in sys.argv[1:]:
    c = CONFIGS[name]
    r = S.hqdwh(make_input(name), c["nmin"], c["eps"])
    t = S.micro_kernel(5, 0, 0)
    f = 1965e3
    print(name, "band-l0: LU %.1f ms, Hager %.1f ms" % ((t[6] - t[5]) / f, (t[7] - t[6]) / f),
          "setup", round(r.info["ms_setup"], 1), "first", round(r.info["ms_first"], 1), flush=True)
