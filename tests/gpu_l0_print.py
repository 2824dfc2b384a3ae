"""Print l0 / alpha (repr) of the tridiagonal configs (A/B of the setup kernels): python tests/gpu_l0_print.py"""
import sys

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

for name in ("pr1", "smallgap", "sweep0.999", "sweep0.5"):
    c = CONFIGS[name]
    r = S.hqdwh(make_input(name), c["nmin"], c["eps"])
    print(name, repr(r.l0), repr(r.alpha), r.iterations, round(r.info["ms_setup"], 2), flush=True)
