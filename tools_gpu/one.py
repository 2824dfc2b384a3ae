"""One projector of a config after a warm-up call (for ncu captures): python tools_gpu/one.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, HEADLINE, make_input  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else HEADLINE]
A = make_input(c)
for _ in range(int(os.environ.get("SPG_ONE_REPS", "2"))):
    r = S.hqdwh(A, c["nmin"], c["eps"])
    print(r.info["ms_total"], r.iterations, flush=True)
    r.close()
