"""Setup-phase breakdown of the banded configs from the clock64 stamps of the sequential
kernels (k_est_l0_band: [5] norm done, [6] LU factor done, [7] Hager done with SPG_HAGER_BAND_SEQ=1).
python tests/gpu_setup_trace.py banded large"""
import json
import sys

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from paper_1608_01164_b200.configs import CONFIGS, make_input  # noqa: E402

GHZ = 1.965
for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = make_input(name)
    for rep in range(2):
        r = S.hqdwh(A, c["nmin"], c["eps"])
        I = dict(r.info)
        l0 = r.l0
        r.close()
    t = S.micro_kernel(5, 0)
    ms = lambda a, b: round((t[b] - t[a]) / GHZ / 1e6, 2)
    print(json.dumps({"config": name, "ms_setup": round(I["ms_setup"], 1), "ms_first": round(I["ms_first"], 1),
                      "ms_total": round(I["ms_total"], 1), "l0": l0, "iters": I["iterations"],
                      "l0_factor_ms": ms(5, 6),
                      # [7] is stamped by the single-warp Hager solves only (SPG_HAGER_BAND_SEQ=1)
                      "l0_hager_seq_ms": ms(6, 7) if t[7] > t[6] else None}), flush=True)
