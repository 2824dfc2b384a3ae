"""A/B of the first-iterate band Cholesky kernels (k_band_chol_w2 / k_band_chol_reg vs the
windowed k_band_chol, SPG_BAND_CHOL_WINDOW=1): same projector bits expected.
python tests/gpu_bandchol_ab.py out.npz   (run once per variant, then: python tests/gpu_bandchol_ab.py cmp a.npz b.npz)"""
import sys

import numpy as np

sys.path.insert(0, ".")

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise equal" if not bad else f"DIFFER: {bad}")
    sys.exit(0 if not bad else 1)

import paper_1608_01164_b200 as S  # noqa: E402

out = {}
for b in (1, 2, 3, 5, 8, 12, 16):
    n = 3000 + 37 * b
    A = S.dimer_chain(n, 1.0, 0.8, 0.05, 100 + b, b=b, s=0.02 / (2 * b + 1)) if b > 1 else S.dimer_chain(n, 1.0, 0.8, 0.05, 101)
    r = S.hqdwh(A, 128, 1e-10)
    f = r.P.to_flat()
    out[f"b{b}_leaf"], out[f"b{b}_lr"] = f[0], f[1]
    out[f"b{b}_it"] = np.array([r.iterations, r.info["ms_first"]])
    print(f"b={b} n={n} iters={r.iterations} ms_first={r.info['ms_first']:.2f} trace={r.P.trace():.6f}", flush=True)
np.savez(sys.argv[1], **{k: v for k, v in out.items() if not k.endswith("_it")})
