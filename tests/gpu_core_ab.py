"""Diagnostics: device truncate of random low-rank pairs vs a numpy SVD reference (error of U V^T)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402

rng = np.random.default_rng(5)
worst = 0.0
for k in [3, 5, 8, 12, 16, 20, 24, 28, 32, 40]:
    for dec in [4, 10, 16]:
        p = 256
        U = rng.standard_normal((p, k)) * np.logspace(0, -dec, k)
        V = rng.standard_normal((p, k))
        eps = 1e-10
        Uo, Vo = S.truncate(U, V, eps)
        B = U @ V.T
        err = np.linalg.norm(B - Uo @ Vo.T, 2)
        sv = np.linalg.svd(B, compute_uv=False)
        r_ref = int((sv > eps).sum())
        bound = np.sqrt(max(sv[r_ref:].size, 1)) * (sv[r_ref] if r_ref < sv.size else 0) + 1e-13 * sv[0]
        worst = max(worst, err / max(bound, 1e-300))
        flag = "" if err <= max(2 * eps, 1e-12 * sv[0]) else "  <-- BAD"
        print(f"k={k:2d} dec={dec:2d}: rank {Uo.shape[1]:2d} (ref {r_ref:2d})  ||B-B'||={err:.2e}{flag}", flush=True)
# exactly rank-deficient concatenations and short blocks (p < k)
for (p, k) in [(256, 12), (64, 24), (16, 24), (20, 30), (97, 30)]:
    U1 = rng.standard_normal((p, k // 2)); V1 = rng.standard_normal((p, k // 2)) * np.logspace(0, -8, k // 2)
    U = np.hstack([U1, 0.5 * U1]); V = np.hstack([V1, V1])
    Uo, Vo = S.truncate(U, V, 1e-10)
    B = U @ V.T
    err = np.linalg.norm(B - Uo @ Vo.T, 2)
    sv = np.linalg.svd(B, compute_uv=False)
    print(f"dup p={p} k={k}: rank {Uo.shape[1]} (ref {(sv > 1e-10).sum()}) err {err:.2e}", "<-- BAD" if err > 2e-10 else "", flush=True)
    U = rng.standard_normal((p, k)); V = rng.standard_normal((p, k)) * np.logspace(0, -12, k)
    Uo, Vo = S.truncate(U, V, 1e-10)
    B = U @ V.T
    err = np.linalg.norm(B - Uo @ Vo.T, 2)
    sv = np.linalg.svd(B, compute_uv=False)
    print(f"rnd p={p} k={k}: rank {Uo.shape[1]} (ref {(sv > 1e-10).sum()}) err {err:.2e}", "<-- BAD" if err > 2e-10 else "", flush=True)
