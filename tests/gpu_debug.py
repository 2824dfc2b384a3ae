"""Ad-hoc GPU bring-up script (not collected by pytest): component parity vs the reference."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
import paper_1608_01164_b200 as S  # noqa: E402
from oracle import ref as R  # noqa: E402
from oracle import hodlr_np as H  # noqa: E402

RL = R.RefLib()


def stage(name, fn):
    t0 = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time() - t0:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def to_np(Hm):
    T = H.Tree(Hm.tree.n, Hm.tree.n_min)
    ranks, data = Hm.to_flat()
    return R.flat_to_hodlr(T, ranks, data)


def from_np(Hn, tree):
    ranks, data = R.hodlr_to_flat(Hn)
    return S.HodlrMatrix.from_flat(tree, ranks, data)


def t_truncate():
    rng = np.random.default_rng(0)
    for p, s, k in [(12, 10, 2), (300, 280, 20), (2000, 2100, 40), (5000, 4000, 100)]:
        U = rng.standard_normal((p, k)); V = rng.standard_normal((s, k))
        U[:, k // 2:] = U[:, :k - k // 2] * 0.5 + 1e-11 * U[:, k // 2:]
        u1, v1 = S.truncate(U, V, 1e-10)
        u2, v2 = RL.truncate(U, V, 1e-10)
        B = U @ V.T
        print("  trunc", p, s, k, "rank", u1.shape[1], u2.shape[1], "err_gpu", np.abs(u1 @ v1.T - B).max(),
              "err_ref", np.abs(u2 @ v2.T - B).max())


def t_ops():
    n, nmin, eps = 512, 64, 1e-10
    A = S.random_banded(n, 2, 5)
    ctx = S.HodlrContext(n, nmin, eps, 4)
    ctx.from_banded(0, A)
    X = ctx.download(0)
    Xr = H.from_banded(A.bands, H.Tree(n, nmin))
    print("  from_banded", np.abs(X.to_dense() - A.to_dense()).max(), X.diagnostics(), H.diagnostics(Xr))
    # multiply
    ctx.op("multiply", 1, 0, 0)
    Z = ctx.download(1)
    Zr = H.multiply(Xr, Xr, eps)
    D = A.to_dense()
    print("  multiply err vs dense", np.abs(Z.to_dense() - D @ D).max(), "vs ref", np.abs(Z.to_dense() - H.to_dense(Zr)).max(),
          Z.diagnostics(), H.diagnostics(Zr))
    # scale shift + cholesky
    ctx.op("scale_shift", 1, alpha=0.3, beta=1.0)
    Z2 = ctx.download(1)
    print("  scale_shift", np.abs(Z2.to_dense() - (0.3 * Z.to_dense() + np.eye(n))).max())
    ctx.op("cholesky", 2, 1)
    W = ctx.download(2)
    Wd = W.to_dense()
    print("  cholesky residual", np.linalg.norm(Wd.T @ Wd - Z2.to_dense(), 2), "lower max", np.abs(np.tril(Wd, -1)).max())
    ctx.op("solve_upper_right", 3, 0, 2)
    Y = ctx.download(3)
    print("  solve_ur residual", np.linalg.norm(Y.to_dense() @ Wd - D, 2))
    ctx.op("solve_upperT_right", 1, 3, 2)
    V = ctx.download(1)
    print("  solve_urt residual", np.linalg.norm(V.to_dense() @ Wd.T - Y.to_dense(), 2))
    ctx.op("axpby", 3, 0, 1, 0.7, -0.2)
    C3 = ctx.download(3)
    print("  axpby", np.abs(C3.to_dense() - (0.7 * D - 0.2 * V.to_dense())).max())
    ctx.op("symmetrize", 3)
    C4 = ctx.download(3).to_dense()
    print("  symmetrize asym", np.abs(C4 - C4.T).max(), "err", np.abs(C4 - 0.5 * (C3.to_dense() + C3.to_dense().T)).max())


def t_hqdwh(n, nmin, t2, eps_dis, seed):
    A = S.dimer_chain(n, 1.0, t2, eps_dis, seed)
    t0 = time.time()
    r = S.hqdwh(A, nmin, 1e-10)
    t1 = time.time()
    print(f"  n={n} gpu iters {r.iterations} alpha {r.alpha:.6f} l0 {r.l0:.4e} wall {t1 - t0:.3f}s info ms_total {r.info['ms_total']:.1f}")
    print("  info", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.info.items()})
    for d in r.per_iteration:
        print("   ", d)
    ref = RL.hqdwh(A.bands, nmin, 1e-10)
    print(f"  ref iters {ref['iterations']} alpha {ref['alpha']:.6f} l0 {ref['l0']:.4e} wall {ref['wall_ms']:.0f}ms")
    P = r.P
    if n <= 4096:
        Pd = P.to_dense()
        Pr = RL.to_dense(ref["P"], n)
        print("  ||P-Pref||_2", np.linalg.norm(Pd - Pr, 2), "trace", np.trace(Pd), "||P^2-P||", np.linalg.norm(Pd @ Pd - Pd, 2))
    RL.L.ref_result_free(ref["handle"])


if __name__ == "__main__":
    which = sys.argv[1:] or ["trunc", "ops", "small", "pr1"]
    if "trunc" in which:
        stage("truncate", t_truncate)
    if "ops" in which:
        stage("ops", t_ops)
    if "small" in which:
        stage("hqdwh n=512", lambda: t_hqdwh(512, 64, 0.5, 0.1, 1))
    if "pr1" in which:
        stage("hqdwh PR1", lambda: t_hqdwh(2048, 128, 0.5, 0.1, 1))
    if "sg" in which:
        stage("hqdwh small-gap", lambda: t_hqdwh(16384, 256, 0.999, 2e-4, 2))
