"""Bring-up: component parity at realistic ranks (inputs = the reference's own iterates)."""
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


def sv_block(p, s, sv, seed):
    rng = np.random.default_rng(seed)
    qu, _ = np.linalg.qr(rng.standard_normal((p, len(sv))))
    qv, _ = np.linalg.qr(rng.standard_normal((s, len(sv))))
    return qu * sv, qv


def t_trunc_drop():
    rng = np.random.default_rng(1)
    for p, k in [(256, 60), (1024, 84), (2048, 84), (4096, 100), (8192, 84), (32768, 80)]:
        sv = np.logspace(0, -15, k)
        U, V = sv_block(p, p, sv, p)
        mix = rng.standard_normal((k, k))
        U2 = U @ mix
        V2 = V @ np.linalg.inv(mix).T
        u1, v1 = S.truncate(U2, V2, 1e-10) if k <= 112 else (None, None)
        u2, v2 = RL.truncate(U2, V2, 1e-10)
        B = U @ V.T
        print(f"  p={p} k={k}: gpu rank {u1.shape[1]} ref rank {u2.shape[1]} expect {int(np.sum(sv > 1e-10))}; "
              f"||B-B'|| gpu {np.linalg.norm(u1 @ v1.T - B, 2):.2e} ref {np.linalg.norm(u2 @ v2.T - B, 2):.2e}", flush=True)


def t_ops_real(n=4096, nmin=256, t2=0.999):
    A = S.dimer_chain(n, 1.0, t2, 0.2 * (1 - t2), 2)
    ref = RL.hqdwh(A.bands, nmin, 1e-10)
    Uref = RL.export(ref["U"], n, nmin)        # converged sign approximant (ranks ~ 40)
    eps = 1e-10
    tree = S.make_tree(n, nmin)
    ctx = S.HodlrContext(n, nmin, eps, 4)
    ranks, data = R.hodlr_to_flat(Uref)
    Xg = S.HodlrMatrix.from_flat(tree, ranks, data)
    ctx.upload(0, Xg)
    back = ctx.download(0)
    print("  upload/download", np.abs(back.to_dense() - H.to_dense(Uref)).max(), back.diagnostics(), H.diagnostics(Uref))
    hX = RL.import_(Uref)
    D = H.to_dense(Uref)
    # multiply
    ctx.op("multiply", 1, 0, 0)
    Z = ctx.download(1)
    hZ = RL.L.ref_multiply(hX, hX, eps)
    Zr = RL.to_dense(hZ, n)
    print("  multiply: ||Z-Zref|| %.2e  ||Z-X^2|| %.2e ranks gpu %s ref %s" % (
        np.linalg.norm(Z.to_dense() - Zr, 2), np.linalg.norm(Z.to_dense() - D @ D, 2), Z.diagnostics(),
        (RL.L.ref_hodlr_max_rank(hZ),)), flush=True)
    # cholesky of I + 3 X^2
    ctx.op("scale_shift", 1, alpha=3.0, beta=1.0)
    RL.L.ref_scale(hZ, 3.0)
    RL.L.ref_add_identity(hZ, 1.0)
    ctx.op("cholesky", 2, 1)
    W = ctx.download(2)
    st = np.zeros(1, dtype=np.int32)
    hW = RL.L.ref_cholesky(hZ, eps, R._i(st))
    Wd = W.to_dense()
    Zd = RL.to_dense(hZ, n)
    print("  cholesky: ||W^TW - Z|| %.2e  ||W-Wref|| %.2e  ranks gpu %d ref %d" % (
        np.linalg.norm(Wd.T @ Wd - Zd, 2), np.linalg.norm(Wd - RL.to_dense(hW, n), 2), W.diagnostics()[0],
        RL.L.ref_hodlr_max_rank(hW)), flush=True)
    # solves with the reference W (isolate)
    ranksW, dataW = R.hodlr_to_flat(RL.export(hW, n, nmin))
    ctx.upload(2, S.HodlrMatrix.from_flat(tree, ranksW, dataW))
    Wr = RL.to_dense(hW, n)
    ctx.op("solve_upper_right", 3, 0, 2)
    Y = ctx.download(3)
    hY = RL.L.ref_solve_upper_right(hX, hW, eps, R._i(st))
    print("  solve_ur: ||YW-X|| %.2e ||Y-Yref|| %.2e ranks gpu %d ref %d" % (
        np.linalg.norm(Y.to_dense() @ Wr - D, 2), np.linalg.norm(Y.to_dense() - RL.to_dense(hY, n), 2),
        Y.diagnostics()[0], RL.L.ref_hodlr_max_rank(hY)), flush=True)
    ranksY, dataY = R.hodlr_to_flat(RL.export(hY, n, nmin))
    ctx.upload(3, S.HodlrMatrix.from_flat(tree, ranksY, dataY))
    ctx.op("solve_upperT_right", 1, 3, 2)
    V = ctx.download(1)
    hV = RL.L.ref_solve_upperT_right(hY, hW, eps, R._i(st))
    Yd = RL.to_dense(hY, n)
    print("  solve_urt: ||VW^T-Y|| %.2e ||V-Vref|| %.2e ranks gpu %d ref %d" % (
        np.linalg.norm(V.to_dense() @ Wr.T - Yd, 2), np.linalg.norm(V.to_dense() - RL.to_dense(hV, n), 2),
        V.diagnostics()[0], RL.L.ref_hodlr_max_rank(hV)), flush=True)
    ctx.op("axpby", 3, 0, 1, 0.6, 0.4)
    C = ctx.download(3)
    hC = RL.L.ref_axpby(0.6, hX, 0.4, hV, eps)
    print("  axpby: ||C-Cref|| %.2e ranks gpu %d ref %d" % (
        np.linalg.norm(C.to_dense() - RL.to_dense(hC, n), 2), C.diagnostics()[0], RL.L.ref_hodlr_max_rank(hC)), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["drop", "real"]
    if "drop" in which:
        stage("truncate with dropping", t_trunc_drop)
    if "real" in which:
        stage("ops at realistic ranks", t_ops_real)


def t_first(n=4096, nmin=256, t2=0.999):
    A = S.dimer_chain(n, 1.0, t2, 0.2 * (1 - t2), 2)
    eps = 1e-10
    RS = R.RestateLib()
    alpha = RS.estimate_2norm(A.bands)
    l0 = RS.estimate_l0(A.bands, alpha)
    a, b, c = RS.qdwh_params(min(l0, 1 - 1e-12))
    sc = np.sqrt(c)
    print(f"  alpha {alpha} l0 {l0:.3e} c0 {c:.3e}")
    Bs = [x * (sc / alpha) for x in A.bands]
    rd, nrot = RS.reduce(Bs)
    Rd = np.zeros((n, n))
    for d in range(rd.shape[0]):
        i = np.arange(n - d)
        Rd[i, i + d] = rd[d, :n - d]
    T = H.Tree(n, nmin)
    WR = H._compress_dense(Rd, T, 1e-15)
    print("  R: cond", np.linalg.cond(Rd), "ranks", H.diagnostics(WR)[0], "||R^TR - (I+cX^2)||",
          np.abs(Rd.T @ Rd - (np.eye(n) + (sc / alpha) ** 2 * A.to_dense() @ A.to_dense())).max())
    tree = S.make_tree(n, nmin)
    ctx = S.HodlrContext(n, nmin, eps, 4)
    ctx.upload(2, S.HodlrMatrix.from_flat(tree, *R.hodlr_to_flat(WR)))
    ctx.from_banded(0, S.BandedSymmetric(n, 1, Bs))
    ctx.op("solve_upper_right", 3, 0, 2)
    Y = ctx.download(3)
    Bd = S.BandedSymmetric(n, 1, Bs).to_dense()
    Q1 = np.linalg.solve(Rd.T, Bd.T).T
    print("  Y=Q1: ||Y - B R^-1|| %.2e  ||YR - B|| %.2e ranks %s" % (np.linalg.norm(Y.to_dense() - Q1, 2),
          np.linalg.norm(Y.to_dense() @ Rd - Bd, 2), Y.diagnostics()), flush=True)
    ctx.op("solve_upperT_right", 1, 3, 2)
    M = ctx.download(1)
    Mex = np.linalg.solve(Rd, Q1.T).T
    hM = RL.L.ref_first_iterate_m(n, 1, R._d(R.pack_bands(Bs)), nmin, eps)
    Mr = RL.to_dense(hM, n)
    print("  M: ||M - Q1 R^-T|| %.2e ||M - Mref|| %.2e ranks gpu %s ref %d" % (
        np.linalg.norm(M.to_dense() - Mex, 2), np.linalg.norm(M.to_dense() - Mr, 2), M.diagnostics(),
        RL.L.ref_hodlr_max_rank(hM)), flush=True)


if __name__ == "__main__" and "first" in sys.argv:
    stage("first iterate", t_first)


def t_first_small(n=512, nmin=64, t2=0.999):
    A = S.dimer_chain(n, 1.0, t2, 0.2 * (1 - t2), 2)
    eps = 1e-10
    RS = R.RestateLib()
    alpha = RS.estimate_2norm(A.bands)
    l0 = RS.estimate_l0(A.bands, alpha)
    a, b, c = RS.qdwh_params(min(l0, 1 - 1e-12))
    for scl in [1.0, np.sqrt(c) / alpha]:
        Bs = [x * scl for x in A.bands]
        rd, nrot = RS.reduce(Bs)
        Rd = np.zeros((n, n))
        for d in range(rd.shape[0]):
            i = np.arange(n - d)
            Rd[i, i + d] = rd[d, :n - d]
        T = H.Tree(n, nmin)
        WR = H._compress_dense(Rd, T, 1e-15)
        Bn = H.from_banded(Bs, T)
        Yn = H.solve_upper_right(Bn, WR, eps)
        tree = S.make_tree(n, nmin)
        ctx = S.HodlrContext(n, nmin, eps, 4)
        ctx.upload(2, S.HodlrMatrix.from_flat(tree, *R.hodlr_to_flat(WR)))
        ctx.upload(0, S.HodlrMatrix.from_flat(tree, *R.hodlr_to_flat(Bn)))
        ctx.op("solve_upper_right", 3, 0, 2)
        Y = ctx.download(3)
        print(f"  scale {scl:.3e}: ||Y - Ynp|| {np.linalg.norm(Y.to_dense() - H.to_dense(Yn), 2):.2e}  "
              f"||Ynp R - B|| {np.linalg.norm(H.to_dense(Yn) @ Rd - H.to_dense(Bn), 2):.2e}", flush=True)
        for i in range(len(T)):
            if T.leaf(i):
                e = np.abs(Y.dense[i] - Yn.dense[i]).max()
                if e > 1e-8:
                    print(f"    leaf {i} begin {T.begin[i]} err {e:.2e}")
            else:
                for nm, g, h in (("up", Y.upper[i], Yn.up[i]), ("lo", Y.lower[i], Yn.lo[i])):
                    e = np.abs(g[0] @ g[1].T - h[0] @ h[1].T).max() if (g[0].shape[1] or h[0].shape[1]) else 0.0
                    if e > 1e-8:
                        print(f"    node {i} {nm} ranks {g[0].shape[1]} {h[0].shape[1]} err {e:.2e}")


if __name__ == "__main__" and "firstsmall" in sys.argv:
    stage("first iterate small", t_first_small)
