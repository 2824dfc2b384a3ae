"""GPU parity tests: the CUDA path (through the C-ABI library) against the
oracle (reference golden vectors, the numpy/C restatement, and oracle/_ref
when it was built).  Tolerances follow north_star: ||P - P_ref||_2 <= 100*eps,
round(trace P) = nu, ||P^2 - P||_2 <= 100*eps."""
import os
import subprocess

import numpy as np
import pytest

import paper_1608_01164_b200 as S
from oracle import hodlr_np as H
from oracle import ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def load(golden_dir, name):
    return dict(np.load(os.path.join(golden_dir, name + ".npz")))


def power_norm(apply, n, iters=60, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 1))
    x /= np.linalg.norm(x)
    lam = 0.0
    for _ in range(iters):
        y = apply(x)
        lam = np.linalg.norm(y)
        if lam == 0.0:
            return 0.0
        x = y / lam
    return lam


def lr_norm(U1, V1, U2, V2):
    """||U1 V1^T - U2 V2^T||_2 from the factors (no dense p x s matrix)."""
    Qa, Ra = np.linalg.qr(np.hstack([U1, -U2]))
    Qb, Rb = np.linalg.qr(np.hstack([V1, V2]))
    return np.linalg.norm(Ra @ Rb.T, 2)


def sv_block(rng, p, s, sv):
    qu, _ = np.linalg.qr(rng.standard_normal((p, len(sv))))
    qv, _ = np.linalg.qr(rng.standard_normal((s, len(sv))))
    return qu * np.asarray(sv), qv


# ------------------------------------------------------------------ truncate (lowrank.hpp:67-86)
def test_truncate_kats():
    rng = np.random.default_rng(7)
    U, V = sv_block(rng, 12, 10, [1.0, 1e-3])
    u, v = S.truncate(U, V, 1e-10)
    assert u.shape[1] == 2 and np.abs(u @ v.T - U @ V.T).max() < 1e-13
    U, V = sv_block(rng, 12, 10, [1.0, 1e-12])
    u, v = S.truncate(U, V, 1e-10)
    assert u.shape[1] == 1 and np.linalg.norm(u @ v.T - U @ V.T, 2) < 2e-12
    U, V = sv_block(rng, 20, 18, [2.0 ** -i for i in range(8)])
    mix = rng.standard_normal((8, 16))
    u, v = S.truncate(U @ mix, V @ np.linalg.solve(mix @ mix.T, mix), 1e-10)
    assert u.shape[1] == 8 and np.abs(u @ v.T - U @ V.T).max() < 1e-10


@pytest.mark.parametrize("p,s,k", [(256, 256, 60), (1000, 900, 84), (3000, 2500, 84), (9000, 9000, 100),
                                   (33000, 32768, 48), (5, 7, 12), (1, 40, 3)])
def test_truncate_contract(p, s, k):
    # discarded part <= eps (test_hodlr.cpp:330-345) and kept rank = #{sigma > eps}
    rng = np.random.default_rng(p + k)
    r = min(p, s, k)
    sv = np.logspace(0, -20, r)          # ~r/2 values above eps: stays within KCAP
    U, V = sv_block(rng, p, s, sv)
    if k > r:
        U = np.hstack([U, np.zeros((p, k - r))])
        V = np.hstack([V, rng.standard_normal((s, k - r))])
    mix = rng.standard_normal((k, k)) + 3 * np.eye(k)
    U2, V2 = U @ mix, V @ np.linalg.inv(mix).T
    u, v = S.truncate(U2, V2, 1e-10)
    assert u.shape[1] == int(np.sum(sv > 1e-10))
    assert lr_norm(u, v, U, V) <= 1e-10 * (1 + 1e-6) + 1e-12


def test_truncate_vs_reference(reflib):
    rng = np.random.default_rng(3)
    for p, s, k in [(300, 280, 40), (2048, 2048, 84)]:
        U = rng.standard_normal((p, k)) * np.logspace(0, -20, k)
        V = rng.standard_normal((s, k))
        u1, v1 = S.truncate(U, V, 1e-10)
        u2, v2 = reflib.truncate(U, V, 1e-10)
        assert u1.shape[1] == u2.shape[1]
        assert lr_norm(u1, v1, u2, v2) < 1e-12 * lr_norm(U, V, 0 * U, V) + 2e-10


# ------------------------------------------------------------------ HODLR operations (hodlr.hpp)
def _random_hodlr(n, nmin, seed, bw=2):
    rng = np.random.default_rng(seed)
    bands = [rng.uniform(-1, 1, n - d) for d in range(bw + 1)]
    return bands, H.from_banded(bands, H.Tree(n, nmin))


def _up(ctx, slot, Hn):
    ranks, data = R.hodlr_to_flat(Hn)
    ctx.upload(slot, S.HodlrMatrix.from_flat(ctx.tree, ranks, data))


@pytest.mark.parametrize("n,nmin", [(96, 12), (300, 40), (777, 64)])
def test_ops_vs_restatement(n, nmin):
    eps = 1e-10
    bands, Xn = _random_hodlr(n, nmin, n)
    ctx = S.HodlrContext(n, nmin, eps, 4)
    ctx.from_banded(0, S.BandedSymmetric(n, 2, bands))
    assert np.abs(ctx.download(0).to_dense() - H.to_dense(Xn)).max() == 0.0   # from_banded is exact
    ctx.op("multiply", 1, 0, 0)
    Zn = H.multiply(Xn, Xn, eps)
    Z = ctx.download(1)
    assert np.abs(Z.to_dense() - H.to_dense(Zn)).max() < 1e-12
    assert Z.diagnostics() == H.diagnostics(Zn)
    ctx.op("scale_shift", 1, alpha=0.5, beta=1.0)
    H.scale(Zn, 0.5); H.add_scaled_identity(Zn, 1.0)
    ctx.op("cholesky", 2, 1)
    Wn = H.cholesky(Zn, eps)
    W = ctx.download(2)
    assert np.abs(W.to_dense() - H.to_dense(Wn)).max() < 1e-12
    assert np.all(np.tril(W.to_dense(), -1) == 0.0)
    ctx.op("solve_upper_right", 3, 0, 2)
    Yn = H.solve_upper_right(Xn, Wn, eps)
    assert np.abs(ctx.download(3).to_dense() - H.to_dense(Yn)).max() < 1e-12
    ctx.op("solve_upperT_right", 1, 3, 2)
    Vn = H.solve_upperT_right(Yn, Wn, eps)
    assert np.abs(ctx.download(1).to_dense() - H.to_dense(Vn)).max() < 1e-12
    ctx.op("axpby", 3, 0, 1, 0.25, -1.5)
    Cn = H.axpby(0.25, Xn, -1.5, Vn, eps)
    assert np.abs(ctx.download(3).to_dense() - H.to_dense(Cn)).max() < 1e-12
    ctx.op("symmetrize", 3)
    H.symmetrize(Cn, eps)
    Cm = ctx.download(3)
    assert_exact_mirror(Cm)
    assert np.abs(Cm.to_dense() - H.to_dense(Cn)).max() < 1e-12
    ctx.close()


def assert_exact_mirror(Hm):
    # hodlr_symmetrize keeps lower = upper^T as exact factor mirrors (hodlr.hpp:357-361)
    for i, (U, V) in Hm.upper.items():
        Ul, Vl = Hm.lower[i]
        assert np.array_equal(Ul, V) and np.array_equal(Vl, U)
    for D in Hm.dense.values():
        assert np.array_equal(D, D.T)


def test_ops_identity_kats():
    # test_hodlr.cpp:127-153, 183-189, 215-232, 256-273
    n, nmin, eps = 32, 8, 1e-12
    T = H.Tree(n, nmin)
    ctx = S.HodlrContext(n, nmin, eps, 4)
    _up(ctx, 0, H.identity(T))
    ctx.op("cholesky", 1, 0)
    assert np.abs(ctx.download(1).to_dense() - np.eye(n)).max() < 1e-15
    four = H.identity(T); H.scale(four, 4.0)
    _up(ctx, 2, four)
    ctx.op("cholesky", 1, 2)
    assert np.abs(ctx.download(1).to_dense() - 2 * np.eye(n)).max() < 1e-15
    bands, Bn = _random_hodlr(n, nmin, 61)
    _up(ctx, 0, Bn)
    ctx.op("solve_upper_right", 3, 0, 1)          # W = 2I
    assert np.abs(ctx.download(3).to_dense() - 0.5 * H.to_dense(Bn)).max() < 1e-14
    ctx.op("solve_upperT_right", 3, 0, 1)
    assert np.abs(ctx.download(3).to_dense() - 0.5 * H.to_dense(Bn)).max() < 1e-14
    ctx.op("axpby", 3, 0, 0, 1.0, -1.0)            # M - M = 0 with rank 0
    D = ctx.download(3)
    assert D.diagnostics()[0] == 0 and np.abs(D.to_dense()).max() == 0.0
    _up(ctx, 2, H.identity(T))
    ctx.op("multiply", 3, 0, 2)                    # H * I = H
    assert np.abs(ctx.download(3).to_dense() - H.to_dense(Bn)).max() < 1e-14
    negI = H.identity(T); H.scale(negI, -1.0)
    _up(ctx, 2, negI)
    with pytest.raises(S.NotPositiveDefiniteError):
        ctx.op("cholesky", 1, 2)
    ctx.close()


# ------------------------------------------------------------------ hqdwh end to end
GOLDEN_SMALL = ["dimer_n128_b1", "dimer_n256_b1_gap", "rand_n200_b3", "dimer_n777_b3", "dimer_n512_b8",
                "synth_n512_gap1e1", "synth_n512_b8_gap1e4", "pr1"]


@pytest.mark.parametrize("name", GOLDEN_SMALL)
def test_hqdwh_vs_golden(golden_dir, name):
    g = load(golden_dir, name)
    n, b, nmin, eps = int(g["n"]), int(g["b"]), int(g["n_min"]), float(g["eps"])
    A = S.BandedSymmetric.from_packed(n, b, g["bands"])
    r = S.hqdwh(A, nmin, eps)
    assert r.iterations == int(g["iterations"])
    assert abs(r.alpha - g["alpha"]) <= 1e-12 * g["alpha"]
    assert abs(r.l0 - g["l0"]) <= 1e-10 * g["l0"]
    np.testing.assert_allclose([d.c for d in r.per_iteration], g["diag"][:, 2], rtol=1e-9)
    P = r.P
    tr = P.trace()
    assert round(tr) == round(float(g["trace"])) and abs(tr - g["trace"]) < 1e-8
    rng = np.random.default_rng(int(g["omega_seed"]))
    Om = rng.standard_normal((n, g["P_omega"].shape[1]))
    assert np.abs(r.apply(Om) - g["P_omega"]).max() < 100 * eps
    Pd = P.to_dense()
    if "P_dense" in g:
        assert np.linalg.norm(Pd - g["P_dense"], 2) <= 100 * eps
    assert_exact_mirror(r.U)                      # X after hodlr_symmetrize
    assert np.abs(Pd - Pd.T).max() < 1e-12        # test_qdwh.cpp:153-166
    assert np.linalg.norm(Pd @ Pd - Pd, 2) <= 100 * eps
    # per-iteration ranks are reported next to the reference's (not required identical)
    ranks = [d.max_rank for d in r.per_iteration]
    assert max(abs(x - int(y)) for x, y in zip(ranks, g["diag"][:, 3])) <= 4, (ranks, g["diag"][:, 3])


def test_hqdwh_vs_reference_dense(reflib):
    # dense ||P - P_ref||_2 against the reference run here (n <= 16384 rule of north_star)
    for n, t2, nmin in [(1024, 0.9, 64), (3000, 0.99, 128)]:
        A = S.dimer_chain(n, 1.0, t2, 0.2 * (1 - t2), 17)
        r = S.hqdwh(A, nmin, 1e-10)
        ref = reflib.hqdwh(A.bands, nmin, 1e-10)
        Pr = reflib.to_dense(ref["P"], n)
        assert r.iterations == ref["iterations"]
        assert np.linalg.norm(r.P.to_dense() - Pr, 2) <= 1e-8
        reflib.L.ref_result_free(ref["handle"])


def test_hqdwh_split_leaves_vs_reference(reflib):
    # leaves above 256 (320, 512): the leaf Cholesky runs as a 2x2 block split
    for n, t2, nmin, b in [(2560, 0.9, 320, 1), (4096, 0.95, 512, 8)]:
        A = S.dimer_chain(n, 1.0, t2, 0.2 * (1 - t2), 23, b=b, s=0.02 / (2 * b + 1)) if b > 1 else \
            S.dimer_chain(n, 1.0, t2, 0.2 * (1 - t2), 23)
        r = S.hqdwh(A, nmin, 1e-10)
        ref = reflib.hqdwh(A.bands, nmin, 1e-10)
        Pr = reflib.to_dense(ref["P"], n)
        assert r.iterations == ref["iterations"]
        D = r.P.to_dense() - Pr
        assert np.abs(np.linalg.eigvalsh(0.5 * (D + D.T))).max() <= 1e-8
        reflib.L.ref_result_free(ref["handle"])


def test_odd_leaves_banded_first_iterate():
    # odd leaf sizes (leaf storage alignment) and every band-Cholesky kernel width (b = 1..16)
    for b, n, nmin in [(1, 3037, 128), (2, 3074, 128), (3, 3111, 100), (5, 1185, 64), (12, 1444, 90), (16, 1592, 128)]:
        A = S.dimer_chain(n, 1.0, 0.8, 0.05, 100 + b, b=b, s=0.02 / (2 * b + 1))
        r = S.hqdwh(A, nmin, 1e-10)
        H = np.zeros((n, n))
        for d in range(b + 1):
            H += np.diag(A.bands[d], d) + (np.diag(A.bands[d], -d) if d else 0)
        nneg = int((np.linalg.eigvalsh(H) < 0).sum())
        assert round(r.P.trace()) == nneg and abs(r.P.trace() - nneg) < 1e-8, (b, n, r.P.trace(), nneg)


def test_smallgap_config(golden_dir):
    # BASELINE config 2: n=16384, t2=0.999, leaf 256, eps 1e-10 (randomized norms above dense scale)
    g = load(golden_dir, "smallgap")
    n, eps = int(g["n"]), float(g["eps"])
    A = S.BandedSymmetric.from_packed(n, 1, g["bands"])
    r = S.hqdwh(A, int(g["n_min"]), eps)
    assert r.iterations == int(g["iterations"])
    assert round(r.info["trace"]) == n // 2 and abs(r.info["trace"] - n / 2) < 1e-8
    rng = np.random.default_rng(int(g["omega_seed"]))
    Om = rng.standard_normal((n, g["P_omega"].shape[1]))
    assert np.abs(r.apply(Om) - g["P_omega"]).max() < 100 * eps
    idem = power_norm(lambda x: r.apply(r.apply(x)) - r.apply(x), n, iters=30)
    assert idem <= 100 * eps


def test_edge_cases():
    # -I -> P = I (test_qdwh.cpp:112-120)
    A = S.BandedSymmetric(32, 1, [-np.ones(32), np.zeros(31)])
    r = S.hqdwh(A, 8, 1e-10)
    assert np.abs(r.P.to_dense() - np.eye(32)).max() < 1e-10
    U = r.U.to_dense()
    assert np.abs(U @ U - np.eye(32)).max() < 1e-10
    # positive definite -> P = 0
    r = S.hqdwh(S.BandedSymmetric(40, 1, [2 + np.arange(40) / 40.0, 0.1 * np.ones(39)]), 8, 1e-10)
    assert np.abs(r.P.to_dense()).max() < 1e-10
    # single leaf (n <= n_min): dense path only
    B = S.dimer_chain(40, 1.0, 0.5, 0.1, 2)
    r = S.hqdwh(B, 64, 1e-10)
    ev, evec = np.linalg.eigh(B.to_dense())
    Pex = evec[:, ev < 0] @ evec[:, ev < 0].T
    assert np.linalg.norm(r.P.to_dense() - Pex, 2) < 1e-9
    # spectral slicing through a shift mu (tools/specproj.cpp:160-161)
    C = S.dimer_chain(300, 1.0, 0.6, 0.1, 5)
    mu = 0.15                                        # inside the spectral gap (-0.3, 0.3)
    r = S.hqdwh(C.shifted(mu), 32, 1e-10)
    ev, evec = np.linalg.eigh(C.to_dense())
    Pex = evec[:, ev < mu] @ evec[:, ev < mu].T
    assert round(r.P.trace()) == int(np.sum(ev < mu))
    assert np.linalg.norm(r.P.to_dense() - Pex, 2) < 1e-8


def test_error_propagation():
    # zero matrix -> SingularMatrixError (qdwh.hpp:201)
    with pytest.raises(S.SingularMatrixError):
        S.hqdwh(S.BandedSymmetric(64, 1), 16, 1e-10)
    # coarse eps against a tiny gap -> NotPositiveDefiniteError (test_qdwh.cpp:184-190);
    # the fixture is the reference test's own input, on which the reference itself throws
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "npd_case.npz"))
    A = S.BandedSymmetric.from_packed(int(g["n"]), int(g["b"]), g["bands"])
    with pytest.raises(S.NotPositiveDefiniteError):
        S.hqdwh(A, int(g["n_min"]), float(g["eps"]))


def test_deterministic():
    A = S.dimer_chain(2048, 1.0, 0.7, 0.05, 9)
    a = S.hqdwh(A, 128, 1e-10).P.to_flat()
    b = S.hqdwh(A, 128, 1e-10).P.to_flat()
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_cpp_dropin_runs(root):
    out = "/tmp/spg_test_dropin_gpu"
    libdir = os.path.dirname(S.lib_path())
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", "test_dropin.cpp"), "-L", libdir, "-lspecproj_b200",
                        f"-Wl,-rpath,{libdir}", "-o", out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    g = np.load(os.path.join(root, "tests", "golden", "npd_case.npz"))
    np.savetxt("/tmp/spg_npd_bands.txt", g["bands"], fmt="%.17g")
    r = subprocess.run([out, "/tmp/spg_npd_bands.txt"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


# chunk-parallel Hager solves of the banded l0 estimate (k_seq.cu k_hg_*): several chunks,
# ragged last chunk, every window width, interchanges; vs the restated estimate_l0
# (estimates.hpp:40-80) on the same alpha
@pytest.mark.gpu
@pytest.mark.parametrize("n,b,seed", [(3000, 2, 5), (2778, 12, 6), (5000, 16, 7), (1290, 5, 8), (700, 9, 9)])
def test_banded_l0_chunked_vs_restatement(restate, n, b, seed):
    A = S.dimer_chain(n, 1.0, 0.8, 0.0, seed, b=b, s=0.05 / (2 * b + 1))
    r = S.hqdwh(A, 128, 1e-10)
    l0 = restate.estimate_l0(A.bands, r.alpha)
    assert abs(r.l0 - l0) <= 1e-12 * l0
    assert round(r.P.trace()) == n // 2
    r.close()
