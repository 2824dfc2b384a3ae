"""CPU: the oracle restatement (oracle/restate.c + oracle/hodlr_np.py) pinned
against the reference's golden vectors (tests/golden/, produced by the
reference itself, tests/golden/make_golden.py) and, when oracle/_ref is
built, against the reference directly.  Also restates the reference tests'
known-answer tests (test_qdwh.cpp, test_hodlr.cpp, test_fastqr.cpp)."""
import glob
import os

import numpy as np
import pytest

from oracle import hodlr_np as H
from oracle import ref as R


def load(golden_dir, name):
    return dict(np.load(os.path.join(golden_dir, name + ".npz")))


SMALL = ["dimer_n128_b1", "dimer_n256_b1_gap", "rand_n200_b3", "dimer_n512_b8"]


# ------------------------------------------------------------------ scalar KATs
def test_qdwh_params_kats(restate):
    # test_qdwh.cpp:30-47
    a, b, c = restate.qdwh_params(1.0)
    assert abs(a - 3) < 1e-14 and abs(b - 1) < 1e-14 and abs(c - 3) < 1e-14
    a, b, c = restate.qdwh_params(0.5)
    assert abs(a - 4.35934) < 1e-4 and abs(b - 2.82125) < 1e-4 and abs(c - 6.18059) < 1e-4
    with pytest.raises(ValueError):
        restate.qdwh_params(0.0)
    with pytest.raises(ValueError):
        restate.qdwh_params(1.5)
    assert restate.L.rs_l_update(1.0, 3.0, 1.0, 3.0) == 1.0


def test_qdwh_params_vs_golden(restate, golden_dir):
    kat = load(golden_dir, "kat")
    for l in [1.0, 0.5, 0.1, 1e-3, 1e-6]:
        np.testing.assert_allclose(restate.qdwh_params(l), kat[f"params_{l:g}"], rtol=1e-14, atol=0)


def test_cubic_convergence(restate):
    # test_qdwh.cpp:66-75
    for d in (1e-2, 1e-3, 1e-4):
        l = 1 - d
        a, b, c = restate.qdwh_params(l)
        assert (1 - restate.L.rs_l_update(l, a, b, c)) / d ** 3 < 2.0


def test_schedule_matches_reference_iterations(restate, golden_dir):
    for name in SMALL + ["pr1", "smallgap"]:
        g = load(golden_dir, name)
        sched = restate.schedule(float(g["l0"]))
        assert len(sched) == int(g["iterations"])
        np.testing.assert_allclose(sched[:, 2], g["diag"][:, 2], rtol=1e-12)   # c_k
        np.testing.assert_allclose(sched[:, 3], g["diag"][:, 1], rtol=1e-12)   # l_k


# ------------------------------------------------------------------ estimates / Givens
def test_estimates_vs_golden(restate, golden_dir):
    kat = load(golden_dir, "kat")
    for n, b in [(64, 1), (50, 3), (33, 2)]:
        bands = R.unpack_bands(kat[f"reduce_n{n}_b{b}_bands"], n, b)
        alpha = restate.estimate_2norm(bands)
        l0 = restate.estimate_l0(bands, alpha)
        np.testing.assert_allclose([alpha, l0], kat[f"est_n{n}_b{b}"], rtol=1e-13)
    for name in SMALL + ["pr1", "smallgap"]:
        g = load(golden_dir, name)
        bands = R.unpack_bands(g["bands"], int(g["n"]), int(g["b"]))
        alpha = restate.estimate_2norm(bands)
        assert abs(alpha - g["alpha"]) <= 1e-13 * g["alpha"]
        assert abs(restate.estimate_l0(bands, alpha) - g["l0"]) <= 1e-12 * g["l0"]


def test_givens_reduction_vs_golden(restate, golden_dir):
    # reduce_tridiag / reduce_banded (fast_qr.hpp:83-232); rotation counts (test_fastqr.cpp:43-68)
    kat = load(golden_dir, "kat")
    for n, b in [(64, 1), (50, 3), (33, 2)]:
        bands = R.unpack_bands(kat[f"reduce_n{n}_b{b}_bands"], n, b)
        rd, nrot = restate.reduce(bands)
        assert nrot == int(kat[f"reduce_n{n}_b{b}_nrot"]) == (2 * b + 1) * n - b * b - b
        np.testing.assert_allclose(rd.ravel(), kat[f"reduce_n{n}_b{b}_R"], rtol=0, atol=1e-13)


def test_givens_r_factor_property(restate):
    # R^T R = A^2 + I (test_fastqr.cpp:126-135) and |R| KAT for [[2,1],[1,2]] (104-114)
    rd, _ = restate.reduce([np.array([2.0, 2.0]), np.array([1.0])])
    Rm = np.array([[rd[0, 0], rd[1, 0]], [0.0, rd[0, 1]]])
    np.testing.assert_allclose(np.abs([Rm[0, 0], Rm[0, 1], Rm[1, 1]]),
                               [np.sqrt(6), 4 / np.sqrt(6), np.sqrt(10 / 3)], rtol=1e-13)
    rng = np.random.default_rng(3)
    bands = [rng.uniform(-1, 1, 40 - d) for d in range(3)]
    rd, _ = restate.reduce(bands)
    Rm = np.zeros((40, 40))
    for d in range(5):
        i = np.arange(40 - d)
        Rm[i, i + d] = rd[d, :40 - d]
    A = H.banded_to_dense(bands)
    np.testing.assert_allclose(Rm.T @ Rm, A @ A + np.eye(40), atol=1e-12)


# ------------------------------------------------------------------ HODLR restatement
def test_truncate_kats():
    # test_hodlr.cpp:96-125
    rng = np.random.default_rng(7)

    def block(p, s, sv):
        qu, _ = np.linalg.qr(rng.standard_normal((p, len(sv))))
        qv, _ = np.linalg.qr(rng.standard_normal((s, len(sv))))
        return qu * sv, qv
    U, V = block(12, 10, [1.0, 1e-3])
    u, v = H.truncate(U, V, 1e-10)
    assert u.shape[1] == 2 and np.abs(u @ v.T - U @ V.T).max() < 1e-13
    U, V = block(12, 10, [1.0, 1e-12])
    u, v = H.truncate(U, V, 1e-10)
    assert u.shape[1] == 1 and np.linalg.norm(u @ v.T - U @ V.T, 2) < 2e-12
    U, V = block(20, 18, [2.0 ** -i for i in range(8)])
    mix = rng.standard_normal((8, 16))
    U16 = U @ mix
    V16 = V @ np.linalg.solve(mix @ mix.T, mix)
    u, v = H.truncate(U16, V16, 1e-10)
    assert u.shape[1] == 8 and np.abs(u @ v.T - U @ V.T).max() < 1e-10


def test_from_banded_exact():
    # test_hodlr.cpp:70-94
    rng = np.random.default_rng(5)
    bands = [rng.uniform(-1, 1, 64 - d) for d in range(5)]
    Hh = H.from_banded(bands, H.Tree(64, 8))
    assert np.abs(H.to_dense(Hh) - H.banded_to_dense(bands)).max() == 0.0
    assert H.diagnostics(Hh)[0] <= 4
    tri = [rng.uniform(-1, 1, 16 - d) for d in range(2)]
    Ht = H.from_banded(tri, H.Tree(16, 4))
    assert all(Ht.up[k][0].shape[1] == 1 and Ht.lo[k][0].shape[1] == 1 for k in Ht.up)


def test_tree_matches_reference(reflib):
    for n, nmin in [(2048, 128), (777, 50), (1000, 7), (5, 2), (16384, 256)]:
        nn = reflib.L.ref_tree(n, nmin, None, None, None, None, None)
        b, s, l, r = (np.zeros(nn, dtype=np.int32) for _ in range(4))
        d = np.zeros(1, dtype=np.int32)
        reflib.L.ref_tree(n, nmin, R._i(b), R._i(s), R._i(l), R._i(r), R._i(d))
        T = H.Tree(n, nmin)
        assert list(b) == T.begin and list(s) == T.size and list(l) == T.left and list(r) == T.right
        assert int(d[0]) == T.depth


@pytest.mark.parametrize("name", SMALL)
def test_restatement_hqdwh_vs_golden(restate, golden_dir, name):
    g = load(golden_dir, name)
    n, b, nmin, eps = int(g["n"]), int(g["b"]), int(g["n_min"]), float(g["eps"])
    bands = R.unpack_bands(g["bands"], n, b)
    alpha = restate.estimate_2norm(bands)
    l0 = restate.estimate_l0(bands, alpha)
    P, U, it, diag = H.hqdwh(bands, nmin, eps, 1e-15, alpha, l0)
    assert it == int(g["iterations"])
    assert [d[3] for d in diag] == [int(x) for x in g["diag"][:, 3]]     # per-iteration max rank
    assert abs(H.trace(P) - g["trace"]) < 1e-9
    rng = np.random.default_rng(int(g["omega_seed"]))
    Om = rng.standard_normal((n, g["P_omega"].shape[1]))
    assert np.abs(H.apply(P, Om) - g["P_omega"]).max() < 100 * eps
    if "P_dense" in g:
        assert np.linalg.norm(H.to_dense(P) - g["P_dense"], 2) < 100 * eps


def test_restatement_ops_vs_reference(reflib):
    """Each HODLR operation of the numpy restatement against the reference op."""
    n, nmin, eps = 96, 12, 1e-10
    rng = np.random.default_rng(11)
    bands = [rng.uniform(-1, 1, n - d) for d in range(3)]
    T = H.Tree(n, nmin)
    X = H.from_banded(bands, T)
    hX = reflib.import_(X)
    Z = H.multiply(X, X, eps)
    hZ = reflib.L.ref_multiply(hX, hX, eps)
    assert np.abs(H.to_dense(Z) - reflib.to_dense(hZ, n)).max() < 1e-12
    H.scale(Z, 0.7); H.add_scaled_identity(Z, 1.0)
    reflib.L.ref_scale(hZ, 0.7); reflib.L.ref_add_identity(hZ, 1.0)
    W = H.cholesky(Z, eps)
    st = np.zeros(1, dtype=np.int32)
    hW = reflib.L.ref_cholesky(hZ, eps, R._i(st))
    assert np.abs(H.to_dense(W) - reflib.to_dense(hW, n)).max() < 1e-12
    Y = H.solve_upper_right(X, W, eps)
    hY = reflib.L.ref_solve_upper_right(hX, hW, eps, R._i(st))
    assert np.abs(H.to_dense(Y) - reflib.to_dense(hY, n)).max() < 1e-12
    V = H.solve_upperT_right(Y, W, eps)
    hV = reflib.L.ref_solve_upperT_right(hY, hW, eps, R._i(st))
    assert np.abs(H.to_dense(V) - reflib.to_dense(hV, n)).max() < 1e-12
    C = H.axpby(0.3, X, -0.6, V, eps)
    hC = reflib.L.ref_axpby(0.3, hX, -0.6, hV, eps)
    assert np.abs(H.to_dense(C) - reflib.to_dense(hC, n)).max() < 1e-12
    H.symmetrize(C, eps)
    reflib.L.ref_symmetrize(hC, eps)
    assert np.abs(H.to_dense(C) - reflib.to_dense(hC, n)).max() < 1e-12
    for h in (hX, hZ, hW, hY, hV, hC):
        reflib.L.ref_hodlr_free(h)


def test_restate_c_vs_reference(reflib, restate):
    rng = np.random.default_rng(9)
    for n, b in [(300, 1), (257, 4)]:
        bands = [rng.uniform(-1, 1, n - d) for d in range(b + 1)]
        p = R.pack_bands(bands)
        a1 = reflib.L.ref_estimate_2norm(n, b, R._d(p))
        assert abs(restate.estimate_2norm(bands) - a1) <= 1e-13 * a1
        st = np.zeros(1, dtype=np.int32)
        l1 = reflib.L.ref_estimate_l0(n, b, R._d(p), a1, R._i(st))
        assert abs(restate.estimate_l0(bands, a1) - l1) <= 1e-12 * l1


def test_golden_fixtures_present(golden_dir):
    names = {os.path.basename(p)[:-4] for p in glob.glob(os.path.join(golden_dir, "*.npz"))}
    assert set(SMALL + ["pr1", "smallgap", "kat", "dimer_n777_b3"]) <= names
