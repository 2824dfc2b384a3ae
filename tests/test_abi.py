"""CPU: the C-ABI library loads, exports every symbol include/specproj_b200.h
declares, and its host-side helpers (tree, QDWH schedule, input generator,
argument validation) behave like the reference.  No GPU compute here."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1608_01164_b200 as S
from oracle import hodlr_np as H


def header_symbols(root):
    txt = open(os.path.join(root, "include", "specproj_b200.h")).read()
    return sorted(set(re.findall(r"\b(spg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol(root, lib):
    syms = header_symbols(root)
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", S.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (spg_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(S.ABI_SYMBOLS) == set(syms)


def test_wide_capacity_library_exports_the_same_abi(lib):
    """libspecproj_b200_w.so (KCAP = 96, loaded by the main library when ranks pass 56) is built from
    the same sources: same C symbols, its C++ symbols in namespace spgw (no clash when both are mapped)."""
    import ctypes as C
    assert os.path.exists(S.WIDE_LIB_PATH)
    W = C.CDLL(S.WIDE_LIB_PATH)
    for name in S.ABI_SYMBOLS:
        assert hasattr(W, name), name
    W.spg_kcap.restype = C.c_int
    assert W.spg_kcap() == 96 and lib.spg_kcap() == 56
    syms = subprocess.run(["nm", "-DC", S.WIDE_LIB_PATH], capture_output=True, text=True).stdout
    assert " T spgw::" in syms and " T spg::" not in syms


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", S.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", S.lib_path()], capture_output=True, text=True).stdout
    assert "DMMA" in sass          # FP64 tensor path (mma.sync m8n8k4 f64)


def test_tree_matches_restatement(lib):
    for n, nmin in [(2048, 128), (777, 50), (1000, 7), (5, 2), (65536, 256)]:
        t = S.make_tree(n, nmin)
        T = H.Tree(n, nmin)
        assert list(t.begin) == T.begin and list(t.size) == T.size
        assert list(t.left) == T.left and list(t.right) == T.right and t.depth == T.depth
    with pytest.raises(ValueError):
        S.make_tree(0, 4)
    with pytest.raises(ValueError):
        S.make_tree(10, 1)


def test_qdwh_params_host(lib, restate):
    for l in (1.0, 0.5, 1e-3, 1e-7):
        np.testing.assert_allclose(S.qdwh_params(l), restate.qdwh_params(l), rtol=1e-15)
    with pytest.raises(ArithmeticError):
        S.qdwh_params(0.0)
    assert S.l_update(1.0, 3.0, 1.0, 3.0) == 1.0


def _mt19937_64(seed):
    """std::mt19937_64 (independent Python restatement for the generator check)."""
    NN, MM = 312, 156
    A, UM, LM, M64 = 0xB5026F5AA96619E9, 0xFFFFFFFF80000000, 0x7FFFFFFF, (1 << 64) - 1
    mt = [seed & M64]
    for i in range(1, NN):
        mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & M64)
    idx = NN
    while True:
        if idx >= NN:
            for i in range(NN):
                x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM)
                xa = (x >> 1) ^ (A if x & 1 else 0)
                mt[i] = mt[(i + MM) % NN] ^ xa
            idx = 0
        y = mt[idx]; idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        yield y & M64


def _uniform(gen):
    # uniform_real_distribution<double>(-1, 1) over generate_canonical<double, 53> (libstdc++)
    return float(next(gen)) / 2.0 ** 64 * 2.0 + (-1.0)


def test_dimer_chain_generator(lib):
    g = _mt19937_64(5489)
    assert next(g) == 14514284786278117030      # std::mt19937_64 default-seed KAT
    n, seed = 40, 7
    A = S.dimer_chain(n, 1.0, 0.5, 0.1, seed)
    gen = _mt19937_64(seed)
    diag = [0.1 * _uniform(gen) for _ in range(n)]
    np.testing.assert_array_equal(A.bands[0], diag)
    np.testing.assert_array_equal(A.bands[1], [1.0 if i % 2 == 0 else 0.5 for i in range(n - 1)])
    B = S.dimer_chain(20, 1.0, 0.8, 0.0, 3, b=3, s=0.01)
    gen = _mt19937_64(3)
    _ = [0.0 * _uniform(gen) for _ in range(20)]
    pert = [[0.01 * _uniform(gen) for _ in range(20 - d)] for d in range(4)]
    np.testing.assert_array_equal(B.bands[0], pert[0])
    np.testing.assert_array_equal(B.bands[1], np.array([1.0 if i % 2 == 0 else 0.8 for i in range(19)]) + pert[1])
    np.testing.assert_array_equal(B.bands[3], pert[3])
    # nu = n/2 bond convention: both chain ends are strong bonds
    ev = np.linalg.eigvalsh(S.dimer_chain(64, 1.0, 0.5, 0.1, 1).to_dense())
    assert np.sum(ev < 0) == 32 and np.min(np.abs(ev)) > 0.3


def test_random_banded_generator(lib):
    A = S.random_banded(10, 2, 19)
    gen = _mt19937_64(19)
    np.testing.assert_array_equal(A.packed(), [_uniform(gen) for _ in range(10 + 9 + 8)])


def test_hqdwh_fails_loudly_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(S.NoDeviceError):
        S.hqdwh(S.dimer_chain(64, 1.0, 0.5, 0.1, 1), 16, 1e-10)


def test_invalid_inputs(lib):
    A = S.dimer_chain(64, 1.0, 0.5, 0.1, 1)
    A.bands[0][3] = np.nan
    with pytest.raises(ValueError):
        S.hqdwh(A, 16, 1e-10)
    with pytest.raises(ValueError):
        S.BandedSymmetric(1, 1)
    with pytest.raises(ValueError):
        S.BandedSymmetric(10, 10)


def test_flat_roundtrip_host(lib):
    # the flat exchange format (include/specproj_b200.h) round-trips through the host mirror
    from oracle import ref as R
    rng = np.random.default_rng(2)
    bands = [rng.uniform(-1, 1, 100 - d) for d in range(3)]
    Hn = H.from_banded(bands, H.Tree(100, 12))
    ranks, data = R.hodlr_to_flat(Hn)
    Hm = S.HodlrMatrix.from_flat(S.make_tree(100, 12), ranks, data)
    r2, d2 = Hm.to_flat()
    np.testing.assert_array_equal(ranks, r2)
    np.testing.assert_array_equal(data, d2)
    np.testing.assert_array_equal(Hm.to_dense(), H.to_dense(Hn))
    assert Hm.diagnostics() == H.diagnostics(Hn)


def test_cpp_dropin_compiles(root, lib):
    # the C++ shim builds against the C-ABI (standalone mirror types)
    out = "/tmp/spg_test_dropin"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                        os.path.join(root, "tests", "cpp", "test_dropin.cpp"), "-L",
                        os.path.dirname(S.lib_path()), "-lspecproj_b200", "-o", out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    if os.path.isdir("/root/reference/proj/include"):
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-DSPECPROJ_B200_USE_REFERENCE_TYPES", "-I",
                            os.path.join(root, "include"), "-I", "/root/reference/proj/include",
                            os.path.join(root, "tests", "cpp", "test_dropin.cpp")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
