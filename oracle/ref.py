"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU checkers.

* ``RefLib``     : oracle/_ref/libspecproj_ref.so, the UNMODIFIED reference headers
                   behind an extern "C" shim (oracle/ref_wrap.cpp).
* ``RestateLib`` : oracle/_build/librestate.so, the plain-C restatement
                   (oracle/restate.c) of the scalar/banded parts.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may use these.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import hodlr_np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libspecproj_ref.so")
# memory-patched variant (oracle/patch_memory.py; bitwise equal, frees assemble_q's aux columns)
REF_PATCHED_SO = os.path.join(HERE, "_ref", "libspecproj_ref_patched.so")
RESTATE_SO = os.path.join(HERE, "_build", "librestate.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def pack_bands(bands):
    """bands: list of b+1 diagonals (d-th has n-d entries) -> packed float64 array."""
    return np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.float64) for x in bands]))


def unpack_bands(packed, n, b):
    out, off = [], 0
    for d in range(b + 1):
        out.append(np.array(packed[off:off + n - d]))
        off += n - d
    return out


def ref_available(patched=False):
    return os.path.exists(REF_PATCHED_SO if patched else REF_SO)


def restate_available():
    return os.path.exists(RESTATE_SO)


class RefError(RuntimeError):
    pass


class RefLib:
    def __init__(self, path=REF_SO):
        L = C.CDLL(path)
        self.L = L
        vp = C.c_void_p
        sig = {
            "ref_last_error": ([], C.c_char_p),
            "ref_set_ftz_daz": ([C.c_int], None),
            "ref_tree": ([C.c_int, C.c_int, _ip, _ip, _ip, _ip, _ip], C.c_int),
            "ref_hodlr_free": ([vp], None),
            "ref_hodlr_flat_size": ([vp], C.c_long),
            "ref_hodlr_nnodes": ([vp], C.c_int),
            "ref_hodlr_export": ([vp, _ip, _dp], None),
            "ref_hodlr_import": ([C.c_int, C.c_int, _ip, _dp], vp),
            "ref_hodlr_to_dense": ([vp, _dp], None),
            "ref_hodlr_apply": ([vp, C.c_int, _dp, _dp], None),
            "ref_hodlr_trace": ([vp], C.c_double),
            "ref_hodlr_max_rank": ([vp], C.c_int),
            "ref_hodlr_memory": ([vp], C.c_long),
            "ref_from_banded": ([C.c_int, C.c_int, _dp, C.c_int], vp),
            "ref_identity": ([C.c_int, C.c_int], vp),
            "ref_copy": ([vp], vp),
            "ref_axpby": ([C.c_double, vp, C.c_double, vp, C.c_double], vp),
            "ref_symmetrize": ([vp, C.c_double], None),
            "ref_scale": ([vp, C.c_double], None),
            "ref_add_identity": ([vp, C.c_double], None),
            "ref_transpose": ([vp], vp),
            "ref_multiply": ([vp, vp, C.c_double], vp),
            "ref_cholesky": ([vp, C.c_double, _ip], vp),
            "ref_solve_upper_right": ([vp, vp, C.c_double, _ip], vp),
            "ref_solve_upperT_right": ([vp, vp, C.c_double, _ip], vp),
            "ref_add_lowrank": ([vp, C.c_int, _dp, _dp, C.c_double], None),
            "ref_truncate": ([C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, _dp, _dp], C.c_int),
            "ref_qdwh_params": ([C.c_double, _dp], C.c_int),
            "ref_l_update": ([C.c_double] * 4, C.c_double),
            "ref_estimate_2norm": ([C.c_int, C.c_int, _dp], C.c_double),
            "ref_estimate_l0": ([C.c_int, C.c_int, _dp, C.c_double, _ip], C.c_double),
            "ref_reduce": ([C.c_int, C.c_int, _dp, _dp], C.c_long),
            "ref_first_iterate_m": ([C.c_int, C.c_int, _dp, C.c_int, C.c_double], vp),
            "ref_hqdwh": ([C.c_int, C.c_int, _dp, C.c_int, C.c_double, C.c_double, _ip], vp),
            "ref_result_free": ([vp], None),
            "ref_result_wall_ms": ([vp], C.c_double),
            "ref_result_iterations": ([vp], C.c_int),
            "ref_result_alpha": ([vp], C.c_double),
            "ref_result_l0": ([vp], C.c_double),
            "ref_result_diag": ([vp, _dp], None),
            "ref_result_hodlr": ([vp, C.c_int], vp),
            "ref_is_patched": ([], C.c_int),
            "ref_make_dimer_chain": ([C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_ulonglong, _dp], C.c_int),
            "ref_synth_banded": ([C.c_int, C.c_int, C.c_double, C.c_ulonglong, _dp], C.c_int),
            "ref_write_sbm": ([C.c_int, C.c_int, _dp, C.c_char_p], C.c_int),
            "ref_read_sbm": ([C.c_char_p, C.POINTER(C.c_int), C.c_void_p], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res

    def err(self):
        return self.L.ref_last_error().decode()

    # ---- HODLR handles <-> python restatement objects
    def export(self, h, n, n_min):
        """flat export -> oracle.hodlr_np.Hodlr"""
        tree = hodlr_np.Tree(n, n_min)
        nn = self.L.ref_hodlr_nnodes(h)
        ranks = np.zeros(2 * nn, dtype=np.int32)
        data = np.zeros(self.L.ref_hodlr_flat_size(h))
        self.L.ref_hodlr_export(h, _i(ranks), _d(data))
        return flat_to_hodlr(tree, ranks, data)

    def import_(self, H):
        ranks, data = hodlr_to_flat(H)
        h = self.L.ref_hodlr_import(H.tree.n, H.tree.n_min, _i(ranks), _d(data))
        if not h:
            raise RefError(self.err())
        return h

    def to_dense(self, h, n):
        out = np.zeros((n, n))
        self.L.ref_hodlr_to_dense(h, _d(out))
        return out

    def apply(self, h, X):
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.zeros_like(X)
        self.L.ref_hodlr_apply(h, X.shape[1], _d(X), _d(Y))
        return Y

    def truncate(self, U, V, eps):
        U = np.ascontiguousarray(U, dtype=np.float64)
        V = np.ascontiguousarray(V, dtype=np.float64)
        p, k = U.shape
        s = V.shape[0]
        Uo = np.zeros((p, k)); Vo = np.zeros((s, k))
        r = self.L.ref_truncate(p, s, k, _d(U), _d(V), eps, _d(Uo), _d(Vo))
        return Uo[:, :r].copy(), Vo[:, :r].copy()

    def write_sbm(self, path, bands):
        """banded.hpp:117-129 (the reference's writer)."""
        n, b = len(bands[0]), len(bands) - 1
        if self.L.ref_write_sbm(n, b, _d(pack_bands(bands)), path.encode()):
            raise RefError(self.err())

    def read_sbm(self, path):
        """banded.hpp:138-154 (the reference's reader)."""
        nb = np.zeros(2, dtype=np.int32)
        if self.L.ref_read_sbm(path.encode(), nb.ctypes.data_as(C.POINTER(C.c_int)), None):
            raise RefError(self.err())
        n, b = int(nb[0]), int(nb[1])
        out = np.zeros((b + 1) * n - b * (b + 1) // 2)
        if self.L.ref_read_sbm(path.encode(), nb.ctypes.data_as(C.POINTER(C.c_int)), out.ctypes.data_as(C.c_void_p)):
            raise RefError(self.err())
        return unpack_bands(out, n, b)

    def dimer_chain(self, n, t1, t2, eps_dis, seed, b=1, s=0.0):
        """SURVEY.md §8d dimer chain generated on the oracle side (no product library)."""
        out = np.zeros((b + 1) * n - b * (b + 1) // 2)
        if self.L.ref_make_dimer_chain(n, b, t1, t2, eps_dis, s, seed, _d(out)):
            raise RefError("ref_make_dimer_chain: invalid arguments")
        return unpack_bands(out, n, b)

    def config_bands(self, c, seed_offset=0):
        """bands of a BASELINE config dict (paper_1608_01164_b200.configs.CONFIGS entry)"""
        return self.dimer_chain(c["n"], c["t1"], c["t2"], c["eps_dis"], c["seed"] + seed_offset, b=c["b"], s=c["s"])

    @property
    def patched(self):
        return bool(self.L.ref_is_patched())

    def synth_banded(self, n, b, gap, seed):
        """synth.hpp:106-137 with SpectrumSpec::uniform_two_sided(n, gap) (the reference tests' inputs)."""
        out = np.zeros((b + 1) * n - b * (b + 1) // 2)
        if self.L.ref_synth_banded(n, b, gap, seed, _d(out)):
            raise RefError(self.err())
        return unpack_bands(out, n, b)

    def hqdwh(self, bands, n_min, eps, delta=1e-15):
        """Runs the reference hqdwh; returns a dict with the result handle."""
        packed = pack_bands(bands)
        n, b = len(bands[0]), len(bands) - 1
        st = np.zeros(1, dtype=np.int32)
        h = self.L.ref_hqdwh(n, b, _d(packed), n_min, eps, delta, _i(st))
        if not h:
            raise RefError(f"status {int(st[0])}: {self.err()}")
        it = self.L.ref_result_iterations(h)
        diag = np.zeros(6 * max(it, 1))
        self.L.ref_result_diag(h, _d(diag))
        return {
            "handle": h,
            "iterations": it,
            "alpha": self.L.ref_result_alpha(h),
            "l0": self.L.ref_result_l0(h),
            "wall_ms": self.L.ref_result_wall_ms(h),
            "diag": diag[: 6 * it].reshape(it, 6),
            "P": self.L.ref_result_hodlr(h, 0),
            "U": self.L.ref_result_hodlr(h, 1),
        }


def hodlr_to_flat(H):
    t = H.tree
    nn = len(t)
    ranks = np.zeros(2 * nn, dtype=np.int32)
    parts = []
    for i in range(nn):
        if t.leaf(i):
            parts.append(np.ascontiguousarray(H.dense[i]).ravel())
            continue
        (Uu, Vu), (Ul, Vl) = H.up[i], H.lo[i]
        ranks[2 * i], ranks[2 * i + 1] = Uu.shape[1], Ul.shape[1]
        parts += [np.ascontiguousarray(x).ravel() for x in (Uu, Vu, Ul, Vl)]
    data = np.concatenate(parts) if parts else np.zeros(0)
    return ranks, np.ascontiguousarray(data, dtype=np.float64)


def flat_to_hodlr(tree, ranks, data):
    H = hodlr_np.Hodlr(tree)
    off = 0

    def take(r, c):
        nonlocal off
        m = np.array(data[off:off + r * c]).reshape(r, c)
        off += r * c
        return m

    for i in range(len(tree)):
        if tree.leaf(i):
            H.dense[i] = take(tree.size[i], tree.size[i])
            continue
        s1, s2 = tree.size[tree.left[i]], tree.size[tree.right[i]]
        ku, kl = int(ranks[2 * i]), int(ranks[2 * i + 1])
        Uu = take(s1, ku); Vu = take(s2, ku); Ul = take(s2, kl); Vl = take(s1, kl)
        H.up[i] = (Uu, Vu)
        H.lo[i] = (Ul, Vl)
    return H


class RestateLib:
    """oracle/restate.c"""

    def __init__(self, path=RESTATE_SO):
        L = C.CDLL(path)
        self.L = L
        L.rs_qdwh_params.argtypes = [C.c_double, _dp]; L.rs_qdwh_params.restype = C.c_int
        L.rs_l_update.argtypes = [C.c_double] * 4; L.rs_l_update.restype = C.c_double
        L.rs_schedule.argtypes = [C.c_double, C.c_double, C.c_int, _dp]; L.rs_schedule.restype = C.c_int
        L.rs_estimate_2norm.argtypes = [C.c_int, C.c_int, _dp]; L.rs_estimate_2norm.restype = C.c_double
        L.rs_estimate_l0.argtypes = [C.c_int, C.c_int, _dp, C.c_double, _ip]; L.rs_estimate_l0.restype = C.c_double
        L.rs_reduce.argtypes = [C.c_int, C.c_int, _dp, _dp]; L.rs_reduce.restype = C.c_long

    def qdwh_params(self, l):
        out = np.zeros(3)
        if self.L.rs_qdwh_params(l, _d(out)):
            raise ValueError("qdwh_params: l must lie in (0, 1]")
        return tuple(out)

    def schedule(self, l0, delta=1e-15):
        out = np.zeros(4 * 60)
        k = self.L.rs_schedule(l0, delta, 60, _d(out))
        return out[: 4 * k].reshape(k, 4)

    def estimate_2norm(self, bands):
        p = pack_bands(bands)
        return self.L.rs_estimate_2norm(len(bands[0]), len(bands) - 1, _d(p))

    def estimate_l0(self, bands, alpha):
        p = pack_bands(bands)
        st = np.zeros(1, dtype=np.int32)
        v = self.L.rs_estimate_l0(len(bands[0]), len(bands) - 1, _d(p), alpha, _i(st))
        if st[0]:
            raise hodlr_np.SingularMatrixError("BandedLu: zero pivot")
        return v

    def reduce(self, bands):
        """R diagonals (2b+1, n) of the stacked QR of [bands; I] and #rotations"""
        n, b = len(bands[0]), len(bands) - 1
        p = pack_bands(bands)
        rd = np.zeros((2 * b + 1) * n)
        nrot = self.L.rs_reduce(n, b, _d(p), _d(rd))
        return rd.reshape(2 * b + 1, n), nrot
