"""B200-native (sm_100a, FP64) hQDWH spectral projectors in HODLR arithmetic.

Python mirror of the reference's C++ surface for the hot path
(/root/reference/proj/include/specproj, namespace ``specproj``):

=====================================  ==========================================
reference (file:line)                  here
=====================================  ==========================================
``BandedSymmetric`` (banded.hpp:19)    :class:`BandedSymmetric`
``make_tree`` (tree.hpp:58)            :func:`make_tree` -> :class:`PartitionTree`
``HodlrMatrix`` (hodlr.hpp:20)         :class:`HodlrMatrix` (host copy of device data)
``hqdwh`` (qdwh.hpp:196)               :func:`hqdwh` -> :class:`ProjectorResult`
``qdwh_params``/``l_update`` (27-40)   :func:`qdwh_params`, :func:`l_update`
``truncate`` (lowrank.hpp:67)          :func:`truncate` (one device recompression)
``to_dense``/``hodlr_trace``/...       methods of :class:`HodlrMatrix`
exceptions (dense_factor.hpp:19-25)    :class:`NotPositiveDefiniteError`, ...
=====================================  ==========================================

Every compute call goes through the C-ABI library ``libspecproj_b200.so``
(include/specproj_b200.h) built for sm_100a; there is no CPU fallback: without
the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "BandedSymmetric", "PartitionTree", "HodlrMatrix", "ProjectorResult", "IterationDiag",
    "hqdwh", "make_tree", "qdwh_params", "l_update", "truncate", "dimer_chain", "random_banded",
    "HodlrContext", "NotPositiveDefiniteError", "SingularMatrixError", "RankCapacityError",
    "NoDeviceError", "lib_path", "load_library", "set_profile",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# SPG_LIB picks another build of the same C-ABI (tests run the wide-capacity build
# libspecproj_b200_w.so through the parity tests this way); default: the in-tree library
_LIB_PATH = os.environ.get("SPG_LIB") or os.path.join(HERE, "libspecproj_b200.so")
WIDE_LIB_PATH = os.path.join(HERE, "libspecproj_b200_w.so")


def lib_path() -> str:
    return _LIB_PATH


# ---------------------------------------------------------------- exceptions
class NotPositiveDefiniteError(RuntimeError):
    """dense_factor.hpp:19-21 (CLI exit code 4)."""


class SingularMatrixError(RuntimeError):
    """dense_factor.hpp:23-25."""


class RankCapacityError(RuntimeError):
    """A truncation kept more columns than the compiled capacity (KCAP)."""


class NoDeviceError(RuntimeError):
    """No CUDA device: the B200 path has no CPU fallback."""


class CudaError(RuntimeError):
    pass


_OK, _NPD, _SING, _INV, _DOM, _RANK, _CUDA, _NODEV = range(8)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class _Info(C.Structure):
    _fields_ = [("n", C.c_int), ("b", C.c_int), ("n_min", C.c_int), ("eps", C.c_double), ("delta", C.c_double),
                ("iterations", C.c_int), ("alpha", C.c_double), ("l0", C.c_double), ("ms_total", C.c_double),
                ("ms_setup", C.c_double), ("ms_first", C.c_double), ("ms_multiply", C.c_double),
                ("ms_cholesky", C.c_double), ("ms_solve", C.c_double), ("ms_solveT", C.c_double),
                ("ms_axpby_sym", C.c_double), ("launches", C.c_longlong), ("max_rank", C.c_int),
                ("memory_bytes", C.c_longlong), ("trace", C.c_double), ("kcap", C.c_int),
                ("trunc_bytes", C.c_double), ("gemm_flops", C.c_double), ("trunc_tasks", C.c_longlong),
                ("profiled", C.c_int), ("prof_ms_trunc", C.c_double), ("prof_ms_gemm", C.c_double),
                ("prof_ms_hsolve", C.c_double), ("prof_ms_leaf", C.c_double),
                ("prof_batches_trunc", C.c_longlong), ("prof_batches_gemm", C.c_longlong),
                ("prof_batches_hsolve", C.c_longlong), ("prof_batches_leaf", C.c_longlong),
                ("graph_used", C.c_int), ("graph_nodes", C.c_longlong),
                ("ph_trunc_bytes", C.c_double * 8), ("ph_qr_flops", C.c_double * 8), ("ph_core_flops", C.c_double * 8),
                ("ph_gemm_flops", C.c_double * 8), ("ph_leaf_flops", C.c_double * 8)]

PHASES = ("setup", "first", "multiply", "cholesky", "solve", "solveT", "axpby_sym")


class _Diag(C.Structure):
    _fields_ = [("k", C.c_int), ("l", C.c_double), ("c", C.c_double), ("max_rank", C.c_int),
                ("memory_bytes", C.c_longlong), ("wall_ms", C.c_double)]


_LIB = None

# exported symbols of include/specproj_b200.h (checked by tests/test_abi.py)
ABI_SYMBOLS = (
    "spg_hqdwh", "spg_result_info", "spg_result_diag", "spg_result_flat_size", "spg_result_export",
    "spg_result_apply", "spg_result_free", "spg_last_error", "spg_tree", "spg_qdwh_params", "spg_l_update",
    "spg_make_dimer_chain", "spg_make_random_banded", "spg_kcap", "spg_ctx_create", "spg_ctx_free",
    "spg_ctx_upload", "spg_ctx_flat_size", "spg_ctx_download", "spg_ctx_op", "spg_ctx_from_banded",
    "spg_truncate", "spg_set_profile", "spg_measure_dmma_tflops", "spg_host_alloc",
    "spg_host_free", "spg_hqdwh_shifts", "spg_hqdwh_shifts_devices", "spg_result_device", "spg_release_plan_cache", "spg_stacked_qr_r",
)


def load_library(path: str | None = None):
    """Loads (once) the in-tree C-ABI library; raises if it is missing."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or _LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(p)
    vp = C.c_void_p
    sig = {
        "spg_hqdwh": ([C.c_int, C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.POINTER(vp)], C.c_int),
        "spg_result_info": ([vp, C.POINTER(_Info)], C.c_int),
        "spg_result_diag": ([vp, C.POINTER(_Diag)], C.c_int),
        "spg_result_flat_size": ([vp, C.c_int, C.POINTER(C.c_longlong)], C.c_int),
        "spg_result_export": ([vp, C.c_int, _ip, _dp], C.c_int),
        "spg_result_apply": ([vp, C.c_int, C.c_int, _dp, _dp], C.c_int),
        "spg_result_free": ([vp], None),
        "spg_last_error": ([], C.c_char_p),
        "spg_tree": ([C.c_int, C.c_int, _ip, _ip, _ip, _ip, _ip], C.c_int),
        "spg_qdwh_params": ([C.c_double, _dp], C.c_int),
        "spg_l_update": ([C.c_double] * 4, C.c_double),
        "spg_make_dimer_chain": ([C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_ulonglong, _dp], C.c_int),
        "spg_make_random_banded": ([C.c_int, C.c_int, C.c_ulonglong, _dp], C.c_int),
        "spg_kcap": ([], C.c_int),
        "spg_release_plan_cache": ([], C.c_int),
        "spg_stacked_qr_r": ([C.c_int, C.c_int, _dp, C.c_int, _dp], C.c_int),
        "spg_ctx_create": ([C.c_int, C.c_int, C.c_double, C.c_int], vp),
        "spg_ctx_free": ([vp], None),
        "spg_ctx_upload": ([vp, C.c_int, _ip, _dp], C.c_int),
        "spg_ctx_flat_size": ([vp, C.c_int, C.POINTER(C.c_longlong)], C.c_int),
        "spg_ctx_download": ([vp, C.c_int, _ip, _dp], C.c_int),
        "spg_ctx_op": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double], C.c_int),
        "spg_ctx_from_banded": ([vp, C.c_int, C.c_int, _dp], C.c_int),
        "spg_truncate": ([C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, _dp, _dp, _ip], C.c_int),
        "spg_set_profile": ([C.c_int], None),
        "spg_measure_dmma_tflops": ([_dp], C.c_int),
        "spg_host_alloc": ([C.c_longlong, C.POINTER(vp)], C.c_int),
        "spg_host_free": ([vp], None),
        "spg_hqdwh_shifts": ([C.c_int, C.c_int, _dp, C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.c_int,
                              C.POINTER(vp)], C.c_int),
        "spg_hqdwh_shifts_devices": ([C.c_int, C.c_int, _dp, C.c_int, _dp, C.c_int, C.c_double, C.c_double, C.c_int,
                                      _ip, C.c_int, C.POINTER(vp), _ip], C.c_int),
        "spg_result_device": ([vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("SPG_LIB") and not hasattr(L, name):
            continue   # an older build of the C-ABI picked through SPG_LIB (bisecting)
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if path is None:
        _LIB = L
    return L


def _raise(code: int):
    if code == _OK:
        return
    msg = load_library().spg_last_error().decode()
    exc = {_NPD: NotPositiveDefiniteError, _SING: SingularMatrixError, _INV: ValueError, _DOM: ArithmeticError,
           _RANK: RankCapacityError, _CUDA: CudaError, _NODEV: NoDeviceError}.get(code, RuntimeError)
    raise exc(msg)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


# ---------------------------------------------------------------- banded input
class BandedSymmetric:
    """banded.hpp:19-51: lower bands ``bands[d][i] = A(i+d, i)``, d = 0..b."""

    def __init__(self, n: int, b: int, bands=None):
        if n < 2:
            raise ValueError("BandedSymmetric: n >= 2 required")
        if b < 1 or b >= n:
            raise ValueError("BandedSymmetric: 1 <= b < n required")
        self.n, self.b = n, b
        self.bands = [np.zeros(n - d) for d in range(b + 1)] if bands is None else \
            [np.asarray(x, dtype=np.float64).copy() for x in bands]
        if len(self.bands) != b + 1 or any(len(self.bands[d]) != n - d for d in range(b + 1)):
            raise ValueError("BandedSymmetric: band lengths must be n - d")

    @classmethod
    def from_packed(cls, n, b, packed):
        out, off = [], 0
        for d in range(b + 1):
            out.append(np.array(packed[off:off + n - d]))
            off += n - d
        return cls(n, b, out)

    def packed(self) -> np.ndarray:
        return np.ascontiguousarray(np.concatenate(self.bands))

    def at(self, i, j):
        d = abs(i - j)
        return 0.0 if d > self.b else float(self.bands[d][min(i, j)])

    def scaled(self, s):
        return BandedSymmetric(self.n, self.b, [x * s for x in self.bands])

    def shifted(self, mu):
        """A - mu I (the CLI's --shift, tools/specproj.cpp:160-161)."""
        B = BandedSymmetric(self.n, self.b, self.bands)
        B.bands[0] = B.bands[0] - mu
        return B

    def all_finite(self):
        return all(np.all(np.isfinite(x)) for x in self.bands)

    def to_dense(self):
        M = np.zeros((self.n, self.n))
        for d, x in enumerate(self.bands):
            i = np.arange(self.n - d)
            M[i + d, i] = x
            M[i, i + d] = x
        return M


def dimer_chain(n, t1, t2, eps_dis, seed, b=1, s=0.0) -> BandedSymmetric:
    """SURVEY.md §8d dimer chain: bond i is t1 for even i, t2 for odd i; diagonal
    eps_dis * U(-1,1); optional symmetric band perturbation s * U(-1,1) for d <= b
    (std::mt19937_64 + uniform_real_distribution<double>(-1, 1))."""
    out = np.zeros((b + 1) * n - b * (b + 1) // 2)
    _raise(load_library().spg_make_dimer_chain(n, b, t1, t2, eps_dis, s, seed, _d(out)))
    return BandedSymmetric.from_packed(n, b, out)


def random_banded(n, b, seed) -> BandedSymmetric:
    """test_hodlr.cpp:19-26 random_banded."""
    out = np.zeros((b + 1) * n - b * (b + 1) // 2)
    _raise(load_library().spg_make_random_banded(n, b, seed, _d(out)))
    return BandedSymmetric.from_packed(n, b, out)


# ---------------------------------------------------------------- tree / HODLR
class PartitionTree:
    """tree.hpp:12-56 (computed by the C-ABI host helper)."""

    def __init__(self, n, n_min):
        L = load_library()
        nn = L.spg_tree(n, n_min, None, None, None, None, None)
        if nn < 0:
            _raise(-nn)
        self.begin, self.size, self.left, self.right = (np.zeros(nn, dtype=np.int32) for _ in range(4))
        depth = np.zeros(1, dtype=np.int32)
        L.spg_tree(n, n_min, _i(self.begin), _i(self.size), _i(self.left), _i(self.right), _i(depth))
        self.n, self.n_min, self.depth = n, n_min, int(depth[0])

    def __len__(self):
        return len(self.begin)

    def leaf(self, i):
        return self.left[i] < 0


def make_tree(n, n_min):
    return PartitionTree(n, n_min)


class _HostSlot:
    """A page-locked host buffer of the export pool (reused across results)."""

    def __init__(self, n):
        L = load_library()
        self.ptr = C.c_void_p()
        self.n = max(int(n), 1)
        _raise(L.spg_host_alloc(8 * self.n, C.byref(self.ptr)))
        self.busy = True

    def release(self):
        self.busy = False

    def __del__(self):
        try:
            load_library().spg_host_free(self.ptr)
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass


_HOST_POOL: list = []


def _host_buffer(n: int) -> _HostSlot:
    for slot in _HOST_POOL:
        if not slot.busy and slot.n >= n:
            slot.busy = True
            return slot
    slot = _HostSlot(n)
    _HOST_POOL.append(slot)
    return slot


class HodlrMatrix:
    """Host copy of a device HODLR matrix (hodlr.hpp:20-48).  Nodes in preorder;
    ``dense[id]`` for leaves, ``upper[id] = (U, V)`` / ``lower[id]`` otherwise."""

    def __init__(self, tree: PartitionTree):
        self.tree = tree
        self.dense, self.upper, self.lower = {}, {}, {}

    @classmethod
    def from_flat(cls, tree, ranks, data):
        H = cls(tree)
        off = 0

        def take(r, c):   # views into the flat buffer (no copies)
            nonlocal off
            m = data[off:off + r * c].reshape(r, c)
            off += r * c
            return m

        for i in range(len(tree)):
            if tree.leaf(i):
                H.dense[i] = take(tree.size[i], tree.size[i])
                continue
            s1, s2 = int(tree.size[tree.left[i]]), int(tree.size[tree.right[i]])
            ku, kl = int(ranks[2 * i]), int(ranks[2 * i + 1])
            Uu = take(s1, ku); Vu = take(s2, ku); Ul = take(s2, kl); Vl = take(s1, kl)
            H.upper[i] = (Uu, Vu)
            H.lower[i] = (Ul, Vl)
        return H

    def to_flat(self):
        t = self.tree
        ranks = np.zeros(2 * len(t), dtype=np.int32)
        parts = []
        for i in range(len(t)):
            if t.leaf(i):
                parts.append(np.ascontiguousarray(self.dense[i]).ravel())
                continue
            (Uu, Vu), (Ul, Vl) = self.upper[i], self.lower[i]
            ranks[2 * i], ranks[2 * i + 1] = Uu.shape[1], Ul.shape[1]
            parts += [np.ascontiguousarray(x).ravel() for x in (Uu, Vu, Ul, Vl)]
        return ranks, np.ascontiguousarray(np.concatenate(parts), dtype=np.float64)

    @property
    def n(self):
        return self.tree.n

    def to_dense(self):
        """to_dense (hodlr.hpp:253-257)"""
        t = self.tree
        M = np.zeros((t.n, t.n))
        for i in range(len(t)):
            b, s = int(t.begin[i]), int(t.size[i])
            if t.leaf(i):
                M[b:b + s, b:b + s] = self.dense[i]
                continue
            m = int(t.begin[t.right[i]])
            s2 = int(t.size[t.right[i]])
            U, V = self.upper[i]
            if U.shape[1]:
                M[b:m, m:m + s2] = U @ V.T
            U, V = self.lower[i]
            if U.shape[1]:
                M[m:m + s2, b:m] = U @ V.T
        return M

    def matmat(self, X):
        """h_apply (hodlr.hpp:277) on the host copy."""
        X = np.asarray(X, dtype=np.float64)
        Y = np.zeros_like(X)
        t = self.tree
        for i in range(len(t)):
            b, s = int(t.begin[i]), int(t.size[i])
            if t.leaf(i):
                Y[b:b + s] += self.dense[i] @ X[b:b + s]
                continue
            m = int(t.begin[t.right[i]])
            s2 = int(t.size[t.right[i]])
            U, V = self.upper[i]
            if U.shape[1]:
                Y[b:m] += U @ (V.T @ X[m:m + s2])
            U, V = self.lower[i]
            if U.shape[1]:
                Y[m:m + s2] += U @ (V.T @ X[b:m])
        return Y

    def trace(self):
        """hodlr_trace (hodlr.hpp:658-663)"""
        return float(sum(np.trace(D) for D in self.dense.values()))

    def diagnostics(self):
        """diagnostics (hodlr.hpp:679-695) -> (max off-diagonal rank, memory bytes)"""
        mx, ent = 0, sum(D.size for D in self.dense.values())
        for i in self.upper:
            for U, V in (self.upper[i], self.lower[i]):
                mx = max(mx, U.shape[1])
                ent += U.shape[1] * (U.shape[0] + V.shape[0])
        return mx, 8 * ent

    def ranks(self):
        """per preorder internal node: (rank upper, rank lower)"""
        return {i: (self.upper[i][0].shape[1], self.lower[i][0].shape[1]) for i in self.upper}


# ---------------------------------------------------------------- hQDWH
@dataclass
class IterationDiag:
    """qdwh.hpp:176-183"""
    k: int
    l: float
    c: float
    max_rank: int
    memory_bytes: int
    wall_ms: float


@dataclass
class ProjectorResult:
    """qdwh.hpp:185-192 plus device timings.  P / U are fetched lazily from device."""
    iterations: int
    alpha: float
    l0: float
    per_iteration: list = field(default_factory=list)
    info: dict = field(default_factory=dict)
    _handle: object = None
    _tree: object = None

    def _fetch(self, which):
        L = load_library()
        nd = C.c_longlong(0)
        _raise(L.spg_result_flat_size(self._handle, which, C.byref(nd)))
        ranks = np.zeros(2 * len(self._tree), dtype=np.int32)
        slot = _host_buffer(nd.value)
        # a fresh ctypes view per lease: every block array of the result keeps it alive,
        # and the pool gets the buffer back only when the last of them is gone
        lease = (C.c_double * max(nd.value, 1)).from_address(slot.ptr.value)
        weakref.finalize(lease, slot.release)
        data = np.ctypeslib.as_array(lease)[:nd.value]
        _raise(L.spg_result_export(self._handle, which, _i(ranks), _d(data)))
        return HodlrMatrix.from_flat(self._tree, ranks, data)

    @property
    def P(self) -> HodlrMatrix:
        if "_P" not in self.__dict__:
            self.__dict__["_P"] = self._fetch(0)
        return self.__dict__["_P"]

    @property
    def U(self) -> HodlrMatrix:
        if "_U" not in self.__dict__:
            self.__dict__["_U"] = self._fetch(1)
        return self.__dict__["_U"]

    def apply(self, X, which=0):
        """P X (which=0) or U X (which=1) on the device, X host n x m (m <= KCAP)."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.zeros_like(X)
        _raise(load_library().spg_result_apply(self._handle, which, X.shape[1], _d(X), _d(Y)))
        return Y

    def close(self):
        if self._handle:
            load_library().spg_result_free(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hqdwh(A: BandedSymmetric, n_min: int, eps: float, delta: float = 1e-15, packed=None) -> ProjectorResult:
    """hqdwh (qdwh.hpp:196-241) on the B200: spectral projector onto the negative
    eigenvalues of A.  Raises the reference's exception types.  ``packed`` may be
    a caller-owned (e.g. pinned) float64 buffer already holding ``A.packed()``."""
    L = load_library()
    h = C.c_void_p()
    if packed is None:
        if not A.all_finite():
            raise ValueError("hqdwh: nonfinite input")
        packed = A.packed()
    _raise(L.spg_hqdwh(A.n, A.b, _d(packed), n_min, eps, delta, C.byref(h)))
    return _result_from_handle(h, A.n, n_min)


def _result_from_handle(h, n, n_min) -> ProjectorResult:
    L = load_library()
    info = _Info()
    _raise(L.spg_result_info(h, C.byref(info)))
    diag = (_Diag * max(info.iterations, 1))()
    _raise(L.spg_result_diag(h, diag))
    per = [IterationDiag(d.k, d.l, d.c, d.max_rank, d.memory_bytes, d.wall_ms) for d in diag[:info.iterations]]
    infod = {name: getattr(info, name) for name, _ in _Info._fields_}
    for name, _ in _Info._fields_:
        if name.startswith("ph_"):
            infod[name] = list(infod[name])[:len(PHASES)]
    return ProjectorResult(info.iterations, info.alpha, info.l0, per, infod, h, PartitionTree(n, n_min))


def hqdwh_shifts(A: BandedSymmetric, shifts, n_min: int, eps: float, delta: float = 1e-15,
                 max_concurrent: int = 2) -> list:
    """Spectral slicing (the CLI's --shift, tools/specproj.cpp:160-161, for several shifts):
    one projector of A - mu I per shift, run concurrently on the device (spg_hqdwh_shifts)."""
    if not A.all_finite():
        raise ValueError("hqdwh: nonfinite input")
    sh = np.ascontiguousarray(shifts, dtype=np.float64)
    hs = (C.c_void_p * len(sh))()
    _raise(load_library().spg_hqdwh_shifts(A.n, A.b, _d(A.packed()), len(sh), _d(sh), n_min, eps, delta,
                                           max_concurrent, hs))
    return [_result_from_handle(C.c_void_p(h), A.n, n_min) for h in hs]


def hqdwh_shifts_devices(A: BandedSymmetric, shifts, n_min: int, eps: float, delta: float = 1e-15,
                         devices=None, per_device_concurrent: int = 2):
    """Spectral slicing over the GPUs of this process (spg_hqdwh_shifts_devices): replicas, one
    projector per GPU at a time and no data-path collective.  Returns
    (results, device_of) in the order of `shifts`."""
    if not A.all_finite():
        raise ValueError("hqdwh: nonfinite input")
    sh = np.ascontiguousarray(shifts, dtype=np.float64)
    hs = (C.c_void_p * len(sh))()
    dev_of = np.full(len(sh), -1, dtype=np.int32)
    dv = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
    _raise(load_library().spg_hqdwh_shifts_devices(
        A.n, A.b, _d(A.packed()), len(sh), _d(sh), n_min, eps, delta, 0 if dv is None else len(dv),
        None if dv is None else dv.ctypes.data_as(_ip), per_device_concurrent, hs, dev_of.ctypes.data_as(_ip)))
    return [_result_from_handle(C.c_void_p(h), A.n, n_min) for h in hs], dev_of.tolist()


def shard_shifts(nshift: int, rank: int, world: int) -> list:
    """Indices of the shifts rank `rank` of `world` evaluates in the one-process-per-GPU model
    (torchrun): round-robin, so neighbouring shifts (similar cost) spread over the ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_shifts: 0 <= rank < world required")
    return list(range(rank, nshift, world))


def hqdwh_shifts_sharded(A: BandedSymmetric, shifts, n_min: int, eps: float, delta: float = 1e-15,
                         rank: int | None = None, world: int | None = None, max_concurrent: int = 2,
                         summarize=None, project=None):
    """Spectral slicing across ranks (one process per GPU, torch.distributed): rank r computes the
    projectors of shifts r, r + world, ... on ITS device; no matrix data crosses ranks.  Only a
    per-shift summary (default: round(trace) = the eigenvalue count below the shift, iterations,
    max rank) is all-gathered, so every rank returns (local_results, summaries_in_shift_order).
    `project` (tests) replaces the device call."""
    import torch.distributed as dist
    inited = dist.is_available() and dist.is_initialized()
    if world is None:
        world = dist.get_world_size() if inited else 1
    if rank is None:
        rank = dist.get_rank() if inited else 0
    sh = [float(x) for x in shifts]
    mine = shard_shifts(len(sh), rank, world)
    run = project or (lambda mus: hqdwh_shifts(A, mus, n_min, eps, delta, max_concurrent) if mus else [])
    local = run([sh[i] for i in mine])
    summ = summarize or (lambda r: {"count": int(round(r.info["trace"])), "iterations": r.iterations,
                                    "max_rank": r.info["max_rank"]})
    part = [(i, summ(r)) for i, r in zip(mine, local)]
    if world > 1:
        if not inited:
            raise RuntimeError("hqdwh_shifts_sharded: world > 1 needs an initialised torch.distributed group")
        parts = [None] * world
        dist.all_gather_object(parts, part)
    else:
        parts = [part]
    out = [None] * len(sh)
    for pr in parts:
        for i, v in pr:
            out[i] = v
    return dict(zip(mine, local)), out


# ------------------------------------------------------------------ wire formats (banded.hpp:115-154)
def write_sbm(path: str, A: BandedSymmetric):
    """SBM text: "SBM <n> <b>", then one line per diagonal (%.17g, full round trip)."""
    with open(path, "w") as f:
        f.write(f"SBM {A.n} {A.b}\n")
        for d in range(A.b + 1):
            f.write(" ".join("%.17g" % v for v in A.bands[d]) + "\n")


def read_sbm(path: str) -> BandedSymmetric:
    with open(path) as f:
        tok = f.read().split()
    if len(tok) < 3 or tok[0] != "SBM":
        raise ValueError("read_sbm: malformed header")
    n, b = int(tok[1]), int(tok[2])
    need = sum(n - d for d in range(b + 1))
    if len(tok) - 3 < need:
        raise ValueError("read_sbm: truncated data")
    vals = np.array([float(t) for t in tok[3:3 + need]])
    if not np.all(np.isfinite(vals)):
        raise ValueError("read_sbm: nonfinite entry")
    return BandedSymmetric.from_packed(n, b, vals)


def run_report(file: str, A: BandedSymmetric, n_min: int, eps: float, delta: float, shift: float,
               r: ProjectorResult, wall_ms: float, errors=None, gap=None, seed=None) -> dict:
    """The JSON run report of tools/specproj.cpp:82-118 (same keys and order)."""
    P = r.P
    mr, mem = P.diagnostics()
    return {
        "input": {"file": file, "n": A.n, "b": A.b, "gap": gap, "seed": seed},
        "params": {"n_min": n_min, "eps": eps, "delta": delta, "shift": shift, "alpha": r.alpha, "l0": r.l0},
        "iterations": r.iterations,
        "per_iteration": [{"k": d.k, "l": d.l, "c": d.c, "max_rank": d.max_rank, "memory_bytes": d.memory_bytes,
                           "wall_ms": d.wall_ms} for d in r.per_iteration],
        "errors": errors,
        "totals": {"wall_ms": wall_ms, "memory_bytes": int(mem), "max_rank": int(mr), "trace_p": P.trace()},
    }


def cli_path() -> str:
    """The GPU-backed CLI (tools/specproj.cpp subcommands), built next to the library."""
    return os.path.join(os.path.dirname(_LIB_PATH), "specproj_b200")


def stacked_qr_r(A: BandedSymmetric, method: str = "givens") -> np.ndarray:
    """R of the stacked QR of [A; I] on the device (reduce_tridiag / reduce_banded,
    fast_qr.hpp:83-232): diagonals (2b+1, n), rd[d, i] = R(i, i+d).  method "givens" is the
    rotation sweep, "cholesky" the band Cholesky of A^2 + I (equal up to row signs)."""
    out = np.zeros((2 * A.b + 1) * A.n)
    _raise(load_library().spg_stacked_qr_r(A.n, A.b, _d(A.packed()), 1 if method == "givens" else 0, _d(out)))
    return out.reshape(2 * A.b + 1, A.n)


def release_plan_cache() -> int:
    """Frees every cached projector plan (spg_release_plan_cache)."""
    return int(load_library().spg_release_plan_cache())


def set_profile(on: bool = True):
    """Profile mode: bracket every batched launch with CUDA events (per-class device times in info)."""
    load_library().spg_set_profile(1 if on else 0)


def measure_dmma_tflops() -> float:
    """Measured FP64 tensor-pipe (DMMA.8x8x4) throughput of device 0 in TFLOP/s."""
    out = np.zeros(1)
    _raise(load_library().spg_measure_dmma_tflops(_d(out)))
    return float(out[0])


def qdwh_params(l):
    """qdwh_params (qdwh.hpp:27-35)"""
    out = np.zeros(3)
    _raise(load_library().spg_qdwh_params(l, _d(out)))
    return tuple(float(x) for x in out)


def l_update(l, a, b, c):
    """l_update (qdwh.hpp:38-40)"""
    return load_library().spg_l_update(l, a, b, c)


def truncate(U, V, eps):
    """truncate (lowrank.hpp:67-86) of one block on the device."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    p, k = U.shape
    s = V.shape[0]
    Uo = np.zeros((p, k)); Vo = np.zeros((s, k))
    r = np.zeros(1, dtype=np.int32)
    _raise(load_library().spg_truncate(p, s, k, _d(U), _d(V), eps, _d(Uo), _d(Vo), _i(r)))
    return Uo[:, :r[0]].copy(), Vo[:, :r[0]].copy()


class HodlrContext:
    """Device slots of HODLR matrices on one tree for component-level operations
    (hodlr_multiply, hodlr_axpby, hodlr_symmetrize, hodlr_cholesky,
    solve_upper_right, solve_upperT_right, hodlr_scale + add_scaled_identity)."""

    OPS = {"multiply": 1, "axpby": 2, "symmetrize": 3, "cholesky": 4, "solve_upper_right": 5,
           "solve_upperT_right": 6, "scale_shift": 7, "multiply_upper": 8, "cholesky_deferred": 9}

    def __init__(self, n, n_min, eps, nslots=4):
        L = load_library()
        self.h = L.spg_ctx_create(n, n_min, eps, nslots)
        if not self.h:
            raise RuntimeError(L.spg_last_error().decode())
        self.tree = PartitionTree(n, n_min)

    def upload(self, slot, H: HodlrMatrix):
        ranks, data = H.to_flat()
        _raise(load_library().spg_ctx_upload(self.h, slot, _i(ranks), _d(data)))

    def from_banded(self, slot, A: BandedSymmetric):
        p = A.packed()
        _raise(load_library().spg_ctx_from_banded(self.h, slot, A.b, _d(p)))

    def download(self, slot) -> HodlrMatrix:
        L = load_library()
        nd = C.c_longlong(0)
        _raise(L.spg_ctx_flat_size(self.h, slot, C.byref(nd)))
        ranks = np.zeros(2 * len(self.tree), dtype=np.int32)
        data = np.zeros(nd.value)
        _raise(L.spg_ctx_download(self.h, slot, _i(ranks), _d(data)))
        return HodlrMatrix.from_flat(self.tree, ranks, data)

    def op(self, name, dst, a=0, b=0, alpha=0.0, beta=0.0):
        _raise(load_library().spg_ctx_op(self.h, self.OPS[name], dst, a, b, alpha, beta))

    def close(self):
        if self.h:
            load_library().spg_ctx_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
