"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's HODLR path.

This is the checker, never the product: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg may import it.  Every function restates the
reference function cited next to it (paths relative to
/root/reference/proj/include/specproj/).  Dense kernels (Householder QR,
one-sided Jacobi SVD, Cholesky, triangular solves) are the same mathematical
operations done by LAPACK through numpy/scipy; the HODLR recursion, truncation
rule (absolute, keep sigma > eps: lowrank.hpp:74) and operation order follow the
reference exactly.  Pinned against oracle/_ref (the reference compiled from its
own sources) in tests/test_oracle.py.  Pure-Python recursion: small n only.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class NotPositiveDefiniteError(RuntimeError):
    """dense_factor.hpp:19-21"""


class SingularMatrixError(RuntimeError):
    """dense_factor.hpp:23-25"""


# --------------------------------------------------------------------------- tree
class Tree:
    """PartitionTree (tree.hpp:12-56): preorder nodes, split at ceil(size/2)."""

    def __init__(self, n: int, n_min: int):
        if n < 1:
            raise ValueError("PartitionTree: n >= 1 required")
        if n_min < 2:
            raise ValueError("PartitionTree: n_min >= 2 required")
        self.n, self.n_min, self.depth = n, n_min, 0
        self.begin, self.size, self.left, self.right = [], [], [], []
        self._build(0, n, 0)

    def _build(self, begin, size, level):
        nid = len(self.begin)
        self.begin.append(begin); self.size.append(size); self.left.append(-1); self.right.append(-1)
        if size > self.n_min:
            self.depth = max(self.depth, level + 1)
            s1 = (size + 1) // 2
            l = self._build(begin, s1, level + 1)
            r = self._build(begin + s1, size - s1, level + 1)
            self.left[nid], self.right[nid] = l, r
        return nid

    def leaf(self, i):
        return self.left[i] < 0

    def __len__(self):
        return len(self.begin)


def _empty(p, s):
    return (np.zeros((p, 0)), np.zeros((s, 0)))


class Hodlr:
    """HodlrMatrix (hodlr.hpp:20-48): dense leaves, (U, V) upper/lower per internal node."""

    def __init__(self, tree: Tree):
        self.tree = tree
        self.dense, self.up, self.lo = {}, {}, {}
        for i in range(len(tree)):
            if tree.leaf(i):
                self.dense[i] = np.zeros((tree.size[i], tree.size[i]))
            else:
                s1, s2 = tree.size[tree.left[i]], tree.size[tree.right[i]]
                self.up[i] = _empty(s1, s2)
                self.lo[i] = _empty(s2, s1)

    def copy(self):
        H = Hodlr.__new__(Hodlr)
        H.tree = self.tree
        H.dense = {k: v.copy() for k, v in self.dense.items()}
        H.up = {k: (u.copy(), v.copy()) for k, (u, v) in self.up.items()}
        H.lo = {k: (u.copy(), v.copy()) for k, (u, v) in self.lo.items()}
        return H

    @property
    def n(self):
        return self.tree.n


def identity(tree):
    """hodlr_identity (hodlr.hpp:56-64)"""
    H = Hodlr(tree)
    for i in H.dense:
        H.dense[i] = np.eye(tree.size[i])
    return H


# ------------------------------------------------------------------ low-rank
def truncate(U, V, eps):
    """truncate (lowrank.hpp:67-86): QR(U), QR(V), SVD(R_u R_v^T), keep sigma > eps."""
    if U.shape[1] == 0:
        return U, V
    Qu, Ru = np.linalg.qr(U)
    Qv, Rv = np.linalg.qr(V)
    core = Ru @ Rv.T
    X, sig, Yt = np.linalg.svd(core, full_matrices=False)
    k = int(np.sum(sig > eps))
    # kept singular values are a prefix (descending order)
    return Qu @ (X[:, :k] * sig[:k]), Qv @ Yt[:k].T


def lr_concat(A, B):
    """lr_concat (lowrank.hpp:43-63)"""
    if A[0].shape[1] == 0:
        return B
    if B[0].shape[1] == 0:
        return A
    return np.hstack([A[0], B[0]]), np.hstack([A[1], B[1]])


def lr_multiply(A, B):
    """lr_multiply (lowrank.hpp:89-93): (Ua (Va^T Ub)) Vb^T"""
    if A[0].shape[1] == 0 or B[0].shape[1] == 0:
        return _empty(A[0].shape[0], B[1].shape[0])
    return A[0] @ (A[1].T @ B[0]), B[1]


def lr_dense(B):
    return B[0] @ B[1].T


# ------------------------------------------------------------------- banded
def banded_at(A, i, j):
    """BandedSymmetric::at (banded.hpp:33-37); A = list of diagonals."""
    d = abs(i - j)
    if d >= len(A):
        return 0.0
    return A[d][min(i, j)]


def banded_to_dense(bands):
    n = len(bands[0])
    M = np.zeros((n, n))
    for d, diag in enumerate(bands):
        idx = np.arange(n - d)
        M[idx + d, idx] = diag
        M[idx, idx + d] = diag
    return M


def _trim(U, V, judge_v):
    """trim_zero_columns (hodlr.hpp:70-86)"""
    W = V if judge_v else U
    keep = [t for t in range(W.shape[1]) if np.any(W[:, t] != 0.0)]
    return U[:, keep], V[:, keep]


def from_banded(bands, tree):
    """from_banded (hodlr.hpp:92-146): exact band-corner factors of rank <= b."""
    b = len(bands) - 1
    H = Hodlr(tree)
    D = banded_to_dense(bands)
    for i in range(len(tree)):
        bg, sz = tree.begin[i], tree.size[i]
        if tree.leaf(i):
            H.dense[i] = D[bg:bg + sz, bg:bg + sz].copy()
            continue
        mid = tree.begin[tree.right[i]]
        s1, s2 = tree.size[tree.left[i]], tree.size[tree.right[i]]
        kr, kc = min(b, s1), min(b, s2)
        if kr <= kc:
            U = np.zeros((s1, kr)); V = np.zeros((s2, kr))
            for t in range(kr):
                U[s1 - kr + t, t] = 1.0
                V[:, t] = D[mid - kr + t, mid:mid + s2]
            H.up[i] = _trim(U, V, True)
        else:
            U = np.zeros((s1, kc)); V = np.zeros((s2, kc))
            for t in range(kc):
                V[t, t] = 1.0
                U[:, t] = D[bg:bg + s1, mid + t]
            H.up[i] = _trim(U, V, False)
        if kc <= kr:
            U = np.zeros((s2, kc)); V = np.zeros((s1, kc))
            for t in range(kc):
                U[t, t] = 1.0
                V[:, t] = D[mid + t, bg:bg + s1]
            H.lo[i] = _trim(U, V, True)
        else:
            U = np.zeros((s2, kr)); V = np.zeros((s1, kr))
            for t in range(kr):
                V[s1 - kr + t, t] = 1.0
                U[:, t] = D[mid:mid + s2, mid - kr + t]
            H.lo[i] = _trim(U, V, False)
    return H


def to_dense(H):
    """to_dense / fill_dense (hodlr.hpp:150-167, 253-257)"""
    t = H.tree
    M = np.zeros((t.n, t.n))
    for i in range(len(t)):
        bg, sz = t.begin[i], t.size[i]
        if t.leaf(i):
            M[bg:bg + sz, bg:bg + sz] = H.dense[i]
        else:
            mid = t.begin[t.right[i]]
            s1, s2 = t.size[t.left[i]], t.size[t.right[i]]
            if H.up[i][0].shape[1]:
                M[bg:mid, mid:mid + s2] = lr_dense(H.up[i])
            if H.lo[i][0].shape[1]:
                M[mid:mid + s2, bg:mid] = lr_dense(H.lo[i])
    return M


def _apply(H, i, X, Y, base):
    """apply_rec (hodlr.hpp:202-224): Y[rows(i)] += H(i) X[rows(i)]"""
    t = H.tree
    l0 = t.begin[i] - base
    if t.leaf(i):
        Y[l0:l0 + t.size[i]] += H.dense[i] @ X[l0:l0 + t.size[i]]
        return
    _apply(H, t.left[i], X, Y, base)
    _apply(H, t.right[i], X, Y, base)
    m = t.begin[t.right[i]] - base
    s1, s2 = t.size[t.left[i]], t.size[t.right[i]]
    U, V = H.up[i]
    if U.shape[1]:
        Y[l0:l0 + s1] += U @ (V.T @ X[m:m + s2])
    U, V = H.lo[i]
    if U.shape[1]:
        Y[m:m + s2] += U @ (V.T @ X[l0:l0 + s1])


def _applyT(H, i, X, Y, base):
    """applyT_rec (hodlr.hpp:226-249)"""
    t = H.tree
    l0 = t.begin[i] - base
    if t.leaf(i):
        Y[l0:l0 + t.size[i]] += H.dense[i].T @ X[l0:l0 + t.size[i]]
        return
    _applyT(H, t.left[i], X, Y, base)
    _applyT(H, t.right[i], X, Y, base)
    m = t.begin[t.right[i]] - base
    s1, s2 = t.size[t.left[i]], t.size[t.right[i]]
    U, V = H.up[i]
    if U.shape[1]:
        Y[m:m + s2] += V @ (U.T @ X[l0:l0 + s1])
    U, V = H.lo[i]
    if U.shape[1]:
        Y[l0:l0 + s1] += V @ (U.T @ X[m:m + s2])


def apply_sub(H, i, X):
    """h_apply_sub (hodlr.hpp:261-267)"""
    Y = np.zeros_like(X)
    _apply(H, i, X, Y, H.tree.begin[i])
    return Y


def applyT_sub(H, i, X):
    """h_applyT_sub (hodlr.hpp:269-275)"""
    Y = np.zeros_like(X)
    _applyT(H, i, X, Y, H.tree.begin[i])
    return Y


def apply(H, X):
    return apply_sub(H, 0, X)


def scale(H, a):
    """hodlr_scale (hodlr.hpp:289-296)"""
    for i in H.dense:
        H.dense[i] = H.dense[i] * a
    for i in H.up:
        H.up[i] = (H.up[i][0] * a, H.up[i][1])
        H.lo[i] = (H.lo[i][0] * a, H.lo[i][1])


def add_scaled_identity(H, mu):
    """add_scaled_identity (hodlr.hpp:299-305)"""
    for i in H.dense:
        H.dense[i] = H.dense[i] + mu * np.eye(H.dense[i].shape[0])


def transpose(H):
    """hodlr_transpose (hodlr.hpp:307-318)"""
    T = Hodlr.__new__(Hodlr)
    T.tree = H.tree
    T.dense = {k: v.T.copy() for k, v in H.dense.items()}
    T.up = {k: (H.lo[k][1], H.lo[k][0]) for k in H.up}
    T.lo = {k: (H.up[k][1], H.up[k][0]) for k in H.up}
    return T


def axpby(a, A, b, B, eps):
    """hodlr_axpby (hodlr.hpp:321-339)"""
    C = Hodlr.__new__(Hodlr)
    C.tree = A.tree
    C.dense = {k: a * A.dense[k] + b * B.dense[k] for k in A.dense}
    C.up, C.lo = {}, {}
    for k in A.up:
        C.up[k] = truncate(*lr_concat((A.up[k][0] * a, A.up[k][1]), (B.up[k][0] * b, B.up[k][1])), eps)
        C.lo[k] = truncate(*lr_concat((A.lo[k][0] * a, A.lo[k][1]), (B.lo[k][0] * b, B.lo[k][1])), eps)
    return C


def symmetrize(H, eps):
    """hodlr_symmetrize (hodlr.hpp:346-364)"""
    for k in H.dense:
        D = H.dense[k]
        H.dense[k] = np.tril(0.5 * (D + D.T), -1) + np.tril(0.5 * (D + D.T), -1).T + np.diag(np.diag(D))
    for k in H.up:
        U, V = H.up[k]
        Ul, Vl = H.lo[k]
        up = truncate(*lr_concat((0.5 * U, V), (0.5 * Vl, Ul)), eps)
        H.up[k] = up
        H.lo[k] = (up[1], up[0])


def _add_lowrank_rec(H, i, U, V, eps):
    """add_lowrank_rec (hodlr.hpp:370-397); U, V hold the block-local rows of node i."""
    t = H.tree
    if U.shape[1] == 0:
        return
    if t.leaf(i):
        H.dense[i] = H.dense[i] + U @ V.T
        return
    s1 = t.size[t.left[i]]
    H.up[i] = truncate(*lr_concat(H.up[i], (U[:s1], V[s1:])), eps)
    H.lo[i] = truncate(*lr_concat(H.lo[i], (U[s1:], V[:s1])), eps)
    _add_lowrank_rec(H, t.left[i], U[:s1], V[:s1], eps)
    _add_lowrank_rec(H, t.right[i], U[s1:], V[s1:], eps)


def add_lowrank_into(H, i, B, eps):
    """add_lowrank_into (hodlr.hpp:400-405)"""
    if B[0].shape[1] == 0:
        return
    _add_lowrank_rec(H, i, B[0], B[1], eps)


def _multiply_rec(A, B, C, i, eps):
    """multiply_rec (hodlr.hpp:409-442)"""
    t = A.tree
    if t.leaf(i):
        C.dense[i] = A.dense[i] @ B.dense[i]
        return
    l, r = t.left[i], t.right[i]
    a12, a21, b12, b21 = A.up[i], A.lo[i], B.up[i], B.lo[i]
    s1, s2 = t.size[l], t.size[r]
    _multiply_rec(A, B, C, l, eps)
    add_lowrank_into(C, l, truncate(*lr_multiply(a12, b21), eps), eps)
    _multiply_rec(A, B, C, r, eps)
    add_lowrank_into(C, r, truncate(*lr_multiply(a21, b12), eps), eps)
    t1 = (apply_sub(A, l, b12[0]), b12[1]) if b12[0].shape[1] else _empty(s1, s2)
    t2 = (a12[0], applyT_sub(B, r, a12[1])) if a12[0].shape[1] else _empty(s1, s2)
    C.up[i] = truncate(*lr_concat(t1, t2), eps)
    u1 = (a21[0], applyT_sub(B, l, a21[1])) if a21[0].shape[1] else _empty(s2, s1)
    u2 = (apply_sub(A, r, b21[0]), b21[1]) if b21[0].shape[1] else _empty(s2, s1)
    C.lo[i] = truncate(*lr_concat(u1, u2), eps)


def multiply(A, B, eps):
    """hodlr_multiply (hodlr.hpp:446-451)"""
    C = Hodlr(A.tree)
    _multiply_rec(A, B, C, 0, eps)
    return C


def _solve_WT(W, i, X, base):
    """solve_WT_rec (hodlr.hpp:456-487): X <- W^{-T} X on subtree i (in place)."""
    t = W.tree
    l0 = t.begin[i] - base
    if t.leaf(i):
        R = W.dense[i]
        if np.any(np.diag(R) == 0.0):
            raise SingularMatrixError("hodlr triangular solve: zero diagonal")
        X[l0:l0 + t.size[i]] = sla.solve_triangular(R, X[l0:l0 + t.size[i]], trans='T', lower=False)
        return
    _solve_WT(W, t.left[i], X, base)
    U, V = W.up[i]
    m = t.begin[t.right[i]] - base
    s1, s2 = t.size[t.left[i]], t.size[t.right[i]]
    if U.shape[1]:
        X[m:m + s2] -= V @ (U.T @ X[l0:l0 + s1])
    _solve_WT(W, t.right[i], X, base)


def _solve_W(W, i, X, base):
    """solve_W_rec (hodlr.hpp:490-521): X <- W^{-1} X on subtree i (in place)."""
    t = W.tree
    l0 = t.begin[i] - base
    if t.leaf(i):
        R = W.dense[i]
        if np.any(np.diag(R) == 0.0):
            raise SingularMatrixError("hodlr triangular solve: zero diagonal")
        X[l0:l0 + t.size[i]] = sla.solve_triangular(R, X[l0:l0 + t.size[i]], lower=False)
        return
    _solve_W(W, t.right[i], X, base)
    U, V = W.up[i]
    m = t.begin[t.right[i]] - base
    s1, s2 = t.size[t.left[i]], t.size[t.right[i]]
    if U.shape[1]:
        X[l0:l0 + s1] -= U @ (V.T @ X[m:m + s2])
    _solve_W(W, t.left[i], X, base)


def solve_WT_left(W, i, X):
    """h_solve_WT_left (hodlr.hpp:527-530)"""
    X = X.copy()
    _solve_WT(W, i, X, W.tree.begin[i])
    return X


def solve_W_left(W, i, X):
    """h_solve_W_left (hodlr.hpp:533-536)"""
    X = X.copy()
    _solve_W(W, i, X, W.tree.begin[i])
    return X


def _cholesky_rec(M, W, i, eps):
    """cholesky_rec (hodlr.hpp:540-563)"""
    t = M.tree
    if t.leaf(i):
        try:
            L = np.linalg.cholesky(np.tril(M.dense[i]))  # reads the lower triangle only
        except np.linalg.LinAlgError as e:
            raise NotPositiveDefiniteError("hodlr_cholesky: leaf factorization failed") from e
        W.dense[i] = L.T.copy()
        return
    l, r = t.left[i], t.right[i]
    _cholesky_rec(M, W, l, eps)
    m12 = M.up[i]
    b12 = (solve_WT_left(W, l, m12[0]), m12[1]) if m12[0].shape[1] else _empty(t.size[l], t.size[r])
    b12 = truncate(*b12, eps)
    if b12[0].shape[1]:
        G = -(b12[0].T @ b12[0])
        add_lowrank_into(M, r, (b12[1] @ G, b12[1]), eps)
    W.up[i] = b12
    _cholesky_rec(M, W, r, eps)


def cholesky(M, eps):
    """hodlr_cholesky (hodlr.hpp:569-574)"""
    work = M.copy()
    W = Hodlr(M.tree)
    _cholesky_rec(work, W, 0, eps)
    return W


def _solve_ur(B, W, Y, i, eps):
    """solve_ur_rec (hodlr.hpp:579-604): Y W = B"""
    t = B.tree
    if t.leaf(i):
        R = W.dense[i]
        if np.any(np.diag(R) == 0.0):
            raise SingularMatrixError("solve_right_upper: zero diagonal")
        Y.dense[i] = sla.solve_triangular(R, B.dense[i].T, trans='T', lower=False).T
        return
    l, r = t.left[i], t.right[i]
    s1, s2 = t.size[l], t.size[r]
    c12 = W.up[i]
    _solve_ur(B, W, Y, l, eps)
    b21 = B.lo[i]
    Y.lo[i] = (b21[0], solve_WT_left(W, l, b21[1])) if b21[0].shape[1] else _empty(s2, s1)
    tt = (apply_sub(Y, l, c12[0]), c12[1]) if c12[0].shape[1] else _empty(s1, s2)
    rhs = truncate(*lr_concat(B.up[i], (-tt[0], tt[1])), eps)
    Y.up[i] = (rhs[0], solve_WT_left(W, r, rhs[1])) if rhs[0].shape[1] else _empty(s1, s2)
    if Y.lo[i][0].shape[1] and c12[0].shape[1]:
        q = truncate(*lr_multiply(Y.lo[i], c12), eps)
        add_lowrank_into(B, r, (-q[0], q[1]), eps)
    _solve_ur(B, W, Y, r, eps)


def _solve_urt(B, W, Y, i, eps):
    """solve_urt_rec (hodlr.hpp:607-636): Y W^T = B"""
    t = B.tree
    if t.leaf(i):
        R = W.dense[i]
        if np.any(np.diag(R) == 0.0):
            raise SingularMatrixError("solve_right_upperT: zero diagonal")
        Y.dense[i] = sla.solve_triangular(R, B.dense[i].T, lower=False).T
        return
    l, r = t.left[i], t.right[i]
    s1, s2 = t.size[l], t.size[r]
    c12 = W.up[i]
    b12 = B.up[i]
    Y.up[i] = (b12[0], solve_W_left(W, r, b12[1])) if b12[0].shape[1] else _empty(s1, s2)
    _solve_urt(B, W, Y, r, eps)
    if Y.up[i][0].shape[1] and c12[0].shape[1]:
        q = truncate(*lr_multiply(Y.up[i], (c12[1], c12[0])), eps)
        add_lowrank_into(B, l, (-q[0], q[1]), eps)
    _solve_urt(B, W, Y, l, eps)
    tt = (apply_sub(Y, r, c12[1]), c12[0]) if c12[0].shape[1] else _empty(s2, s1)
    rhs = truncate(*lr_concat(B.lo[i], (-tt[0], tt[1])), eps)
    Y.lo[i] = (rhs[0], solve_W_left(W, l, rhs[1])) if rhs[0].shape[1] else _empty(s2, s1)


def solve_upper_right(B, W, eps):
    """solve_upper_right (hodlr.hpp:641-647)"""
    work = B.copy()
    Y = Hodlr(B.tree)
    _solve_ur(work, W, Y, 0, eps)
    return Y


def solve_upperT_right(B, W, eps):
    """solve_upperT_right (hodlr.hpp:650-656)"""
    work = B.copy()
    Y = Hodlr(B.tree)
    _solve_urt(work, W, Y, 0, eps)
    return Y


def trace(H):
    """hodlr_trace (hodlr.hpp:658-663)"""
    return float(sum(np.trace(D) for D in H.dense.values()))


def diagnostics(H):
    """diagnostics (hodlr.hpp:679-695): (max off-diagonal rank, memory bytes)"""
    mx, ent = 0, 0
    for D in H.dense.values():
        ent += D.size
    for k in H.up:
        for (U, V) in (H.up[k], H.lo[k]):
            mx = max(mx, U.shape[1])
            ent += U.shape[1] * (U.shape[0] + V.shape[0])
    return mx, ent * 8


# ----------------------------------------------------------------- first iterate
def _compress_dense(M, tree, tol=0.0):
    """Exact HODLR of a dense matrix whose off-diagonal blocks are exactly low
    rank (Q1/Q2 of the stacked QR: ranks <= 2b by the theorems at PAPER.md:998-1033)."""
    H = Hodlr(tree)
    t = tree
    for i in range(len(t)):
        bg, sz = t.begin[i], t.size[i]
        if t.leaf(i):
            H.dense[i] = M[bg:bg + sz, bg:bg + sz].copy()
            continue
        mid = t.begin[t.right[i]]
        s2 = t.size[t.right[i]]
        for which, blk in (("up", M[bg:mid, mid:mid + s2]), ("lo", M[mid:mid + s2, bg:mid])):
            X, s, Yt = np.linalg.svd(blk, full_matrices=False)
            k = int(np.sum(s > tol * max(1.0, s[0] if s.size else 0.0)))
            getattr(H, which)[i] = (X[:, :k] * s[:k], Yt[:k].T)
    return H


def first_iterate_m(bands_scaled, tree, eps):
    """fast_stacked_qr + q1q2t (fast_qr.hpp:509-533) restated densely for small n:
    Q = qr([cA; I]) (the same factorisation reduce_banded computes with Givens,
    fast_qr.hpp:83-172), Q1/Q2 compressed exactly, then M = sym(Q1 *_H Q2^T)."""
    n = len(bands_scaled[0])
    S = np.vstack([banded_to_dense(bands_scaled), np.eye(n)])
    Q, _ = np.linalg.qr(S)
    q1 = _compress_dense(Q[:n], tree, 1e-14)
    q2 = _compress_dense(Q[n:], tree, 1e-14)
    M = multiply(q1, transpose(q2), eps)
    symmetrize(M, eps)
    return M


# --------------------------------------------------------------------- driver
def qdwh_params(l):
    """qdwh_params (qdwh.hpp:27-35)"""
    if not (l > 0.0) or l > 1.0:
        raise ValueError("qdwh_params: l must lie in (0, 1]")
    l2 = l * l
    gamma = np.cbrt(4.0 * (1.0 - l2) / (l2 * l2))
    sq = np.sqrt(1.0 + gamma)
    a = sq + 0.5 * np.sqrt(8.0 - 4.0 * gamma + 8.0 * (2.0 - l2) / (l2 * sq))
    b = 0.25 * (a - 1.0) ** 2
    return a, b, a + b - 1.0


def l_update(l, a, b, c):
    """l_update (qdwh.hpp:38-40)"""
    return l * (a + b * l * l) / (1.0 + c * l * l)


def hqdwh(bands, n_min, eps, delta, alpha, l0):
    """hqdwh (qdwh.hpp:196-241) with alpha / l0 supplied (computed by the C
    restatement of estimates.hpp, oracle/restate.c).  Returns (P, U, iters, diag)."""
    n = len(bands[0])
    l = min(l0, 1.0 - 1e-12)
    tree = Tree(n, n_min)
    X = from_banded([d / alpha for d in bands], tree)
    k, diag = 0, []
    while abs(1.0 - l) > delta and k < 60:
        a, b, c = qdwh_params(l)
        if k == 0:
            sc = np.sqrt(c)
            M = first_iterate_m([d * (sc / alpha) for d in bands], tree, eps)
            X = axpby(b / c, X, (a - b / c) / sc, M, eps)
        else:
            Z = multiply(X, X, eps)
            scale(Z, c)
            add_scaled_identity(Z, 1.0)
            W = cholesky(Z, eps)
            Y = solve_upper_right(X, W, eps)
            V = solve_upperT_right(Y, W, eps)
            X = axpby(b / c, X, a - b / c, V, eps)
        symmetrize(X, eps)
        l = l_update(l, a, b, c)
        k += 1
        diag.append((k, l, c, diagnostics(X)[0]))
    P = X.copy()
    scale(P, -0.5)
    add_scaled_identity(P, 0.5)
    return P, X, k, diag
