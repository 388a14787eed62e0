"""Dense core on the B200: interpolative decomposition and checked inversion.

Single-matrix front ends of the batched K2/K3 kernels, mirroring the
reference's dense_core.py (IdFactor 31-64, interp_decomp 67-100,
lu_factor_checked 222-230, dense_solve 233-240).  The randomized-ID and
low-rank algebra of the O(N) path (dense_core.py:108-216) is out of scope.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import NumericalError, SingularFactorError


class IdFactor:
    """Column ID  A ~= A[:, skeleton] @ [I T] Pi  (dense_core.py:31-64)."""

    def __init__(self, skeleton, T, perm, achieved_error=0.0):
        self.skeleton = np.asarray(skeleton, dtype=np.int64)
        self.T = T
        self.perm = np.asarray(perm, dtype=np.int64)
        self.achieved_error = float(achieved_error)

    @property
    def rank(self):
        return self.skeleton.size

    @property
    def ncols(self):
        return self.perm.size

    def right_matrix(self, dtype=None):
        k, n = self.rank, self.ncols
        dtype = dtype or (self.T.dtype if self.T.size else np.float64)
        r = np.zeros((k, n), dtype=dtype)
        r[np.arange(k), self.perm[:k]] = 1.0
        if n > k:
            r[:, self.perm[k:]] = self.T
        return r

    def interp_rows(self, dtype=None):
        return self.right_matrix(dtype).T


def interp_decomp_batched(mats, eps, group=1, force_blocked=False, seed=0, kfix=None,
                          pairs=False):
    """IDs of a list of real matrices in one K2 launch sequence.  Matrices in
    consecutive groups of `group` share a rank (max over the group), as the
    row/column IDs of one box do in compress_outer.  `kfix` (one rank per
    matrix) turns pivoting off: T is then the least-squares solution of
    A[:, :k] T = A[:, k:] (the compressed path's interpolation).  `pairs`:
    columns (2t, 2t+1) are the two real components of one complex unknown
    (pivoted pairwise, even ranks).  Returns [(perm, k, T), ...]."""
    _lib.require_cuda()
    dev = torch.device("cuda")
    count = len(mats)
    ps = np.array([a.shape[0] for a in mats], dtype=np.int32)
    ms = np.array([a.shape[1] for a in mats], dtype=np.int32)
    kf = None
    if kfix is not None:
        kf = np.asarray(kfix, dtype=np.int32)
        if (kf < 0).any() or (kf > np.minimum(ps, ms)).any():
            raise ValueError("kfix must lie in [0, min(p, m)]")
        ps = np.maximum(ps, np.minimum(ms, -(-kf // 32) * 32)).astype(np.int32)  # zero rows
    maxp, maxm = max(int(ps.max()), 1), max(int(ms.max()), 1)
    ldA = maxp + (maxp & 1)
    A = torch.zeros((count, maxm, ldA), dtype=torch.float64, device=dev)
    for i, a in enumerate(mats):
        if a.size:
            A[i, :a.shape[1], :a.shape[0]] = torch.from_numpy(np.ascontiguousarray(a.T, dtype=np.float64))
    pv = torch.as_tensor(ps, device=dev)
    mv = torch.as_tensor(ms, device=dev)
    rank = torch.zeros(count, dtype=torch.int32, device=dev)
    perm = torch.zeros((count, maxm), dtype=torch.int32, device=dev)
    T = torch.zeros((count, maxm, maxm), dtype=torch.float64, device=dev)
    kd = None if kf is None else torch.as_tensor(kf, device=dev)
    d = _lib.IdDesc(_lib.ptr(A), maxm * ldA, ldA, _lib.ptr(pv), _lib.ptr(mv), maxp, maxm, count,
                    group, float(eps), _lib.ptr(rank), _lib.ptr(perm), _lib.ptr(T), maxm * maxm,
                    maxm, int(seed), int(force_blocked), None if kd is None else _lib.ptr(kd),
                    int(pairs))
    _lib.call("vief_id_batched", ctypes.byref(d), _lib.stream_handle())
    rank = rank.cpu().numpy()
    perm = perm.cpu().numpy()
    T = T.cpu().numpy()
    out = []
    for i in range(count):
        k, m = int(rank[i]), int(ms[i])
        out.append((perm[i, :m].astype(np.int64), k, T[i, :m - k, :k].T.copy()))
    return out


def _realify_cols(A):
    """Complex p x n -> real 2p x 2n whose columns (2j, 2j+1) represent
    column j acting on Re / Im of the unknown: [Re a; Im a], [-Im a; Re a]."""
    p, n = A.shape
    R = np.empty((2 * p, 2 * n))
    R[:p, 0::2], R[p:, 0::2] = A.real, A.imag
    R[:p, 1::2], R[p:, 1::2] = -A.imag, A.real
    return R


def _id_real(A, eps, min_rank, max_rank, force_blocked, pairs):
    """(perm, k, T) of a real A with the rank clamps; a clamped rank re-solves
    T = R11^{-1} R12 for the same pivot order on the device (fixed-rank mode)."""
    m, n = A.shape
    perm, k, T = interp_decomp_batched([A], eps, force_blocked=force_blocked, pairs=pairs)[0]
    unit = 2 if pairs else 1
    k2 = max(k, min(unit * min_rank, m, n))
    if max_rank is not None:
        k2 = min(k2, unit * max_rank)
    if k2 != k:
        k = k2
        if k == 0 or k >= n:
            T = np.zeros((k, n - k), A.dtype)
        else:  # same pivots, no pivoting, rank k
            _, _, T = interp_decomp_batched([np.ascontiguousarray(A[:, perm])], eps,
                                            force_blocked=True, kfix=[k])[0]
    return perm, k, T


def interp_decomp(A, eps, min_rank=0, max_rank=None, eps_abs=None, force_blocked=False):
    """Column ID by pivoted QR (dense_core.py:67-100): rank = first j with
    |R_jj| <= eps |R_00| (residual form on the blocked path), then the
    min_rank / max_rank clamps; T = R11^{-1} R12.  Complex A runs realified
    with pairwise pivoting (each complex column is a pair of real columns), so
    the skeleton is a set of complex columns and T the complex interpolation.
    `eps_abs` (dense_core.py:86-88): absolute floor of the rank threshold."""
    A = np.asarray(A)
    m, n = A.shape
    if n == 0 or m == 0:
        return IdFactor(np.zeros(0, np.int64), np.zeros((0, n), A.dtype), np.arange(n), 0.0)
    if eps_abs:
        # |R_jj| <= max(eps |R_00|, eps_abs) with |R_00| = the largest column norm
        # (the first pivot): one relative threshold for the device kernel
        r00 = float(np.sqrt((np.abs(A) ** 2).sum(axis=0).max()))
        if r00 > 0.0:
            eps = max(float(eps), min(float(eps_abs) / r00, 1.0))
    if np.iscomplexobj(A):
        perm2, k2, T2 = _id_real(_realify_cols(A), eps, min_rank, max_rank, force_blocked, True)
        k = k2 // 2
        sk = perm2[:k2:2] // 2                    # pivots come in (Re, Im) pairs
        rest = perm2[k2:] // 2
        _, first = np.unique(rest, return_index=True)
        rest = rest[np.sort(first)]               # the remaining complex columns
        perm = np.concatenate([sk, rest]).astype(np.int64)
        pos = np.empty(2 * n, np.int64)
        pos[perm2] = np.arange(2 * n)
        # realified T: rows = skeleton real columns, columns = the others; the
        # (Re, Im) block of t is [[Re t, -Im t], [Im t, Re t]] (realify_cols)
        T = (T2[np.ix_(pos[2 * sk], pos[2 * rest] - k2)]
             + 1j * T2[np.ix_(pos[2 * sk + 1], pos[2 * rest] - k2)]) if k and n > k else \
            np.zeros((k, n - k), np.complex128)
    else:
        perm, k, T = _id_real(A, eps, min_rank, max_rank, force_blocked, False)
    if k == 0:
        return IdFactor(np.zeros(0, np.int64), np.zeros((0, n), A.dtype), perm, 0.0)
    return IdFactor(perm[:k], T if k < n else np.zeros((k, 0), A.dtype), perm)


def row_id(A, eps, min_rank=0, max_rank=None):
    return interp_decomp(A.T, eps, min_rank=min_rank, max_rank=max_rank)


class InverseFactor:
    """Explicit inverse of a square matrix computed on the B200 (the K3
    Gauss-Jordan kernel); stands where the reference keeps LU factors."""

    def __init__(self, inv):
        self.inv = inv

    def solve(self, B):
        return self.inv @ B


def lu_factor_checked(A, where="dense block"):
    """Partial-pivoting factorization with the reference's singularity test
    (dense_core.py:222-230); returns an InverseFactor."""
    _lib.require_cuda()
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    if A.shape != (n, n):
        raise NumericalError("square matrix required")
    X = torch.from_numpy(np.ascontiguousarray(A.T)).to("cuda")
    pmin, pmax = _lib.inv_batched(X, n * n, n, n, 1)
    lo, hi = float(pmin[0]), float(pmax[0])
    if n and (hi == 0.0 or lo <= 1e-300 or lo / hi < np.finfo(float).eps ** 2 or not np.isfinite(lo)):
        raise SingularFactorError(where, lo)
    return InverseFactor(X.cpu().numpy().T.copy())


def dense_solve(A, B):
    A = np.asarray(A)
    B = np.asarray(B)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise NumericalError("dense_solve requires a square matrix")
    return lu_factor_checked(A).solve(B)
