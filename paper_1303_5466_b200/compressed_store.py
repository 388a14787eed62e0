"""1-D HSS storage of a factored level's large blocks (compressed path).

The reference's compressed solver keeps, for every box with more than `k_cut`
skeleton points, F^-1 (as Finv_rs / F_sr / F_rs_off / Sinv) and the reduced
operator E in 1-D HSS form over the box's [skeleton ring | residual interface]
ordering, and applies  phi = F^-1 u,  ups = E ([I T_up] phi),
nu = u - [I; T_dn^T](ups - E phi_dn)  through them (`solver_compressed.py:
109-139,313-424`, `hss1d/`): that is what makes its memory O(N).

Here the blocks of a level are formed densely on the device (batched
Gauss-Jordan / GEMMs) and then compressed for storage, one batch per level
(hss1d.Hss1dBatch):

* F^-1 permuted to [sk, rs] with the tree's root cut at |sk| -- the root's
  sibling blocks are the reference's low-rank F_sr / F_rs_off, its two
  subtrees the HSS forms of the skeleton and residual diagonal blocks;
* E over the skeleton ring.

The level then drops the dense F^-1, E and the products W = F^-1 L, C = E R the
dense sweeps use (3.06 m^2 doubles per box at k = 0.75 m) and the sweeps apply
the reference's formulas with T_up / T_dn kept dense (k x r).  Boxes too small
for the forms to pay (HSS_MIN_SIZE) keep F^-1 and E as dense blocks but drop
W and C the same way ("lean", 1.6 m^2 doubles per box).  Only levels of
the a-priori (finite k_cut) path qualify: their work ordering is geometric
(ring walk, then the children's interface), row and column skeletons
coincide, and every box of a level has the same m and k.
"""

import numpy as np
import torch

from . import _lib
from .hss1d import Hss1dBatch, _mm

_F64 = torch.float64


def level_dense_bytes(L):
    m, k = int(L.mmax), int(L.kmax)
    return L.nb * (m * m + k * k + 2 * k * m) * 8


# boxes smaller than this keep dense F^-1 / E (at eps = 1e-10 the HSS ranks of a
# box's blocks are 100-300: below m ~ 1200 the forms are larger than the blocks)
HSS_MIN_SIZE = 1200


def compact_level(H, L, eps=None, leaf_size=None, min_size=None, force_hss=False):
    """Replace level L's dense F^-1 / C / E / W by F^-1 (rows in perm_c order,
    columns in perm_r order: [sk, rs] on both sides) and E alone -- in 1-D HSS
    form when that is smaller (a-priori levels whose boxes have at least
    `min_size` points are tried), else as dense blocks ("lean": the products
    W = F^-1 L and C = E R are not stored either way; the sweeps apply
    T_up / T_dn).  Returns "hss", "lean" or None (the level does not qualify).
    `force_hss` (tests): the HSS form whatever its size.  Lean storage also
    serves the ID path (k_cut = None: pivot-ordered skeletons, ranks that vary
    from box to box); the HSS forms need the a-priori path's geometric
    ordering and uniform ranks."""
    if (L.lv == 0 or getattr(L, "hss", None)
            or getattr(L, "ti", False) or getattr(L, "refine", False) or getattr(L, "rb", None)
            or getattr(L, "Finv", None) is None or not L.Finv.is_cuda
            or getattr(L, "virtual", False)):
        return None
    m = np.asarray(L.m)
    k = np.asarray(L.k)
    n = int(L.mmax)
    if (k >= m).all() or int(L.kmax) <= (H.opts.k_cut or 0):
        return None
    eps = float(H.eps if eps is None else eps)
    leaf = int(leaf_size or H.opts.inner_leaf_size)
    min_size = HSS_MIN_SIZE if min_size is None else min_size
    dev = H.device
    nb = L.nb
    # boxes smaller than the level's largest are identity-padded (as F^-1 is):
    # pad positions map to themselves
    jj = torch.arange(n, device=dev)[None, :]
    live = jj < L.m_d.long()[:, None]
    pr = torch.where(live, L.perm_r.long()[:, :n], jj)
    pc = pr if L.perm_c is L.perm_r else torch.where(live, L.perm_c.long()[:, :n], jj)
    bidx = torch.arange(nb, device=dev)[:, None, None]
    Fp = L.Finv[bidx, pr[:, :, None], pc[:, None, :]]     # F^-1(perm_c[r'], perm_r[c'])
    big = L.Finv.numel() * 8 > (1 << 30)
    L.Finv = L.C = L.W = None
    if big and torch.cuda.mem_get_info()[0] < 0.35 * torch.cuda.mem_get_info()[1]:
        torch.cuda.empty_cache()   # the HSS compression's workspace comes from the library's pool
    kind = "lean"
    hF = hE = None
    k0 = int(k[0])
    geometric = (bool(getattr(H, "apriori", None)) and L.perm_c is L.perm_r
                 and bool((k == k0).all()) and bool((m == n).all()))
    if geometric and k0 == L.kmax and 0 < k0 < n and (n >= min_size or force_hss):
        hF = Hss1dBatch.compress(Fp, n, eps, leaf_size=leaf, align=k0, seed=H.opts.seed + 17 * L.lv)
        hE = Hss1dBatch.compress(L.E, k0, eps, leaf_size=leaf, seed=H.opts.seed + 17 * L.lv + 1)
        if force_hss or hF.nbytes() + hE.nbytes() < nb * (n * n + k0 * k0) * 8:
            kind = "hss"
    if kind == "lean":
        hF, hE = Hss1dBatch.from_dense(Fp, n), Hss1dBatch.from_dense(L.E, int(L.kmax))
    L.hss = (hF, hE)
    L.hss_kind = kind
    L.E = None
    # per-box offsets of the residual part (ranks may vary from box to box)
    L.hss_koff = np.arange(nb, dtype=np.int64) * n + k.astype(np.int64)
    return kind


def compact(inv, eps=None, leaf_size=None, min_size=None, force_hss=False):
    """Convert every qualifying level of a factored DenseBlockInverse, leaves
    first; returns the number of levels stored in 1-D HSS form (the other
    qualifying levels are "lean" dense)."""
    H = inv.H
    done = 0
    for L in reversed([x for x in H.levels if x is not None and not getattr(x, "virtual", False)]):
        if compact_level(H, L, eps, leaf_size, min_size, force_hss) == "hss":
            done += 1
        torch.cuda.empty_cache()
    return done


def hss_bytes(L):
    hF, hE = L.hss
    return hF.nbytes() + hE.nbytes()


# -- sweeps of a compacted level (called from solver_dense) --------------------

def sweep_up_level(H, L, U, phi, ups, r):
    """phi = F^-1 u (kept in [sk, rs] order for the down sweep),
    ups = E ([I T_up] phi)  (solver_compressed.py:186-199)."""
    from .solver_dense import _ptrs
    hF, hE = L.hss
    dev = H.device
    nb, n, kk = L.nb, L.mmax, L.kmax
    ld = nb * n
    Up = torch.zeros((r, ld), dtype=_F64, device=dev)
    _lib.gather_rows(U, n, ld, L.perm_r, n, Up, n, ld, L.m_d, n, None, r, nb)
    Pp = hF.matvec(Up)
    del Up
    phi[("p", L.lv)] = Pp
    phi[L.lv] = None
    R = torch.zeros((r, nb * kk), dtype=_F64, device=dev)
    _lib.copy2d(Pp, n, ld, R, kk, nb * kk, L.k_d, kk, None, r, nb)
    # + T_up phi_rs  (T stored k x (n - k) column-major, ld kmax)
    _mm(L.Tc, L.ntmax * kk, kk, 0, None, 0, ld, R, kk, nb * kk, kk, L.ntmax, nb, r, 1.0, 1.0,
        Mb=L.k_d, Kb=L.nT_d, xptr=_ptrs(Pp, L.hss_koff, dev))
    ups[L.lv] = hE.matvec(R)


def sweep_down_level(H, L, PD, phi, ups, r):
    """res = phi - F^-1 [I; T_dn^T] (ups - E phi_dn)  (solver_compressed.py:
    200-215), returned in the level's work order."""
    from .solver_dense import _ptrs
    hF, hE = L.hss
    dev = H.device
    nb, n, kk = L.nb, L.mmax, L.kmax
    ld = nb * n
    Ups = ups[L.lv]
    hE.matvec(PD, Ups, alpha=-1.0, beta=1.0)
    Z = torch.zeros((r, ld), dtype=_F64, device=dev)
    _lib.copy2d(Ups, kk, nb * kk, Z, n, ld, L.k_d, kk, None, r, nb)
    _mm(L.Tr, L.ntmax * kk, kk, 1, Ups, kk, nb * kk, None, 0, ld, L.ntmax, kk, nb, r,
        Mb=L.nT_d, Kb=L.k_d, yptr=_ptrs(Z, L.hss_koff, dev))
    Pp = phi.pop(("p", L.lv))
    hF.matvec(Z, Pp, alpha=-1.0, beta=1.0)
    del Z
    Phi = torch.zeros((r, ld), dtype=_F64, device=dev)
    _lib.scatter_rows(Pp, n, ld, L.perm_c, n, Phi, n, ld, L.m_d, n, None, r, nb)
    phi[L.lv] = Phi
    return Phi
