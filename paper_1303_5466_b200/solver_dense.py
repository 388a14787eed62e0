"""Dense-block recursive skeletonization (HSS-D) on the B200.

Drop-in for the reference's solver_dense.py (compress_outer 234-272,
invert_dense_block 332-368, DenseBlockInverse.apply 293-329, Hss2dMatrix
.matvec 143-178).  The reference walks boxes one by one; here every level is
one batch ("boxes within a level are independent"):

  compress_outer, per level fine -> coarse
     work rows/cols  leaf: owned points; else children's skeletons concatenated
     D (leaf) or B12/B21 (siblings)              K1  vief_gen_block
     proxy ring + near field sources             K1  vief_box_sources
     ID matrices (row block^T, column block)     K1  vief_gen_idmat
     pivoted-QR IDs, ranks coupled per box       K2  vief_id_batched
  invert_dense_block, per level fine -> coarse
     F = D | [[E1, B12], [B21, E2]]  -> F^{-1}   K3  vief_inv_batched (Gauss-Jordan, partial pivoting)
     W = F^{-1} L,  G = R W,  E = G^{-1},  C = E R   gathers + DMMA GEMMs
  apply (solve), per level
     up:   phi = F^{-1} u ;  ups = C phi            (= E R F^{-1} u, solver_dense.py:309-310)
     down: res = phi - W (ups - E phi_dn)           (= F^{-1}(u - L ups + L E phi_dn), 317-321)

The down-pass identity  F^{-1}(u - L(ups - E phi_dn)) = phi - W (ups - E phi_dn)
uses W = F^{-1} L from the factorization, so the down sweep reads W (m x k)
instead of F (m x m).  All per-box blocks of a level live in one padded HBM
buffer (column-major, leading dimension = level maximum).
"""

import contextlib
import ctypes
import gc
import math

import numpy as np
import torch

from . import _lib
from .config import SolverOptions
from .errors import ConfigError, SingularFactorError
from .kernels import PLAIN, get_assembler
from .tree import proxy_count_v, near_count, proxy_count

_I32 = torch.int32
_F64 = torch.float64


class StageTimer:
    """Optional per-(stage, level) CUDA-event timing of the factor/solve
    sweeps (set solver_dense.TIMER = StageTimer() to enable)."""

    def __init__(self):
        self.events = []

    def mark(self, tag):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.append((tag, e))

    def report(self):
        torch.cuda.synchronize()
        out = []
        for (t0, e0), (t1, e1) in zip(self.events, self.events[1:]):
            out.append((t1, e0.elapsed_time(e1)))
        return out


TIMER = None


def _mark(tag):
    if TIMER is not None:
        TIMER.mark(tag)


def _even(x):
    return int(x) + (int(x) & 1)


def _h2d(a, device):
    """Host array -> device tensor through pinned memory, asynchronously on the
    current stream (a pageable copy would block the host until the stream
    drains, serialising the two streams of `factorize`)."""
    t = torch.from_numpy(a)
    if torch.device(device).type != "cuda":
        return t.to(device)
    return t.pin_memory().to(device, non_blocking=True)


def _dev_i32(a, device):
    return _h2d(np.ascontiguousarray(a, dtype=np.int32), device)


def _ptrs(base, offsets_elems, device):
    """Device int64 array of base.data_ptr() + 8*offset (pointer arrays)."""
    off = np.asarray(offsets_elems, dtype=np.int64) * base.element_size() + base.data_ptr()
    return _h2d(np.ascontiguousarray(off), device)


class _Level:
    """Device state of one tree level (all its boxes as one batch)."""

    def __init__(self, lv, ids, rects, leaf):
        self.lv = lv
        self.ids = np.asarray(ids)
        self.rects = np.asarray(rects, dtype=np.int64)
        self.nb = len(ids)
        self.leaf = leaf


class FactoredInterp:
    """Host view of one box's interpolation operator (perm, T)
    (solver_dense.py:58-95): R = [I T] Pi, L = Pi^T [I; T^T]."""

    def __init__(self, perm, T):
        self.perm = np.asarray(perm, dtype=np.int64)
        self.T = T
        self.k = T.shape[0]
        self.m = self.perm.size

    def apply_R(self, x):
        return x[self.perm[:self.k]] + self.T @ x[self.perm[self.k:]]

    def apply_L(self, w):
        out = np.empty((self.m,) + w.shape[1:], dtype=np.result_type(self.T.dtype, w.dtype))
        out[self.perm[:self.k]] = w
        out[self.perm[self.k:]] = self.T.T @ w
        return out

    def dense_L(self, dtype):
        out = np.zeros((self.m, self.k), dtype=dtype)
        out[self.perm[:self.k], np.arange(self.k)] = 1.0
        out[self.perm[self.k:]] = self.T.T
        return out

    def dense_R(self, dtype):
        return self.dense_L(dtype).T.copy()

    def nbytes(self):
        return self.T.nbytes


class _BoxView:
    """Read-only dict-like access {box idx: host array} over level buffers."""

    def __init__(self, owner, getter, keys):
        self._owner, self._get, self._keys = owner, getter, keys

    def __getitem__(self, i):
        if i not in self._keys():
            raise KeyError(i)
        return self._get(i)

    def __contains__(self, i):
        return i in self._keys()

    def get(self, i, default=None):
        return self[i] if i in self else default

    def keys(self):
        return list(self._keys())

    def __iter__(self):
        return iter(self.keys())

    def __len__(self):
        return len(self._keys())

    def items(self):
        return [(i, self[i]) for i in self.keys()]

    def values(self):
        return [self[i] for i in self.keys()]


class Hss2dMatrix:
    """Outer skeleton compression of the system matrix, resident in HBM
    (solver_dense.py:98-231)."""

    def __init__(self, spec, grid, tree, eps, opts, quad=PLAIN, level_slices=None):
        """`level_slices` (sharded use, distributed.py): {level: (lo, hi)} box
        ranges this object factors; other levels are absent (None)."""
        _lib.require_cuda()
        self.spec, self.grid, self.tree = spec, grid, tree
        self.eps, self.opts, self.quad = eps, opts, quad
        self.asm = get_assembler(spec, grid, quad)
        self.device = self.asm.device
        # complex (helmholtz2d) systems are factored in realified form: every
        # point carries two real unknowns (Re, Im) and each complex entry the
        # real block [[Re, -Im], [Im, Re]]; the hierarchy, skeletonization and
        # all kernels are the real ones.  Complex symmetry is not real symmetry,
        # so row and column IDs are both computed.
        self.realified = bool(spec.is_complex)
        self.problem = _lib.Problem.from_buffer_copy(self.asm.problem)
        self.problem.realify = int(self.realified)
        self.symmetric = spec.symmetric and not self.realified
        self.group = 1 if self.symmetric else 2
        self.levels = []
        for lv in range(tree.depth + 1):
            sl = (0, len(tree.ids[lv])) if level_slices is None else level_slices.get(lv)
            if sl is None:
                self.levels.append(None)
                continue
            L = _Level(lv, tree.ids[lv][sl[0]:sl[1]], tree.rects[lv][sl[0]:sl[1]],
                       lv == tree.depth)
            L.sl = sl
            self.levels.append(L)
        self.sharded = level_slices is not None
        self._lvl_of_cache = None
        self._interp_cache = {}

    # dict-like host views (created on access: a stored view would close a
    # reference cycle through its getter and keep the HBM buffers alive until
    # the cyclic GC runs)
    def _nonroot(self):
        return [i for i in self._lvl_of if i != 0]

    def _nonleaf(self):
        return [i for i in self._lvl_of if not self._lvl_of[i][0].leaf]

    def _leaves(self):
        return [i for i in self._lvl_of if self._lvl_of[i][0].leaf]

    @property
    def row_skel(self):
        return _BoxView(self, lambda i: self._skel(i, "rskel"), self._nonroot)

    @property
    def col_skel(self):
        return _BoxView(self, lambda i: self._skel(i, "cskel"), self._nonroot)

    @property
    def Lfac(self):
        return _BoxView(self, lambda i: self._interp(i, "row"), self._nonroot)

    @property
    def Rfac(self):
        return _BoxView(self, lambda i: self._interp(i, "col"), self._nonroot)

    @property
    def D(self):
        return _BoxView(self, self._dblock, self._leaves)

    @property
    def B(self):
        return _BoxView(self, self._bblock, self._nonleaf)

    @property
    def _lvl_of(self):
        """box id -> (level, index in level); built on first use (host views)."""
        if self._lvl_of_cache is None:
            d = {}
            for L in self.levels:
                if L is None:
                    continue
                for j, i in enumerate(L.ids.tolist()):
                    d[i] = (L, j)
            self._lvl_of_cache = d
        return self._lvl_of_cache

    @property
    def n(self):
        return self.grid.n

    # -- host views ---------------------------------------------------------
    def _skel(self, i, which):
        L, j = self._lvl_of[i]
        k = int(L.k[j])
        return getattr(L, which)[j, :k].cpu().numpy().astype(np.int64)

    def _interp(self, i, which):
        key = (i, "row" if (which == "row" or self.symmetric) else "col")
        if key in self._interp_cache:
            return self._interp_cache[key]
        L, j = self._lvl_of[i]
        k, m = int(L.k[j]), int(L.m[j])
        perm = (L.perm_r if key[1] == "row" else L.perm_c)[j, :m].cpu().numpy()
        Tbuf = L.Tr if key[1] == "row" else L.Tc
        T = Tbuf[j, :m - k, :k].cpu().numpy().T.copy()
        f = FactoredInterp(perm, T)
        self._interp_cache[key] = f
        if self.symmetric:
            self._interp_cache[(i, "col")] = f
        return f

    def _dblock(self, i):
        L, j = self._lvl_of[i]
        m = int(L.m[j])
        return L.D[j, :m, :m].t().cpu().numpy()

    def _bblock(self, i):
        L, j = self._lvl_of[i]
        C = self.levels[L.lv + 1]
        k1, k2 = int(C.k[2 * j]), int(C.k[2 * j + 1])
        return (L.B12[j, :k2, :k1].t().cpu().numpy(), L.B21[j, :k1, :k2].t().cpu().numpy())

    def work_rows(self, box):
        if box.is_leaf:
            return self.tree.owned_indices(box)
        c1, c2 = box.children
        return np.concatenate([self.row_skel[c1], self.row_skel[c2]])

    def work_cols(self, box):
        if box.is_leaf:
            return self.tree.owned_indices(box)
        c1, c2 = box.children
        return np.concatenate([self.col_skel[c1], self.col_skel[c2]])

    def nbytes(self):
        """D + B + T bytes of the real entries (solver_dense.py:132-139)."""
        tot = 0
        for L in _real_levels(self):
            if L.leaf:
                tot += int((L.m.astype(np.int64) ** 2).sum()) * 8
            if not L.leaf:
                C = self.levels[L.lv + 1]
                k1, k2 = C.k[0::2].astype(np.int64), C.k[1::2].astype(np.int64)
                tot += int((2 * k1 * k2).sum()) * 8
            if L.lv > 0:
                t = int((L.k.astype(np.int64) * (L.m - L.k)).sum()) * 8
                tot += t * (1 if self.symmetric else 2)
        return tot  # realified complex blocks are counted as the real doubles they occupy

    # -- forward operator ---------------------------------------------------
    def matvec(self, x):
        return _matvec(self, x)

    def save(self, path):
        """Write the compression to `path` (persist.py)."""
        from . import persist
        persist.save(self, path)

    @staticmethod
    def load(path, device=None):
        from . import persist
        return persist.load(path, device)

    def densify(self):
        """Dense reconstruction (tests, small N)."""
        n = self.grid.n
        eye = np.eye(n)
        return self.matvec(eye)


# ---------------------------------------------------------------------------
# compress_outer

def _level_sources(H, L, pad):
    dev = H.device
    w = L.rects[:, 1] - L.rects[:, 0]
    h = L.rects[:, 3] - L.rects[:, 2]
    p = proxy_count_v(w, h, pad)
    p += near_count(L.rects, H.grid.n_side, pad)
    pmax = int(p.max())
    rects = _dev_i32(L.rects, dev)
    src_xy = torch.empty((L.nb, pmax, 2), dtype=_I32, device=dev)
    src_g = torch.empty((L.nb, pmax), dtype=_I32, device=dev)
    p_d = torch.empty(L.nb, dtype=_I32, device=dev)
    _lib.call("vief_box_sources", _lib.ptr(rects), L.nb, pad, H.grid.n_side, _lib.ptr(src_xy),
              _lib.ptr(src_g), pmax, _lib.ptr(p_d), _lib.stream_handle())
    return p.astype(np.int32), pmax, src_xy, src_g


def _compress_level(H, L, pad, seed):
    _compress_level_blocks(H, L)
    _compress_level_id(H, L, pad, seed)


def _compress_level_blocks(H, L):
    """First half of a level's compression: work rows/columns and the D / B
    blocks (all F of this level needs besides the children's E)."""
    dev = H.device
    prob = ctypes.byref(H.problem)
    st = _lib.stream_handle
    nb = L.nb
    _lib.prof_mark("py.rows")
    # work rows / cols
    if L.leaf:
        own = H.tree.owned_level(L.lv)[L.sl[0]:L.sl[1]]
        cnt = (own >= 0).sum(axis=1)          # ragged leaves: valid points first
        own = np.where(own >= 0, own, 0)
        if H.realified:  # unknowns u = 2*point + component, interleaved per point
            own = np.stack([2 * own, 2 * own + 1], axis=-1).reshape(own.shape[0], -1)
            cnt = 2 * cnt
        L.m = cnt.astype(np.int32)
        L.mmax = int(L.m.max())
        L.rows = _dev_i32(own, dev)
        L.cols = L.rows
        L.cat_idx = None
    else:
        C = H.levels[L.lv + 1]
        k1, k2 = C.k[0::2].astype(np.int64), C.k[1::2].astype(np.int64)
        L.m = (k1 + k2).astype(np.int32)
        L.mmax = int(L.m.max())
        t = np.arange(L.mmax)[None, :]
        cat = np.where(t < k1[:, None], t, C.kmax + t - k1[:, None])
        cat = np.where(t < L.m[:, None], cat, 0)
        L.cat_idx = _dev_i32(cat, dev)
        L.rows = torch.zeros((nb, L.mmax), dtype=_I32, device=dev)
        m_d = _dev_i32(L.m, dev)
        _lib.gather_int(C.rskel, 2 * C.kmax, L.cat_idx, L.mmax, L.rows, L.mmax, m_d, L.mmax, nb)
        if H.symmetric:
            L.cols = L.rows
        else:
            L.cols = torch.zeros((nb, L.mmax), dtype=_I32, device=dev)
            _lib.gather_int(C.cskel, 2 * C.kmax, L.cat_idx, L.mmax, L.cols, L.mmax, m_d, L.mmax, nb)
    L.m_d = _dev_i32(L.m, dev)
    _lib.prof_mark("py.entries_DB")
    # leaf D / sibling B blocks (solver_dense.py:243-249)
    if L.leaf:
        L.D = torch.empty((nb, L.mmax, L.mmax), dtype=_F64, device=dev)
        _lib.call("vief_gen_block", prob, _lib.ptr(L.rows), L.mmax, _lib.ptr(L.m_d), L.mmax,
                  _lib.ptr(L.rows), L.mmax, _lib.ptr(L.m_d), L.mmax, _lib.ptr(L.D),
                  L.mmax * L.mmax, None, L.mmax, nb, st())
    else:
        C = H.levels[L.lv + 1]
        kc = C.kmax
        k1d, k2d = C.k_d[0::2].contiguous(), C.k_d[1::2].contiguous()
        L.B12 = torch.zeros((nb, kc, kc), dtype=_F64, device=dev)   # [item, col, row]
        L.B21 = torch.zeros((nb, kc, kc), dtype=_F64, device=dev)
        rs, cs = C.rskel, C.cskel
        _lib.call("vief_gen_block", prob, _lib.ptr(rs), 2 * kc, _lib.ptr(k1d), kc,
                  _lib.ptr(cs) + 4 * kc, 2 * kc, _lib.ptr(k2d), kc, _lib.ptr(L.B12), kc * kc, None,
                  kc, nb, st())
        _lib.call("vief_gen_block", prob, _lib.ptr(rs) + 4 * kc, 2 * kc, _lib.ptr(k2d), kc,
                  _lib.ptr(cs), 2 * kc, _lib.ptr(k1d), kc, _lib.ptr(L.B21), kc * kc, None,
                  kc, nb, st())


def _compress_level_id(H, L, pad, seed):
    """Second half of a level's compression: proxy/near sources, the ID
    matrices, the batched IDs, T and the skeleton lists."""
    dev = H.device
    prob = ctypes.byref(H.problem)
    st = _lib.stream_handle
    nb = L.nb
    if L.lv == 0:
        return
    if getattr(H, "apriori", None):
        return _compress_level_apriori(H, L, H.apriori)
    _lib.prof_mark("py.sources+idmat")
    # proxy + near sources and the ID matrices (solver_dense.py:250-263)
    p, pmax, src_xy, src_g = _level_sources(H, L, pad)
    L.p = p
    if getattr(H, "id_split", None) is not None:
        return _compress_level_id_split(H, L, p, pmax, src_xy, src_g, seed)
    g = H.group
    count = nb * g
    mm = L.mmax
    p_d = _dev_i32(p, dev)
    if H.realified:  # the realified ID matrices have (source, component) rows
        p = 2 * p
    ldA = _even(p.max())
    A = torch.zeros((count, mm, ldA), dtype=_F64, device=dev)
    _lib.call("vief_gen_idmat", prob, 0, _lib.ptr(L.rows), mm, _lib.ptr(L.m_d), mm,
              _lib.ptr(src_xy), _lib.ptr(src_g), pmax, _lib.ptr(p_d), pmax, _lib.ptr(A),
              g * mm * ldA, ldA, nb, st())
    if g == 2:
        _lib.call("vief_gen_idmat", prob, 1, _lib.ptr(L.cols), mm, _lib.ptr(L.m_d), mm,
                  _lib.ptr(src_xy), _lib.ptr(src_g), pmax, _lib.ptr(p_d), pmax,
                  _lib.ptr(A) + 8 * mm * ldA, g * mm * ldA, ldA, nb, st())
    del src_xy, src_g
    pv = _dev_i32(np.repeat(p, g), dev)
    mv = _dev_i32(np.repeat(L.m, g), dev)
    rank = torch.zeros(count, dtype=_I32, device=dev)
    perm = torch.zeros((count, mm), dtype=_I32, device=dev)
    T = torch.zeros((count, mm, mm), dtype=_F64, device=dev)
    _id_batched(dev, A, mm * ldA, ldA, pv, mv, int(p.max()), mm, count, g, float(H.eps), rank,
                perm, T, int(seed) * 1000003 + L.lv, int(getattr(H, "_force_blocked", 0)),
                pairs=H.realified)
    del A
    L.k = rank[0::g].cpu().numpy().astype(np.int32)
    L.kmax = max(int(L.k.max()), 1)
    L.k_d = _dev_i32(L.k, dev)
    nT = L.m - L.k
    L.ntmax = max(int(nT.max()), 1)
    L.nT_d = _dev_i32(nT, dev)
    L.perm_r = perm[0::g].contiguous()
    L.perm_c = perm[1::g].contiguous() if g == 2 else L.perm_r
    _lib.prof_mark("py.T+skel")
    # T compacted to [item, col (m-k), row (k)] with ld = kmax
    L.Tr = torch.zeros((nb, L.ntmax, L.kmax), dtype=_F64, device=dev)
    _lib.copy2d(T, g * mm * mm, mm, L.Tr, L.ntmax * L.kmax, L.kmax, L.k_d, L.kmax, L.nT_d,
                L.ntmax, nb)
    if g == 2:
        L.Tc = torch.zeros_like(L.Tr)
        _lib.copy2d(_lib.ptr(T) + 8 * mm * mm, g * mm * mm, mm, L.Tc, L.ntmax * L.kmax, L.kmax,
                    L.k_d, L.kmax, L.nT_d, L.ntmax, nb)
    else:
        L.Tc = L.Tr
    del T
    # skeletons in pivot order: rows[perm[:k]] (solver_dense.py:270-271)
    L.rskel = torch.zeros((nb, L.kmax), dtype=_I32, device=dev)
    _lib.gather_int(L.rows, mm, L.perm_r, mm, L.rskel, L.kmax, L.k_d, L.kmax, nb)
    if g == 2:
        L.cskel = torch.zeros((nb, L.kmax), dtype=_I32, device=dev)
        _lib.gather_int(L.cols, mm, L.perm_c, mm, L.cskel, L.kmax, L.k_d, L.kmax, nb)
    else:
        L.cskel = L.rskel


def _compress_level_id_split(H, L, p, pmax, src_xy, src_g, seed):
    """One side of a top box's ID pair on this process (distributed.py): the
    row ID (side 0, the box's owner) or the column ID (side 1, a helper rank),
    with the ranks coupled across the two processes by the library's per-block
    callback (the reference's min_rank rule, solver_dense.py:263-266, as in the
    single-process group of two).  Side 1 hands its perm / T to `send`; side 0
    takes the column side's from `recv` and finishes the level as
    _compress_level_id does."""
    side, couple, send, recv = H.id_split
    dev = H.device
    prob = ctypes.byref(H.problem)
    st = _lib.stream_handle
    if L.nb != 1 or H.group != 2:
        raise ValueError("split IDs take one box of a non-symmetric problem")
    mm = L.mmax
    p_d = _dev_i32(p, dev)
    if H.realified:
        p = 2 * p
    ldA = _even(p.max())
    A = torch.zeros((1, mm, ldA), dtype=_F64, device=dev)
    _lib.call("vief_gen_idmat", prob, side, _lib.ptr(L.rows if side == 0 else L.cols), mm,
              _lib.ptr(L.m_d), mm, _lib.ptr(src_xy), _lib.ptr(src_g), pmax, _lib.ptr(p_d), pmax,
              _lib.ptr(A), mm * ldA, ldA, 1, st())
    del src_xy, src_g
    pv = _dev_i32(p, dev)
    rank = torch.zeros(1, dtype=_I32, device=dev)
    perm = torch.zeros((1, mm), dtype=_I32, device=dev)
    T = torch.zeros((1, mm, mm), dtype=_F64, device=dev)
    # the same per-item seed as the item's position in the single-process batch
    _id_batched(dev, A, mm * ldA, ldA, pv, L.m_d, int(p.max()), mm, 1, 1, float(H.eps), rank,
                perm, T, int(seed) * 1000003 + L.lv, int(getattr(H, "_force_blocked", 0)),
                pairs=H.realified, couple=couple)
    del A
    L.k = rank.cpu().numpy().astype(np.int32)
    L.kmax = max(int(L.k.max()), 1)
    L.k_d = _dev_i32(L.k, dev)
    nT = L.m - L.k
    L.ntmax = max(int(nT.max()), 1)
    L.nT_d = _dev_i32(nT, dev)
    Tk = torch.zeros((1, L.ntmax, L.kmax), dtype=_F64, device=dev)
    _lib.copy2d(T, mm * mm, mm, Tk, L.ntmax * L.kmax, L.kmax, L.k_d, L.kmax, L.nT_d, L.ntmax, 1)
    del T
    if side == 1:
        send(perm, Tk)
        return
    L.perm_r, L.Tr = perm, Tk
    L.perm_c, L.Tc = recv()
    L.rskel = torch.zeros((1, L.kmax), dtype=_I32, device=dev)
    _lib.gather_int(L.rows, mm, L.perm_r, mm, L.rskel, L.kmax, L.k_d, L.kmax, 1)
    L.cskel = torch.zeros((1, L.kmax), dtype=_I32, device=dev)
    _lib.gather_int(L.cols, mm, L.perm_c, mm, L.cskel, L.kmax, L.k_d, L.kmax, 1)


class _View:
    """Attribute overrides over a _Level: a subset of its boxes presented to
    the per-level routines (TI mode runs them on the first box only)."""

    def __init__(self, base, **over):
        self.__dict__["_base"] = base
        self.__dict__.update(over)

    def __getattr__(self, name):
        return getattr(self.__dict__["_base"], name)


def _first_box(L, attrs):
    """One-box view of L: the per-box arrays / tensors named in `attrs` cut to
    box 0; padded sizes (mmax, kmax, ...) stay the level's."""
    over = dict(nb=1, ids=L.ids[:1], rects=L.rects[:1], sl=(L.sl[0], L.sl[0] + 1))
    for a in attrs:
        v = getattr(L, a, None)
        if v is not None:
            over[a] = v[:1]
    return _View(L, **over)


def _compress_level_apriori(H, L, layers):
    """Second half of a level's compression on the compressed path
    (solver_compressed.py:223-266, 437-483): the skeleton is the a-priori
    boundary band (tree.annotate_skeletons), and the interpolation
    T_up (column fields c) / T_dn (row fields b) is the least-squares solution
    of K(Z, X_sk) T = K(Z, X_rs) against the `layers` proxy rings Z.  It runs
    as the batched blocked Householder QR of [A_sk | A_rs] without pivoting
    and with the rank fixed to |sk| (vief_id_batched, kfix): T = R11^-1 R12.
    TI sharing (H.ti_share, translation-invariant kernel, every box a
    translate of the first): the fit runs for the first box only and its T is
    every box's (solver_compressed.py:548-552 factors boxes[0] only)."""
    dev = H.device
    prob = ctypes.byref(H.problem)
    st = _lib.stream_handle
    nb, mm, g = L.nb, L.mmax, H.group
    kall, pall = H.tree.ann_levels[L.lv]
    lo, hi = L.sl
    k = kall[lo:hi].astype(np.int32)
    pall = pall[lo:hi]
    if H.realified:  # unknown u = 2 * point + component; T is the realified complex fit
        k = 2 * k
        pall = (2 * pall[:, :, None] + np.arange(2)).reshape(pall.shape[0], -1)
    if pall.shape[1] != mm:
        raise ConfigError(f"level {L.lv}: annotated work sets ({pall.shape[1]}) do not match "
                          f"the children's skeletons ({mm})")
    wperm = pall.astype(np.int32)
    w = L.rects[:, 1] - L.rects[:, 0]
    h = L.rects[:, 3] - L.rects[:, 2]
    pp = proxy_count_v(w, h, layers).astype(np.int32)   # proxy points
    p = 2 * pp if H.realified else pp                  # rows of the fit
    # zero rows pad the QR to whole 32-column blocks (least squares unchanged)
    kup = np.minimum(L.m, -(-k // 32) * 32)
    if (p < k).any():
        j = int(np.argmax(k - p))
        raise ConfigError(f"box {int(L.ids[j])}: {int(p[j])} proxy points for {int(k[j])} "
                          "skeleton points (least-squares interpolation needs p >= k)")
    pv = np.maximum(p, kup).astype(np.int32)
    L.p = pp
    L.perm_r = _dev_i32(wperm, dev)
    ti = bool(getattr(H, "ti_share", False)) and nb > 1
    Fv = _first_box(L, ("m", "m_d", "rows", "cols", "perm_r")) if ti else L
    nf = Fv.nb
    _, pmax, src_xy, src_g = _level_sources(H, Fv, layers)   # proxy rings come first
    p_d = _dev_i32(pp[:nf], dev)
    pts = torch.zeros((nf, mm), dtype=_I32, device=dev)       # [sk, rs] order
    _lib.gather_int(Fv.rows, mm, Fv.perm_r, mm, pts, mm, Fv.m_d, mm, nf)
    ldA = _even(pv[:nf].max())
    A = torch.zeros((nf * g, mm, ldA), dtype=_F64, device=dev)
    # kind 0: h^2 b_i K(x_i, z) (row fields: T_dn); kind 1: h^2 K(z, x_j) c_j (T_up)
    _lib.call("vief_gen_idmat", prob, 0, _lib.ptr(pts), mm, _lib.ptr(Fv.m_d), mm,
              _lib.ptr(src_xy), _lib.ptr(src_g), pmax, _lib.ptr(p_d), pmax, _lib.ptr(A),
              g * mm * ldA, ldA, nf, st())
    if g == 2:
        _lib.call("vief_gen_idmat", prob, 1, _lib.ptr(pts), mm, _lib.ptr(Fv.m_d), mm,
                  _lib.ptr(src_xy), _lib.ptr(src_g), pmax, _lib.ptr(p_d), pmax,
                  _lib.ptr(A) + 8 * mm * ldA, g * mm * ldA, ldA, nf, st())
    del src_xy, src_g, pts
    count = nf * g
    pvd = _dev_i32(np.repeat(pv[:nf], g), dev)
    mv = _dev_i32(np.repeat(L.m[:nf], g), dev)
    kfix = _dev_i32(np.repeat(k[:nf], g), dev)
    rank = torch.zeros(count, dtype=_I32, device=dev)
    perm = torch.zeros((count, mm), dtype=_I32, device=dev)
    T = torch.zeros((count, mm, mm), dtype=_F64, device=dev)
    _id_batched(dev, A, mm * ldA, ldA, pvd, mv, int(pv[:nf].max()), mm, count, g, float(H.eps),
                rank, perm, T, 0, 1, kfix)
    del A, perm
    L.k = k
    L.kmax = max(int(k.max()), 1)
    L.k_d = _dev_i32(k, dev)
    nT = L.m - k
    L.ntmax = max(int(nT.max()), 1)
    L.nT_d = _dev_i32(nT, dev)
    L.perm_c = L.perm_r
    L.Tr = torch.zeros((nf, L.ntmax, L.kmax), dtype=_F64, device=dev)
    _lib.copy2d(T, g * mm * mm, mm, L.Tr, L.ntmax * L.kmax, L.kmax, L.k_d, L.kmax, L.nT_d,
                L.ntmax, nf)
    if g == 2:
        L.Tc = torch.zeros_like(L.Tr)
        _lib.copy2d(_lib.ptr(T) + 8 * mm * mm, g * mm * mm, mm, L.Tc, L.ntmax * L.kmax, L.kmax,
                    L.k_d, L.kmax, L.nT_d, L.ntmax, nf)
    else:
        L.Tc = L.Tr
    del T
    if ti:  # every box's interpolation is the first box's
        L.Tr = L.Tr.expand(nb, -1, -1).contiguous()
        L.Tc = L.Tr if g == 1 else L.Tc.expand(nb, -1, -1).contiguous()
    L.rskel = torch.zeros((nb, L.kmax), dtype=_I32, device=dev)
    _lib.gather_int(L.rows, mm, L.perm_r, mm, L.rskel, L.kmax, L.k_d, L.kmax, nb)
    if g == 2:
        L.cskel = torch.zeros((nb, L.kmax), dtype=_I32, device=dev)
        _lib.gather_int(L.cols, mm, L.perm_r, mm, L.cskel, L.kmax, L.k_d, L.kmax, nb)
    else:
        L.cskel = L.rskel


# The IDs (compression) are the factorization's critical path; the inversions
# fill the gaps.  Their stream gets the highest priority, so the ID chain's
# latency-bound cluster kernels (sketch selection, QR panels) are placed as soon
# as SMs free up instead of queueing behind the inversion's GEMM waves.  A
# level's IDs run as one batch on that stream: splitting the batch over two or
# more streams (each with its own host thread) was measured slower once the
# inversion stream fills the ID chain's gaps (1913 ms/step with one batch vs
# 1934 / 1946 / 1955 ms with 2 / 3 / 4 slices).
_ID_PRIORITY = -100


def _id_batched(dev, A, sA, ldA, pv, mv, maxp, mm, count, g, eps, rank, perm, T, seed, forced,
                kfix=None, pairs=False, couple=None):
    """vief_id_batched over `count` items (groups of g share a rank); `kfix`
    (device int32, count) fixes the ranks and disables pivoting; `pairs`: the
    columns are realified complex unknowns, pivoted pairwise; `couple`: a
    _lib.COUPLE_FN coupling this item's rank with another process's."""
    d = _lib.IdDesc(_lib.ptr(A), sA, ldA, _lib.ptr(pv), _lib.ptr(mv), maxp, mm, count, g, eps,
                    _lib.ptr(rank), _lib.ptr(perm), _lib.ptr(T), mm * mm, mm, seed, forced,
                    None if kfix is None else _lib.ptr(kfix), int(pairs),
                    None if couple is None else ctypes.cast(couple.fn, ctypes.c_void_p), None)
    _lib.call("vief_id_batched", ctypes.byref(d), _lib.stream_handle())
    err = getattr(couple, "error", None)
    if err is not None:
        raise err


def compress_outer(spec, grid, tree, eps, opts, quad=PLAIN, spill=None):
    """Skeletonize all boxes fine-to-coarse, one batch per level
    (solver_dense.py:234-272).  The compressed operator's blocks stay in HBM
    (they feed the inversion level by level); `spill` is accepted for the
    reference's signature -- the factor tier is invert_dense_block(spill=)."""
    H = Hss2dMatrix(spec, grid, tree, eps, opts, quad)
    return compress_levels(H)


def compress_levels(H):
    """Run the per-level compression over every level H factors (fine to
    coarse); sharded objects (distributed.py) call this directly."""
    pad = H.opts.resolved_proxy_layers(H.spec)
    _mark("compress:start")
    with _host_quiet():
        for L in reversed(_real_levels(H)):
            _lib.prof_prefix(f"L{L.lv:02d}.")
            _compress_level(H, L, pad, H.opts.seed)
            _mark(f"compress:{L.lv}")
    return H


# ---------------------------------------------------------------------------
# invert_dense_block

def _check_singular(H, L, pmin, pmax, what):
    lo, hi = pmin.cpu().numpy(), pmax.cpu().numpy()
    eps2 = np.finfo(float).eps ** 2
    bad = (hi == 0.0) | (lo <= 1e-300) | (lo / np.where(hi == 0.0, 1.0, hi) < eps2) | ~np.isfinite(lo)
    if bad.any():
        j = int(np.flatnonzero(bad)[0])
        i = int(L.ids[j])
        where = f"box {i} level {L.lv}" if what == "F" else f"E of box {i}"
        raise SingularFactorError(where, float(lo[j]))


def _invert_level(inv, L, checks=None):
    """`checks`: if a list, singularity tests are queued there instead of being
    run now (running them reads device data and would block the host)."""
    _invert_level_F(inv, L, checks)
    _invert_level_rest(inv, L, checks)


def _invert_root_block(inv, L, checks=None):
    """Root F = [[E1, B12], [B21, E2]] by block elimination instead of an
    explicit inverse: E1^{-1} = G1 is level 1's G (kept before inverting it),
    so only the Schur complement S = E2 - B21 G1 B12 (k2 x k2) is inverted:
    ~1.4 TF instead of 2 m^3 = 3.7 TF at 1024^2 (the root needs F^{-1} only
    applied to vectors).  The singularity test runs on S (F is singular iff S
    is: E1 is invertible, its inverse G1 was checked at level 1)."""
    H = inv.H
    dev = H.device
    C = H.levels[1]
    kc = C.kmax
    k1, k2 = int(C.k[0]), int(C.k[1])
    _lib.prof_mark("py.root_schur")
    G1 = C.Gkeep[0]                                     # (kc, kc) storage [col, row]
    T1 = torch.zeros((kc, kc), dtype=_F64, device=dev)   # G1 B12 (k1 x k2)
    _lib.gemm(G1, L.B12[0], T1, M=k1, N=k2, K=k1, lda=kc, ldb=kc, ldc=kc)
    S = torch.zeros((1, kc, kc), dtype=_F64, device=dev)
    S[0, :k2, :k2] = C.E[1, :k2, :k2]
    _lib.gemm(L.B21[0], T1, S[0], M=k2, N=k2, K=k1, lda=kc, ldb=kc, ldc=kc, alpha=-1.0, beta=1.0)
    del T1
    k2d = C.k_d[1:2].contiguous()
    _lib.pad_identity(S, kc * kc, kc, k2d, kc, 1)
    pmin, pmax = _lib.inv_batched(S, kc * kc, kc, kc, 1)
    L._fpiv = (pmin, pmax)
    if checks is None:
        _check_singular(H, L, pmin, pmax, "F")
    else:
        checks.append((L, pmin, pmax, "F"))
    L.rb = (G1, L.B12[0], L.B21[0], S[0], k1, k2, kc)
    C.Gkeep = None  # the root's block factors hold the one G1 the solve needs
    L.Finv = None


def _root_block_solve(L, U, ldu, r, Phi, ldp):
    """Phi = F^{-1} U at the root from the block factors (U, Phi: (r, ld) with
    the k1 + k2 root unknowns first)."""
    G1, B12, B21, Sinv, k1, k2, kc = L.rb
    dev = U.device
    Y1 = torch.zeros((r, kc), dtype=_F64, device=dev)
    _mv(G1, 0, kc, U, 0, ldu, Y1, 0, kc, k1, k1, None, None, 1, r, 1.0, 0.0)       # G1 u1
    Z2 = U[:, k1:k1 + k2].contiguous()
    _mv(B21, 0, kc, Y1, 0, kc, Z2, 0, k2, k2, k1, None, None, 1, r, -1.0, 1.0)     # u2 - B21 y1
    X2 = Phi[:, k1:]
    _mv(Sinv, 0, kc, Z2, 0, k2, X2, 0, ldp, k2, k2, None, None, 1, r, 1.0, 0.0)    # x2
    Wt = torch.zeros((r, kc), dtype=_F64, device=dev)
    _mv(B12, 0, kc, X2, 0, ldp, Wt, 0, kc, k1, k2, None, None, 1, r, 1.0, 0.0)     # B12 x2
    Phi[:, :k1] = Y1[:, :k1]
    _mv(G1, 0, kc, Wt, 0, kc, Phi, 0, ldp, k1, k1, None, None, 1, r, -1.0, 1.0)    # x1


def _invert_level_F_block(inv, L, checks=None):
    """Explicit F^{-1} of F = [[E1, B12], [B21, E2]] by block elimination with
    E1^{-1} = G1 (the first child's G, kept before it was inverted):
        T1 = G1 B12,  S = E2 - B21 T1,  S^{-1} (GJ, k2 x k2),  T2 = B21 G1,
        F^{-1} = [[G1 - T1 X21, -T1 S^{-1}], [X21 = -S^{-1} T2, S^{-1}]].
    1.75 m^3 flops, all but the k2 x k2 inversion as batched GEMMs, instead of
    a 2 m^3 Gauss-Jordan of the whole F.  F is singular iff S is (G1 is the
    checked-invertible inverse of E1), so the singularity test runs on S."""
    H = inv.H
    dev = H.device
    nb, mm = L.nb, L.mmax
    C = H.levels[L.lv + 1]
    kc = C.kmax
    k1 = C.k[0::2].astype(np.int64)
    k1d, k2d = C.k_d[0::2].contiguous(), C.k_d[1::2].contiguous()
    s2 = kc * kc
    _lib.prof_mark("py.F_block")
    G1 = C.Gkeep                                         # (nb, kc, kc) [item, col, row]
    T1 = torch.zeros((nb, kc, kc), dtype=_F64, device=dev)
    _lib.gemm(G1, L.B12, T1, M=kc, N=kc, K=kc, lda=kc, ldb=kc, ldc=kc, sA=s2, sB=s2, sC=s2,
              batch=nb, Mb=k1d, Nb=k2d, Kb=k1d)
    S = torch.zeros((nb, kc, kc), dtype=_F64, device=dev)
    _lib.copy2d(_lib.ptr(C.E) + 8 * s2, 2 * s2, kc, S, s2, kc, k2d, kc, k2d, kc, nb)  # E2
    _lib.gemm(L.B21, T1, S, M=kc, N=kc, K=kc, lda=kc, ldb=kc, ldc=kc, sA=s2, sB=s2, sC=s2,
              alpha=-1.0, beta=1.0, batch=nb, Mb=k2d, Nb=k2d, Kb=k1d)
    _lib.pad_identity(S, s2, kc, k2d, kc, nb)
    pmin, pmax = _lib.inv_batched(S, s2, kc, kc, nb)
    L._fpiv = (pmin, pmax)
    if checks is None:
        _check_singular(H, L, pmin, pmax, "F")
    else:
        checks.append((L, pmin, pmax, "F"))
    T2 = torch.zeros((nb, kc, kc), dtype=_F64, device=dev)
    _lib.gemm(L.B21, G1, T2, M=kc, N=kc, K=kc, lda=kc, ldb=kc, ldc=kc, sA=s2, sB=s2, sC=s2,
              batch=nb, Mb=k2d, Nb=k1d, Kb=k1d)
    F = torch.zeros((nb, mm, mm), dtype=_F64, device=dev)
    base = np.arange(nb, dtype=np.int64) * mm * mm
    p21 = _ptrs(F, base + k1, dev)                       # rows k1.., cols 0..
    p12 = _ptrs(F, base + k1 * mm, dev)                  # rows 0.., cols k1..
    p22 = _ptrs(F, base + k1 * mm + k1, dev)
    _lib.gemm(S, T2, None, M=kc, N=kc, K=kc, lda=kc, ldb=kc, ldc=mm, sA=s2, sB=s2,
              alpha=-1.0, beta=0.0, batch=nb, Mb=k2d, Nb=k1d, Kb=k2d, Cptr=p21)   # X21
    del T2
    _lib.copy2d(G1, s2, kc, F, mm * mm, mm, k1d, kc, k1d, kc, nb)                  # G1
    _lib.gemm(T1, None, F, M=kc, N=kc, K=kc, lda=kc, ldb=mm, ldc=mm, sA=s2, sC=mm * mm,
              alpha=-1.0, beta=1.0, batch=nb, Mb=k1d, Nb=k1d, Kb=k2d, Bptr=p21)   # X11
    _lib.gemm(T1, S, None, M=kc, N=kc, K=kc, lda=kc, ldb=kc, ldc=mm, sA=s2, sB=s2,
              alpha=-1.0, beta=0.0, batch=nb, Mb=k1d, Nb=k2d, Kb=k2d, Cptr=p12)   # X12
    _lib.copy2d(S, s2, kc, None, 0, mm, k2d, kc, k2d, kc, nb, dstp=p22)            # X22
    del T1, S
    C.Gkeep = None  # consumed: only this block elimination reads the children's G1
    _lib.pad_identity(F, mm * mm, mm, L.m_d, mm, nb)
    L.Finv = F


def _assemble_F(H, L):
    """The level's F blocks, nb x mm x mm padded with identity: D at the leaves,
    [[E1, B12], [B21, E2]] above (solver_dense.py:346-352)."""
    dev = H.device
    nb, mm = L.nb, L.mmax
    F = torch.zeros((nb, mm, mm), dtype=_F64, device=dev)
    if L.leaf:
        F.copy_(L.D)
    else:
        C = H.levels[L.lv + 1]
        kc = C.kmax
        CE = C.E if C.E.is_cuda else C.E.to(dev)
        if getattr(C, "ti", False) and CE.shape[0] < C.nb:   # one shared record
            CE = CE[0:1].expand(C.nb, -1, -1).contiguous()
        k1 = C.k[0::2].astype(np.int64)
        k1d, k2d = C.k_d[0::2].contiguous(), C.k_d[1::2].contiguous()
        base = np.arange(nb, dtype=np.int64) * mm * mm
        # F[:k1,:k1] = E1 ; F[k1:,k1:] = E2 ; F[:k1,k1:] = B12 ; F[k1:,:k1] = B21
        _lib.copy2d(CE, 2 * kc * kc, kc, F, mm * mm, mm, k1d, kc, k1d, kc, nb)
        _lib.copy2d(_lib.ptr(CE) + 8 * kc * kc, 2 * kc * kc, kc, None, 0, mm, k2d, kc, k2d, kc, nb,
                    dstp=_ptrs(F, base + k1 * mm + k1, dev))
        _lib.copy2d(L.B12, kc * kc, kc, None, 0, mm, k1d, kc, k2d, kc, nb,
                    dstp=_ptrs(F, base + k1 * mm, dev))
        _lib.copy2d(L.B21, kc * kc, kc, None, 0, mm, k2d, kc, k1d, kc, nb,
                    dstp=_ptrs(F, base + k1, dev))
    _lib.pad_identity(F, mm * mm, mm, L.m_d, mm, nb)
    return F


# Ill-conditioned box solves.  The factors hold explicit inverses (F^-1 and E
# by Gauss-Jordan, W = F^-1 L by GEMM); applying an explicit inverse to a
# vector is not backward stable, so where F is badly conditioned (near-
# resonant Helmholtz boxes: cond(F) ~ 1e10+ at kappa = 40, config c3) the
# sweeps' x = F^-1 u would leave residuals cond(F) eps |F| |x|, where the
# reference's LU solves (solver_dense.py:309,321 lu_solve) leave eps |F| |x|.
# Such levels refine every box solve against F itself (x += F^-1 (u - F x),
# _REFINE_STEPS times), which restores the LU solve's accuracy.  A level is
# flagged when the pivot spread of its elimination, max|U_ii| / min|U_ii| (a
# lower bound on cond(F)), exceeds _REFINE_COND; well-conditioned problems
# (all Laplace configs) run the plain sweeps.
_REFINE_COND = 1e6
_REFINE_STEPS = 2
_BLOCK_E_MAX = 1e4   # largest child |E| entry for which F^-1 is formed by block elimination


def _level_cond_est(H, L):
    """Device scalar: the largest max|U_ii| / min|U_ii| of the level's
    Gauss-Jordan eliminations of F (or of its Schur complement S in block
    form) -- a lower bound on cond(F) that costs nothing (the kernel reports
    the pivot extremes for the singularity test)."""
    pmin, pmax = L.__dict__.pop("_fpiv")
    return (pmax / pmin).amax()


def _flag_refinement(H, ests):
    """ests: {level: device scalar}; one host read for all levels."""
    if not ests:
        return
    lv = list(ests)
    vals = torch.stack([ests[l] for l in lv]).cpu().numpy()
    for l, v in zip(lv, vals):
        H.levels[l].cond_est = float(v)
        H.levels[l].refine = bool(not np.isfinite(v) or v > _REFINE_COND)


def _invert_level_F(inv, L, checks=None):
    """F = D (leaf) or [[E1, B12], [B21, E2]] and its inverse; records the
    level's conditioning estimate for _flag_refinement."""
    _invert_level_F_impl(inv, L, checks)
    ests = getattr(inv, "_ests", None)
    if ests is None:
        ests = inv._ests = {}
    ests[L.lv] = _level_cond_est(inv.H, L)


def _invert_level_F_impl(inv, L, checks=None):
    H = inv.H
    dev = H.device
    nb, mm = L.nb, L.mmax
    C1 = H.levels[L.lv + 1] if L.lv + 1 < len(H.levels) else None
    if not L.leaf and getattr(C1, "Gkeep", None) is not None:
        # block elimination substitutes G1 = E1^{-1} for the children's explicit
        # E1; with an ill-conditioned G1 (|E| >> 1: near-resonant boxes) the two
        # differ by cond(G1) eps |E1|, so such levels invert the assembled F
        if float(torch.linalg.vector_norm(C1.E, float("inf"))) <= _BLOCK_E_MAX:
            if L.lv == 0:
                return _invert_root_block(inv, L, checks)
            return _invert_level_F_block(inv, L, checks)
        C1.Gkeep = None
    _lib.prof_mark("py.F_assemble")
    F = _assemble_F(H, L)
    pmin, pmax = _lib.inv_batched(F, mm * mm, mm, mm, nb)
    L._fpiv = (pmin, pmax)
    if checks is None:
        _check_singular(H, L, pmin, pmax, "F")
    else:
        checks.append((L, pmin, pmax, "F"))
    L.Finv = F


def _invert_level_rest(inv, L, checks=None):
    """W = F^{-1} L, G = R W, E = G^{-1}, C = E R (needs the level's ID)."""
    H = inv.H
    dev = H.device
    nb, mm = L.nb, L.mmax
    F = L.Finv
    if L.lv == 0:
        return
    kk = L.kmax
    k = L.k.astype(np.int64)
    base = np.arange(nb, dtype=np.int64)
    _lib.prof_mark("py.W")
    # W = F^{-1} L = Fp[:, :k] + Fp[:, k:] Tr^T,  Fp = F^{-1}[:, perm_r]
    Fp = torch.empty((nb, mm, mm), dtype=_F64, device=dev)
    _lib.gather_cols(F, mm * mm, mm, L.perm_r, mm, Fp, mm * mm, mm, L.m_d, mm, L.m_d, mm, nb)
    W = torch.zeros((nb, kk, mm), dtype=_F64, device=dev)
    _lib.copy2d(Fp, mm * mm, mm, W, kk * mm, mm, L.m_d, mm, L.k_d, kk, nb)
    _lib.gemm(None, L.Tr, W, M=mm, N=kk, K=L.ntmax, lda=mm, ldb=kk, ldc=mm,
              sB=L.ntmax * kk, sC=kk * mm, tB=1, alpha=1.0, beta=1.0, batch=nb,
              Mb=L.m_d, Nb=L.k_d, Kb=L.nT_d, Aptr=_ptrs(Fp, base * mm * mm + k * mm, dev))
    del Fp
    _lib.prof_mark("py.G")
    # G = R W = Wp[:k] + Tc Wp[k:],  Wp = W[perm_c, :]
    Wp = torch.empty((nb, kk, mm), dtype=_F64, device=dev)
    _lib.gather_rows(W, kk * mm, mm, L.perm_c, mm, Wp, kk * mm, mm, L.m_d, mm, L.k_d, kk, nb)
    G = torch.zeros((nb, kk, kk), dtype=_F64, device=dev)
    _lib.copy2d(Wp, kk * mm, mm, G, kk * kk, kk, L.k_d, kk, L.k_d, kk, nb)
    _lib.gemm(L.Tc, None, G, M=kk, N=kk, K=L.ntmax, lda=kk, ldb=mm, ldc=kk,
              sA=L.ntmax * kk, sC=kk * kk, alpha=1.0, beta=1.0, batch=nb,
              Mb=L.k_d, Nb=L.k_d, Kb=L.nT_d, Bptr=_ptrs(Wp, base * kk * mm + k, dev))
    del Wp
    if nb >= 2 or H.sharded:  # the parent's block elimination needs G1 = E1^{-1}
        # (a sharded slice keeps it for a single box too: its parent may be
        # factored by the same rank from a virtual child level, distributed.py)
        L.Gkeep = G[0::2].clone()
    _lib.pad_identity(G, kk * kk, kk, L.k_d, kk, nb)
    pmin, pmax = _lib.inv_batched(G, kk * kk, kk, kk, nb)
    if checks is None:
        _check_singular(H, L, pmin, pmax, "E")
    else:
        checks.append((L, pmin, pmax, "E"))
    L.E = G
    L.W = W
    _lib.prof_mark("py.C")
    # C = E R: Cp = [E, E Tc] then columns scattered to perm_c
    Cp = torch.zeros((nb, mm, kk), dtype=_F64, device=dev)
    _lib.copy2d(G, kk * kk, kk, Cp, mm * kk, kk, L.k_d, kk, L.k_d, kk, nb)
    _lib.gemm(G, L.Tc, None, M=kk, N=L.ntmax, K=kk, lda=kk, ldb=kk, ldc=kk,
              sA=kk * kk, sB=L.ntmax * kk, alpha=1.0, beta=0.0, batch=nb,
              Mb=L.k_d, Nb=L.nT_d, Kb=L.k_d, Cptr=_ptrs(Cp, base * mm * kk + k * kk, dev))
    Cm = torch.zeros((nb, mm, kk), dtype=_F64, device=dev)
    _lib.scatter_cols(Cp, mm * kk, kk, L.perm_c, mm, Cm, mm * kk, kk, L.k_d, kk, L.m_d, mm, nb)
    L.C = Cm


class DenseBlockInverse:
    """Per-box factors of the telescoping inverse (solver_dense.py:275-329),
    held in HBM as per-level batches: F^{-1}, W = F^{-1}L, E, C = E R."""

    def __init__(self, H):
        self.H = H
        self.tree = H.tree

    def _ids(self, nonroot):
        return [int(i) for L in _real_levels(self.H) if (L.lv > 0 or not nonroot) for i in L.ids]

    @property
    def E(self):
        return _BoxView(self, lambda i: self._get(i, "E"), lambda: self._ids(True))

    @property
    def Finv(self):
        return _BoxView(self, lambda i: self._get(i, "Finv"), lambda: self._ids(False))

    def _get(self, i, which):
        L, j = self.H._lvl_of[i]
        m = int(L.m[j])
        jr = 0 if getattr(L, "ti", False) else j   # TI: the level's shared record
        if getattr(L, "hss", None) is not None:    # densified from the HSS forms (small n)
            hF, hE = L.hss
            if which == "E":
                k = int(L.k[j])
                return hE.to_dense()[j, :k, :k].t().cpu().numpy()
            P = hF.to_dense()[j].t()[:m, :m].cpu().numpy()  # rows perm_c, columns perm_r
            out = np.empty_like(P)
            out[np.ix_(L.perm_c[j, :m].cpu().numpy(), L.perm_r[j, :m].cpu().numpy())] = P
            return out
        if which == "E":
            k = int(L.k[j])
            return L.E[jr, :k, :k].t().cpu().numpy()
        j = jr
        if getattr(L, "rb", None) is not None:  # root in block form: F^{-1} = solve(I)
            eye = torch.eye(m, dtype=_F64, device=self.H.device)
            X = torch.zeros_like(eye)
            _root_block_solve(L, eye, m, m, X, m)
            return X.cpu().numpy()
        return L.Finv[j, :m, :m].t().cpu().numpy()

    def nbytes(self):
        """Bytes of the factors this object holds (F^{-1}, E, W, C, T)."""
        tot = 0
        H = self.H
        for L in _real_levels(H):
            m = L.m.astype(np.int64)
            k = L.k.astype(np.int64) if L.lv > 0 else None
            if getattr(L, "hss", None) is not None:   # 1-D HSS blocks + the dense T
                from . import compressed_store
                tot += compressed_store.hss_bytes(L)
                tot += int((k * (m - k)).sum()) * 8 * H.group
                continue
            if getattr(L, "ti", False):  # one shared record per level
                m = m[:1]
                k = k[:1]
            tot += int((m * m).sum()) * 8
            if L.lv > 0:
                tot += int((k * k + 2 * k * m).sum()) * 8
                tot += int((k * (m - k)).sum()) * 8 * H.group
        return tot

    def nbytes_reference_layout(self):
        """What the reference's inv.nbytes() would count for the same ranks:
        F + E + T (solver_dense.py:284-291)."""
        tot = 0
        H = self.H
        for L in _real_levels(H):
            m = L.m.astype(np.int64)
            tot += int((m * m).sum()) * 8
            if L.lv > 0:
                k = L.k.astype(np.int64)
                tot += int((k * k).sum()) * 8 + int((k * (m - k)).sum()) * 8 * H.group
        return tot

    def apply(self, f):
        return _apply(self, f)

    def save(self, path):
        """Write the factors to `path` (persist.py); `load` restores them."""
        from . import persist
        persist.save(self, path)

    @staticmethod
    def load(path, device=None):
        from . import persist
        return persist.load(path, device)


class _Spill:
    """Host-memory tier for factor blocks (the reference's _Spill,
    solver_dense.py:37-55, backs blocks of >= threshold_mb by .npy memmaps).
    Here a level's factor batches (F^-1, C, E, W) of >= threshold_mb MB move
    to pinned host memory as soon as the factorization no longer needs them
    (after the parent level is inverted); the solve streams each level back
    to HBM on a copy stream one level ahead of the sweep, so at most two
    levels' factors are resident.  threshold_mb=None: nothing spills."""

    def __init__(self, threshold_mb=None):
        self.threshold = None if threshold_mb is None else threshold_mb * (1 << 20)

    def hold(self, t):
        if self.threshold is None or not t.is_cuda or t.numel() * t.element_size() < self.threshold:
            return t
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        return h

    def spill_level(self, L):
        if self.threshold is None or L is None or getattr(L, "virtual", False):
            return
        for name in _FACTOR_NAMES:
            t = getattr(L, name, None)
            if isinstance(t, torch.Tensor):
                setattr(L, name, self.hold(t))


_FACTOR_NAMES = ("Finv", "C", "E", "W")


def _as_spill(spill):
    if spill is None:
        return None
    if isinstance(spill, _Spill):
        return spill
    if isinstance(spill, (int, float)):
        return _Spill(spill)
    thr = getattr(spill, "threshold", None)   # a reference-style _Spill (bytes)
    sp = _Spill(None)
    sp.threshold = thr
    return sp


class _Prefetch:
    """Device copies of spilled factor batches, one level ahead of the sweep
    (copy stream + event; the caching allocator's record_stream keeps each
    buffer alive until the sweep has used it).  Levels held in HBM pass
    through untouched (get() returns None)."""

    def __init__(self, H, order, names):
        self.H, self.order, self.names = H, order, names
        self.pending = {}
        self.stream = None

    def _spilled(self, L):
        return any(isinstance(getattr(L, n, None), torch.Tensor) and not getattr(L, n).is_cuda
                   for n in self.names)

    def _issue(self, i):
        L = self.order[i]
        if not self._spilled(L):
            self.pending[i] = None
            return
        if self.stream is None:
            self.stream = torch.cuda.Stream(self.H.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.H.device))
        out = {}
        with torch.cuda.stream(self.stream):
            for n in self.names:
                t = getattr(L, n, None)
                out[n] = t.to(self.H.device, non_blocking=True) if t is not None and not t.is_cuda else t
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.pending[i] = (out, ev)

    def get(self, i):
        if i not in self.pending:
            self._issue(i)
        if i + 1 < len(self.order) and i + 1 not in self.pending:
            self._issue(i + 1)
        ent = self.pending.pop(i)
        if ent is None:
            return None
        out, ev = ent
        cur = torch.cuda.current_stream(self.H.device)
        cur.wait_event(ev)
        for t in out.values():
            if t is not None and t.is_cuda:
                t.record_stream(cur)
        return out


def invert_dense_block(H, spill=None, free_source=False, storage="dense", compress=False):
    """Fine-to-coarse telescoping inversion, one batch per level
    (solver_dense.py:332-368).  `free_source` drops D/B once consumed;
    `spill` (a _Spill, or a threshold in MB) moves each finished level's
    factor batches above the threshold to pinned host memory.  `storage`:
    "dense" keeps F^-1, E, W = F^-1 L and C = E R per box (fastest solve);
    "lean" keeps F^-1 and E only, as the reference does (F_lu, E, T:
    solver_dense.py:284-291), and the sweeps apply T (compressed_store.py);
    "hss1d" also stores large a-priori-path blocks in 1-D HSS form.  Either way
    a level is converted as soon as its parent is factored.  `compress`: H's
    levels are compressed here, each just before it is inverted (a level's
    compression needs its children's skeleton lists only), so that with
    `free_source` one level's D / B / ID matrices are resident at a time
    instead of the whole tree's -- the low-memory schedule for the largest
    grids (compress_outer + invert_dense_block hold all levels' sources)."""
    if storage not in ("dense", "lean", "hss1d"):
        raise ConfigError(f"unknown storage {storage!r}")
    inv = DenseBlockInverse(H)
    sp = _as_spill(spill)
    _mark("invert:start")
    with _host_quiet():
        levels = list(reversed(_real_levels(H)))
        pad = H.opts.resolved_proxy_layers(H.spec)
        for i, L in enumerate(levels):
            _lib.prof_prefix(f"L{L.lv:02d}.")
            if compress and getattr(L, "m", None) is None:
                # cached blocks back to the driver when memory runs short: torch's
                # allocator and the library's stream-ordered pool share the HBM
                _lib.release_memory_if_low()
                _compress_level(H, L, pad, H.opts.seed)
                _mark(f"compress:{L.lv}")
            _invert_level(inv, L)
            _mark(f"invert:{L.lv}")
            if free_source:  # a level whose box solves are refined keeps its F blocks
                _flag_refinement(H, {L.lv: inv._ests.pop(L.lv)})
                if L.refine:
                    pass
                elif L.leaf:
                    L.D = None
                else:
                    L.B12 = L.B21 = None
            if storage in ("hss1d", "lean") and i > 0:   # the parent's F is assembled
                from . import compressed_store
                if compress:
                    _lib.release_memory_if_low()
                compressed_store.compact_level(
                    H, levels[i - 1], min_size=None if storage == "hss1d" else float("inf"))
            if sp is not None and i > 0:   # the child level is no longer needed here
                sp.spill_level(levels[i - 1])
        if sp is not None and levels:
            sp.spill_level(levels[-1])
            torch.cuda.current_stream(H.device).synchronize()   # pinned copies complete
            torch.cuda.empty_cache()
        _flag_refinement(H, inv.__dict__.pop("_ests", {}))
    return inv


_SIDE = {}


_QUIET_DEPTH = [0]


_TPC = [None, -1]


def _threadpools():
    """threadpoolctl controller of the loaded BLAS/OpenMP libraries (rebuilt
    when modules were imported since: a fresh scan costs ~1 ms)."""
    import sys
    if _TPC[0] is None or _TPC[1] != len(sys.modules):
        from threadpoolctl import ThreadpoolController
        _TPC[0], _TPC[1] = ThreadpoolController(), len(sys.modules)
    return _TPC[0]


@contextlib.contextmanager
def _host_quiet():
    """Keep the host quiet while the level loops drive the GPU from several
    threads (caller, ID slices, inversion worker), each of which waits on its
    stream once per ID column block:
      * host BLAS / OpenMP pools limited to one thread -- their idle workers
        spin after every call and starved the stream-driving threads (measured
        at 1024^2: random 100-480 ms stalls of a level, none with one thread);
      * Python's cyclic GC held (a collection stops every thread at the GIL;
        the loops create no reference cycles)."""
    if _QUIET_DEPTH[0] > 0:
        yield
        return
    gc_was = gc.isenabled()
    nthr = torch.get_num_threads()
    _QUIET_DEPTH[0] += 1
    try:
        with _threadpools().limit(limits=1):
            torch.set_num_threads(1)
            gc.disable()
            yield
    finally:
        _QUIET_DEPTH[0] -= 1
        torch.set_num_threads(nthr)
        if gc_was:
            gc.enable()


def factor_solve(spec, grid, tree, eps, opts, f, quad=PLAIN, apriori=None):
    """factorize() and the solve of f in one pass: the up sweep of level l runs
    (third stream) as soon as level l is inverted, overlapping the
    factorization of the coarser levels; the down sweep follows.  Returns
    (H, inv, x) with x = inv.apply(f) (bitwise: same kernels, same order per
    level)."""
    with _host_quiet():
        H, inv, (fd, single, phi, ups) = _factorize(spec, grid, tree, eps, opts, quad, rhs=f,
                                                    apriori=apriori)
        if any(getattr(L, "refine", False) for L in _real_levels(H)):
            phi, ups = {}, {}      # refined box solves: the pipelined up sweep ran without
            _sweep_up(H, fd, phi, ups)
        out = torch.zeros_like(fd)
        _sweep_down(H, phi, ups, out)
        return H, inv, _from_device(out, f, single, H.realified)


def factorize(spec, grid, tree, eps, opts, quad=PLAIN, apriori=None, ti=False):
    """`apriori` = boundary-layer width: skeletons from tree.annotate_skeletons
    (the compressed path's a-priori choice) instead of the IDs.  `ti` (with
    `apriori`, a translation-invariant kernel and uniform levels): factor the
    first box of every level only and share its record (TI mode,
    solver_compressed.py:548-552)."""
    with _host_quiet():
        H, inv, _ = _factorize(spec, grid, tree, eps, opts, quad, apriori=apriori, ti=ti)
    return H, inv


def _factorize(spec, grid, tree, eps, opts, quad=PLAIN, rhs=None, apriori=None, ti=False,
               H=None):
    """compress_outer + invert_dense_block with the levels pipelined over two
    CUDA streams: level l is inverted (side stream) while level l-1 is being
    compressed (current stream).  Inverting level l needs only level l's
    compression and level l+1's inversion, so this is the same computation in
    a different order; the latency-bound panels of one stage overlap the
    GEMMs of the other.  Singularity checks run at the end (same exception)."""
    if H is None:   # (a sharded slice passes its own object, distributed.py)
        H = Hss2dMatrix(spec, grid, tree, eps, opts, quad)
    H.apriori = apriori
    H.ti_share = bool(ti and apriori)
    pad = H.opts.resolved_proxy_layers(H.spec)
    inv = DenseBlockInverse(H)
    # compression on the caller's stream, inversions on a second stream (a
    # high-priority compression stream was measured slower: 2.54 vs 2.46 s)
    caller = torch.cuda.current_stream(H.device)
    if H.device not in _SIDE:
        _SIDE[H.device] = (torch.cuda.Stream(H.device), torch.cuda.Stream(H.device),
                           torch.cuda.Stream(H.device, priority=_ID_PRIORITY))
    side, third, main = _SIDE[H.device]
    solve = None
    if rhs is not None:
        fd, single = _as_device_rhs(rhs, grid.n, H.device, H.realified)
        solve = (fd, single, {}, {})
    main.wait_stream(caller)
    with torch.cuda.stream(main):
        _factorize_levels(H, inv, pad, main, side, third, solve)
    caller.wait_stream(main)
    caller.wait_stream(side)
    caller.wait_stream(third)
    checks, inv._checks = inv._checks, []
    for L, pmin, pmax, what in checks:
        _check_singular(H, L, pmin, pmax, what)
    _flag_refinement(H, inv.__dict__.pop("_ests", {}))
    return H, inv, solve


class _Worker:
    """A persistent host thread that enqueues work on one CUDA stream (started
    once per device: a fresh thread pays the CUDA per-thread setup)."""

    def __init__(self, dev_index, stream):
        import queue
        import threading
        self.tasks = queue.Queue()
        self.stream = stream
        self.dev_index = dev_index
        self.th = threading.Thread(target=self._run, name="vief-invert", daemon=True)
        self.th.start()

    def _run(self):
        torch.cuda.set_device(self.dev_index)
        with torch.cuda.stream(self.stream):
            while True:
                fn, args, ev, box = self.tasks.get()
                if box.get("error") is not None:
                    fn = args = ev = None
                    with box["cv"]:
                        box["pending"] -= 1
                        box["cv"].notify_all()
                    continue
                try:
                    if ev is not None:
                        self.stream.wait_event(ev)
                    fn(*args)
                except BaseException as e:  # re-raised on the caller's thread
                    box["error"] = e
                # drop the task's references (the factor object) before idling
                fn = args = ev = None
                with box["cv"]:
                    box["pending"] -= 1
                    box["cv"].notify_all()
                box = None

    def submit(self, box, fn, args, ev):
        with box["cv"]:
            box["pending"] += 1
        self.tasks.put((fn, args, ev, box))

    @staticmethod
    def wait(box):
        with box["cv"]:
            box["cv"].wait_for(lambda: box["pending"] == 0)


_WORKERS = {}


# K window of the background GEMMs while an ID chain shares the GPU
# (vief_gemm_desc.kwin).  The chain's cluster kernels (sketch selection, QR
# panels) need whole SMs and wait for resident GEMM CTAs to retire; at K = 8192
# one 64 x 64 tile runs ~1 ms.  Measured at 1024^2 (compression stream / tail /
# step, ms): off 1686 / 204 / 1890; see DESIGN section 8.
_BG_KWIN = 1024


def _windowed(kwin, fn):
    """Worker task `fn` with _lib.GEMM_KWIN = kwin while it enqueues."""
    if not kwin:
        return fn

    def run(*args):
        old = _lib.GEMM_KWIN
        _lib.GEMM_KWIN = kwin
        try:
            return fn(*args)
        finally:
            _lib.GEMM_KWIN = old
    return run


def _up_level_on(stream, H, L, fd, phi, ups):
    """Worker task: the up sweep of level L on `stream`, after the side
    stream's inversion of L (the task runs on the worker right after it)."""
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        _sweep_up_level(H, L, fd, phi, ups)


def _ti_child_view(C):
    """The two children of a TI parent box, both the child level's one record
    (solver_compressed.py:548-552: factor_of(c) is the level's record)."""
    E2 = C.E[0:1].expand(2, -1, -1).contiguous()
    return _View(C, nb=2, k=C.k[:2], k_d=C.k_d[:2].contiguous(), E=E2, Gkeep=None)


def _ti_invert_F(inv, L, checks=None):
    """TI sharing: F^-1 of the level's first box only (every box is its
    translate); the parent's F is assembled from the child level's record."""
    H = inv.H
    V = _first_box(L, ("m", "m_d", "D", "B12", "B21"))
    lv1 = L.lv + 1
    swap = not L.leaf
    saved = H.levels[lv1] if swap else None
    if swap:
        H.levels[lv1] = _ti_child_view(saved)
    try:
        _invert_level_F(inv, V, checks)
    finally:
        if swap:
            H.levels[lv1] = saved
    for name in ("Finv", "rb"):
        if name in V.__dict__:
            setattr(L, name, V.__dict__[name])
    L._ti_view = V


def _ti_invert_rest(inv, L, checks=None):
    """W, G, E, C of the first box; the level then holds one shared record
    (L.ti: the sweeps read it with batch stride 0)."""
    V = L.__dict__.pop("_ti_view")
    if L.lv > 0:
        V.__dict__.update({a: getattr(L, a)[:1] for a in
                           ("k", "k_d", "perm_r", "perm_c", "Tr", "Tc", "nT_d")})
        _invert_level_rest(inv, V, checks)
        for name in ("E", "W", "C"):
            setattr(L, name, V.__dict__[name])
    L.ti = L.nb > 1


def _factorize_levels(H, inv, pad, main, side, third=None, solve=None):
    """Compression on this thread (main stream); the inversion work is
    enqueued on the side stream by a worker thread.  Enqueueing a large
    Gauss-Jordan inversion blocks the host for as long as the GPU runs it (the
    launch queue fills), and the ID loop synchronises with the host once per
    block, so a single host thread would serialise the two streams."""
    import threading
    checks = inv._checks = []
    dev_index = torch.cuda.current_device() if H.device.index is None else H.device.index
    w = _WORKERS.get(dev_index)
    if w is None or w.stream is not side:
        w = _WORKERS[dev_index] = _Worker(dev_index, side)
    box = {"pending": 0, "error": None, "cv": threading.Condition()}
    try:
        _mark("compress:start")
        for L in reversed(_real_levels(H)):
            _lib.prof_prefix(f"L{L.lv:02d}.")
            # F of this level needs only its D/B blocks and the children's E:
            # its inversion overlaps this level's IDs
            _compress_level_blocks(H, L)
            ev = torch.cuda.Event()
            ev.record(main)
            ti = bool(getattr(H, "ti_share", False))
            # work that runs next to an ID chain (this level's F^-1 next to this
            # level's IDs, the rest and the up sweep next to the parent level's)
            # issues its long-K GEMMs in K windows; level 1's rest, the root and
            # the down sweep have the GPU to themselves
            kw_rest = _BG_KWIN if L.lv >= 2 else 0
            w.submit(box, _windowed(_BG_KWIN, _ti_invert_F if ti else _invert_level_F),
                     (inv, L, checks), ev)
            _compress_level_id(H, L, pad, H.opts.seed)
            ev = torch.cuda.Event()
            ev.record(main)
            w.submit(box, _windowed(kw_rest, _ti_invert_rest if ti else _invert_level_rest),
                     (inv, L, checks), ev)
            if solve is not None:
                fd, _, phi, ups = solve
                w.submit(box, _windowed(kw_rest, _up_level_on), (third, H, L, fd, phi, ups), None)
            _mark(f"compress:{L.lv}")
            if box["error"] is not None:
                break
    finally:
        _Worker.wait(box)
    if box["error"] is not None:
        raise box["error"]


# ---------------------------------------------------------------------------
# solve sweeps

class _Split:
    """Layout marker: a complex right-hand side of a real system, solved as
    its real and imaginary parts stacked as 2r real right-hand sides."""

    def __init__(self, single, r):
        self.single, self.r = single, r


def _as_device_rhs(x, n, device, realified=False):
    """(N,) or (N, r) numpy/torch -> ((r, N') float64 device tensor, single).
    Realified (complex) systems interleave (Re, Im) per point: N' = 2N.  The
    result dtype follows np.result_type(spec.dtype, f.dtype) as in the
    reference (solver_dense.py:296): a complex f on a real system is solved
    as Re and Im (2r real columns) and returned complex."""
    if isinstance(x, torch.Tensor):
        cplx = x.is_complex()
        t = x.to(device=device, dtype=torch.complex128 if (realified or cplx) else _F64)
    else:
        arr = np.asarray(x)
        cplx = np.iscomplexobj(arr)
        dt = np.complex128 if (realified or cplx) else np.float64
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=dt)).to(device)
    single = t.dim() == 1
    t2 = t[:, None] if single else t
    if t2.dim() != 2 or t2.shape[0] != n:
        raise ValueError(f"rhs has shape {tuple(t.shape)}, expected ({n},) or ({n}, nrhs)")
    tt = t2.t().contiguous()
    if realified:
        tt = torch.view_as_real(tt).reshape(tt.shape[0], 2 * n)
    elif cplx:
        r = tt.shape[0]
        tt = torch.cat([tt.real, tt.imag], dim=0).contiguous()
        return tt, _Split(single, r)
    return tt, single


def _from_device(out, like, single, realified):
    """(r, N') device result -> the caller's layout/type (solver_dense.py:296-329)."""
    if isinstance(single, _Split):
        r = single.r
        out = torch.complex(out[:r], out[r:])
        single = single.single
    elif realified:
        out = torch.view_as_complex(out.reshape(out.shape[0], -1, 2).contiguous())
    res = out.t()
    if isinstance(like, torch.Tensor):
        res = res.to(like.device)
        return res[:, 0] if single else res
    arr = res.cpu().numpy()
    return arr[:, 0].copy() if single else np.ascontiguousarray(arr)


def _level_dn_idx(H, L):
    """Absolute offsets of each child's phi_dn slice in the parent's result
    buffer ([r, nb_p * mm_p] layout)."""
    if getattr(L, "dn_idx", None) is not None:
        return L.dn_idx
    P = H.levels[L.lv - 1]
    j = np.arange(L.nb)
    off = (j // 2) * P.mmax + np.where(j % 2 == 1, np.roll(L.k, 1), 0)
    t = np.arange(L.kmax)[None, :]
    idx = np.where(t < L.k[:, None], off[:, None] + t, 0)
    L.dn_idx = _dev_i32(idx, H.device)
    return L.dn_idx


def _fs(L, stride):
    """Batch stride of a level's factor arrays: 0 once the level shares one
    record (TI mode, share_level_records)."""
    return 0 if getattr(L, "ti", False) else stride


def share_level_records(inv):
    """TI mode (solver_compressed.py:33-37,548-552): with a-priori skeletons and
    a translation-invariant kernel every box of a level is a translate of the
    first, so its factors are the first box's; keep that record (F^-1, C, E, W)
    per level and let the sweeps read it with batch stride 0.  Factor memory
    drops from O(N log N) to one record per level.

    A level is shared only when its boxes really are translates: same
    rectangle size, same m and k (a ragged grid -- e.g. 49/56/64-point leaves
    -- or a support mask can make them differ).  Such a level keeps its
    per-box records, so the sweeps stay correct (the reference's shared
    record would fail with a shape mismatch there)."""
    for L in _real_levels(inv.H):
        if L.nb < 2 or not _level_is_uniform(L):
            continue
        for name in ("Finv", "C", "E", "W"):
            t = getattr(L, name, None)
            if t is not None:
                setattr(L, name, t[:1].clone())
        L.ti = True
    torch.cuda.empty_cache()


def _level_is_uniform(L):
    """Every box of the level has the first box's width/height, m and k."""
    r = np.asarray(L.rects)
    wh = np.stack([r[:, 1] - r[:, 0], r[:, 3] - r[:, 2]], 1)
    if not (wh == wh[0]).all() or not (np.asarray(L.m) == L.m[0]).all():
        return False
    k = getattr(L, "k", None)
    return k is None or bool((np.asarray(k) == k[0]).all())


def _mv(A, sA, lda, X, sx, ldx, Y, sy, ldy, M, K, Mb, Kb, nb, r, alpha, beta):
    """Y_b = alpha * A_b X_b + beta * Y_b for r right-hand sides."""
    if r == 1:
        _lib.gemv(A, X, Y, M=M, K=K, lda=lda, sA=sA, sx=sx, sy=sy, alpha=alpha, beta=beta,
                  batch=nb, Mb=Mb, Kb=Kb)
    else:
        _lib.gemm(A, X, Y, M=M, N=r, K=K, lda=lda, ldb=ldx, ldc=ldy, sA=sA, sB=sx, sC=sy,
                  alpha=alpha, beta=beta, batch=nb, Mb=Mb, Kb=Kb)


def _real_levels(H):
    """Levels this object factors (absent levels are None; a 'virtual' level
    only carries a sharded neighbour's interface data)."""
    return [L for L in H.levels if L is not None and not getattr(L, "virtual", False)]


def _sweep_up_level(H, L, fd, phi, ups, fac=None):
    """One level of the up sweep: phi = F^{-1} u, ups = C phi.  `fac`: the
    level's device factors when they are spilled to host memory."""
    Finv, Cf = ((L.Finv, getattr(L, "C", None)) if fac is None
                else (fac["Finv"], fac.get("C")))
    dev = H.device
    r, n = fd.shape
    nb, mm = L.nb, L.mmax
    ldv = nb * mm
    U = torch.zeros((r, ldv), dtype=_F64, device=dev)
    if L.leaf:
        _lib.gather_rows(fd, 0, n, L.rows, mm, U, mm, ldv, L.m_d, mm, None, r, nb)
    else:
        C = H.levels[L.lv + 1]
        _lib.gather_rows(ups[C.lv], 2 * C.kmax, C.nb * C.kmax, L.cat_idx, mm, U, mm, ldv,
                         L.m_d, mm, None, r, nb)
    if getattr(L, "hss", None) is not None:   # 1-D HSS blocks (compressed_store.py)
        from . import compressed_store
        compressed_store.sweep_up_level(H, L, U, phi, ups, r)
        return
    Phi = torch.zeros((r, ldv), dtype=_F64, device=dev)
    _apply_Finv(L, Finv, U, Phi, r, 0.0)
    if getattr(L, "refine", False):
        _refine_box_solve(H, L, Finv, U, Phi, r)
        if L.lv > 0:
            phi[("u", L.lv)] = U      # the down sweep refines against the same u
    del U
    phi[L.lv] = Phi
    if L.lv == 0:
        return
    kk = L.kmax
    Ups = torch.zeros((r, nb * kk), dtype=_F64, device=dev)
    _mv(Cf, _fs(L, mm * kk), kk, Phi, mm, ldv, Ups, kk, nb * kk, kk, mm, L.k_d, L.m_d, nb, r,
        1.0, 0.0)
    ups[L.lv] = Ups


def _apply_Finv(L, Finv, U, Out, r, beta):
    """Out = F^{-1} U + beta Out for the level's boxes (vectors: (r, nb*mm))."""
    nb, mm = L.nb, L.mmax
    ldv = nb * mm
    if getattr(L, "rb", None) is not None:
        if beta == 0.0:
            _root_block_solve(L, U, ldv, r, Out, ldv)
        else:
            T = torch.zeros_like(Out)
            _root_block_solve(L, U, ldv, r, T, ldv)
            Out.add_(T)
    else:
        _mv(Finv, _fs(L, mm * mm), mm, U, mm, ldv, Out, mm, ldv, mm, mm, L.m_d, L.m_d, nb, r,
            1.0, beta)


def _level_Fmat(H, L):
    """F of a refined level (cached; the leaves' D is used as is)."""
    if L.leaf:
        return L.D
    F = getattr(L, "_Fmat", None)
    if F is None:
        F = L._Fmat = _assemble_F(H, L)
    return F


def _refine_box_solve(H, L, Finv, U, X, r):
    """X += F^{-1} (U - F X), _REFINE_STEPS times (iterative refinement of
    the level's box solves against F; see _REFINE_COND)."""
    nb, mm = L.nb, L.mmax
    ldv = nb * mm
    F = _level_Fmat(H, L)
    for _ in range(_REFINE_STEPS):
        R = U.clone()
        _mv(F, mm * mm, mm, X, mm, ldv, R, mm, ldv, mm, mm, L.m_d, L.m_d, nb, r, -1.0, 1.0)
        _apply_Finv(L, Finv, R, X, r, 1.0)


def _apply_L(H, L, D, r):
    """Z = L D per box (interp_L: D to perm_r[:k], Tr^T D to perm_r[k:],
    solver_dense.py:75-80); D: (r, nb*kk) -> Z: (r, nb*mm)."""
    dev = H.device
    nb, mm, kk = L.nb, L.mmax, L.kmax
    ldv = nb * mm
    Tmp = torch.zeros((r, ldv), dtype=_F64, device=dev)
    _lib.copy2d(D, kk, nb * kk, Tmp, mm, ldv, L.k_d, kk, None, r, nb)
    base = np.arange(nb, dtype=np.int64) * mm + L.k.astype(np.int64)
    _lib.gemm(L.Tr, D, None, M=L.ntmax, N=r, K=kk, lda=kk, ldb=nb * kk, ldc=ldv,
              sA=0 if getattr(L, "ti", False) else L.ntmax * kk, sB=kk, tA=1, alpha=1.0,
              beta=0.0, batch=nb, Mb=L.nT_d, Kb=L.k_d, Cptr=_ptrs(Tmp, base, dev))
    Z = torch.zeros((r, ldv), dtype=_F64, device=dev)
    _lib.scatter_rows(Tmp, mm, ldv, L.perm_r, mm, Z, mm, ldv, L.m_d, mm, None, r, nb)
    return Z


def _sweep_up(H, fd, phi, ups):
    """Up sweep (solver_dense.py:303-310): phi = F^{-1} u, ups = C phi = E R phi.
    ups of a virtual child level must be present in `ups` beforehand."""
    order = list(reversed(_real_levels(H)))
    pf = _Prefetch(H, order, ("Finv", "C"))
    for i, L in enumerate(order):
        _sweep_up_level(H, L, fd, phi, ups, pf.get(i))
        if L.lv == 0:
            break


def _phi_dn(H, L, phi, r):
    """phi_dn of level L's boxes: slices of the parent level's result."""
    P = H.levels[L.lv - 1]
    kk = L.kmax
    PD = torch.zeros((r, L.nb * kk), dtype=_F64, device=H.device)
    _lib.gather_rows(phi[P.lv], 0, P.nb * P.mmax, _level_dn_idx(H, L), kk, PD, kk, L.nb * kk,
                     L.k_d, kk, None, r, L.nb)
    return PD


def _sweep_down(H, phi, ups, out, pd_top=None):
    """Down sweep (solver_dense.py:312-328): res = phi - W (ups - E phi_dn),
    leaves scattered into `out`.  `pd_top` supplies phi_dn of the coarsest
    level when its parent is factored elsewhere (sharded subtree)."""
    r, n = out.shape
    order = _real_levels(H)
    pf = _Prefetch(H, order, ("E", "W"))
    for i, L in enumerate(order):
        fac = pf.get(i)
        Ef, Wf = ((getattr(L, "E", None), getattr(L, "W", None)) if fac is None
                  else (fac.get("E"), fac.get("W")))
        nb, mm = L.nb, L.mmax
        ldv = nb * mm
        Phi = phi[L.lv]
        if getattr(L, "hss", None) is not None:
            from . import compressed_store
            par = H.levels[L.lv - 1]
            PD = pd_top if par is None else _phi_dn(H, L, phi, r)
            Phi = compressed_store.sweep_down_level(H, L, PD, phi, ups, r)
            del PD
        elif L.lv > 0:
            kk = L.kmax
            par = H.levels[L.lv - 1]
            PD = pd_top if par is None else _phi_dn(H, L, phi, r)
            Ups = ups[L.lv]
            _mv(Ef, _fs(L, kk * kk), kk, PD, kk, nb * kk, Ups, kk, nb * kk, kk, kk, L.k_d, L.k_d, nb, r,
                -1.0, 1.0)
            _mv(Wf, _fs(L, kk * mm), mm, Ups, kk, nb * kk, Phi, mm, ldv, mm, kk, L.m_d, L.k_d, nb, r,
                -1.0, 1.0)
            del PD
        if L.lv > 0 and getattr(L, "refine", False):  # res = F^{-1} (u - L (ups - E phi_dn))
            U = phi.pop(("u", L.lv)) - _apply_L(H, L, Ups, r)
            Finv = L.Finv if L.Finv.is_cuda else L.Finv.to(H.device)
            _refine_box_solve(H, L, Finv, U, Phi, r)
            del U
        if L.leaf:
            _lib.scatter_rows(Phi, mm, ldv, L.rows, mm, out, 0, n, L.m_d, mm, None, r, nb)


def _apply_device(inv, fd):
    """fd: (r, N) device tensor -> (r, N) solution (device)."""
    H = inv.H
    phi, ups = {}, {}
    _sweep_up(H, fd, phi, ups)
    out = torch.zeros_like(fd)
    _sweep_down(H, phi, ups, out)
    return out


def _apply(inv, f):
    H = inv.H
    with _host_quiet():
        fd, single = _as_device_rhs(f, H.grid.n, H.device, H.realified)
        if fd.shape[0] == 0:  # no right-hand sides
            return _from_device(fd, f, single, H.realified)
        return _from_device(_apply_device(inv, fd), f, single, H.realified)


def apply_inverse_dense_block(inv, f):
    return inv.apply(f)


# ---------------------------------------------------------------------------
# forward operator (solver_dense.py:143-178)

def _matvec_device(H, xd):
    if H.sharded:
        raise NotImplementedError("matvec of a sharded (distributed) compression")
    dev = H.device
    r, n = xd.shape
    levels = H.levels
    phi = {}
    for L in reversed(levels):
        if L.lv == 0:
            break
        nb, mm, kk = L.nb, L.mmax, L.kmax
        ldv = nb * mm
        Wv = torch.zeros((r, ldv), dtype=_F64, device=dev)
        if L.leaf:
            _lib.gather_rows(xd, 0, n, L.rows, mm, Wv, mm, ldv, L.m_d, mm, None, r, nb)
        else:
            C = levels[L.lv + 1]
            _lib.gather_rows(phi[C.lv], 2 * C.kmax, C.nb * C.kmax, L.cat_idx, mm, Wv, mm, ldv,
                             L.m_d, mm, None, r, nb)
        # phi = R w = wp[:k] + Tc wp[k:],  wp = w[perm_c]
        Wp = torch.zeros((r, ldv), dtype=_F64, device=dev)
        _lib.gather_rows(Wv, mm, ldv, L.perm_c, mm, Wp, mm, ldv, L.m_d, mm, None, r, nb)
        Ph = torch.zeros((r, nb * kk), dtype=_F64, device=dev)
        _lib.copy2d(Wp, mm, ldv, Ph, kk, nb * kk, L.k_d, kk, None, r, nb)
        k = L.k.astype(np.int64)
        base = np.arange(nb, dtype=np.int64) * mm
        _gemm_ptr_rhs(L.Tc, L.ntmax * kk, kk, Wp, base + k, ldv, Ph, kk, nb * kk,
                      kk, L.ntmax, L.k_d, L.nT_d, nb, r, 1.0, 1.0, dev)
        phi[L.lv] = Ph
    out = torch.zeros((r, n), dtype=_F64, device=dev)
    wdn = {}
    for L in levels:
        nb, mm = L.nb, L.mmax
        ldv = nb * mm
        t = None
        if L.lv > 0:
            # t = L w_in : tp = [w; Tr^T w] scattered by perm_r
            kk = L.kmax
            win = wdn[L.lv]
            tp = torch.zeros((r, ldv), dtype=_F64, device=dev)
            _lib.copy2d(win, kk, nb * kk, tp, mm, ldv, L.k_d, kk, None, r, nb)
            k = L.k.astype(np.int64)
            base = np.arange(nb, dtype=np.int64) * mm
            # tp[k:m] = Tr^T w   (Tr stored [item, col, row]: Tr^T is (m-k) x k, ld kmax, trans)
            _gemm_ptr_out(L.Tr, L.ntmax * kk, kk, win, kk, nb * kk, tp, base + k, ldv,
                          L.ntmax, kk, L.nT_d, L.k_d, nb, r, dev)
            t = torch.zeros((r, ldv), dtype=_F64, device=dev)
            _lib.scatter_rows(tp, mm, ldv, L.perm_r, mm, t, mm, ldv, L.m_d, mm, None, r, nb)
        if L.leaf:
            y = torch.zeros((r, ldv), dtype=_F64, device=dev)
            xin = torch.zeros((r, ldv), dtype=_F64, device=dev)
            _lib.gather_rows(xd, 0, n, L.rows, mm, xin, mm, ldv, L.m_d, mm, None, r, nb)
            _mv(L.D, mm * mm, mm, xin, mm, ldv, y, mm, ldv, mm, mm, L.m_d, L.m_d, nb, r, 1.0, 0.0)
            if t is not None:
                y += t
            _lib.scatter_rows(y, mm, ldv, L.rows, mm, out, 0, n, L.m_d, mm, None, r, nb)
            continue
        # children: w1 = B12 phi[c2] + t[:k1], w2 = B21 phi[c1] + t[k1:]
        C = levels[L.lv + 1]
        kc = C.kmax
        wc = torch.zeros((r, C.nb * kc), dtype=_F64, device=dev)
        k1d, k2d = C.k_d[0::2].contiguous(), C.k_d[1::2].contiguous()
        ph = phi[C.lv]
        # wc[2j] = B12_j phi[2j+1] ; wc[2j+1] = B21_j phi[2j]
        _mv(L.B12, kc * kc, kc, _lib.ptr(ph) + 8 * kc, 2 * kc, C.nb * kc, wc, 2 * kc, C.nb * kc,
            kc, kc, k1d, k2d, nb, r, 1.0, 0.0)
        _mv(L.B21, kc * kc, kc, ph, 2 * kc, C.nb * kc, _lib.ptr(wc) + 8 * kc, 2 * kc, C.nb * kc,
            kc, kc, k2d, k1d, nb, r, 1.0, 0.0)
        if t is not None:
            # add t (parent order: [k1 | k2]) into the children slices
            _scatter_add_children(t, L, C, wc, r, dev)
        wdn[C.lv] = wc
    return out


def _gemm_ptr_rhs(A, sA, lda, X, xoff, ldx, Y, sy, ldy, M, K, Mb, Kb, nb, r, alpha, beta, dev):
    """Y_b += A_b X[xoff_b : xoff_b + K] for r right-hand sides (pointer arrays)."""
    xp = _ptrs(X, xoff, dev)
    if r == 1:
        _lib.gemv(A, None, Y, M=M, K=K, lda=lda, sA=sA, sy=sy, alpha=alpha, beta=beta,
                  batch=nb, Mb=Mb, Kb=Kb, xptr=xp)
    else:
        _lib.gemm(A, None, Y, M=M, N=r, K=K, lda=lda, ldb=ldx, ldc=ldy, sA=sA, sC=sy,
                  alpha=alpha, beta=beta, batch=nb, Mb=Mb, Kb=Kb, Bptr=xp)


def _gemm_ptr_out(A, sA, lda, X, sx, ldx, Y, yoff, ldy, M, K, Mb, Kb, nb, r, dev):
    """Y[yoff_b : yoff_b + M] = op(A_b)^T X_b where A_b is stored K x M (trans)."""
    yp = _ptrs(Y, yoff, dev)
    if r == 1:
        _lib.gemv(A, X, None, M=M, K=K, lda=lda, sA=sA, sx=sx, tA=1, alpha=1.0, beta=0.0,
                  batch=nb, Mb=Mb, Kb=Kb, yptr=yp)
    else:
        _lib.gemm(A, X, None, M=M, N=r, K=K, lda=lda, ldb=ldx, ldc=ldy, sA=sA, sB=sx, tA=1,
                  alpha=1.0, beta=0.0, batch=nb, Mb=Mb, Kb=Kb, Cptr=yp)


def _scatter_add_children(t, L, C, wc, r, dev):
    """wc[child slice] += t[parent rows] with parent rows = [k1 | k2]."""
    if getattr(L, "_child_scatter", None) is None:
        # absolute destination offset in wc for parent row i of box j
        k1, k2 = C.k[0::2].astype(np.int64), C.k[1::2].astype(np.int64)
        j = np.arange(L.nb)[:, None]
        i = np.arange(L.mmax)[None, :]
        dst = np.where(i < k1[:, None], (2 * j) * C.kmax + i, (2 * j + 1) * C.kmax + i - k1[:, None])
        dst = np.where(i < (k1 + k2)[:, None], dst, 0)
        src = j * L.mmax + i
        L._child_scatter = (_dev_i32(dst, dev), _dev_i32(src, dev))
    dst, src = L._child_scatter
    tmp = torch.zeros_like(wc)
    # gather t rows into child layout then add
    _lib.scatter_rows(t, L.mmax, L.nb * L.mmax, dst, L.mmax, tmp, 0, C.nb * C.kmax, L.m_d,
                      L.mmax, None, r, L.nb)
    wc += tmp


def _matvec(H, x):
    xd, single = _as_device_rhs(x, H.grid.n, H.device, H.realified)
    if xd.shape[0] == 0:
        return _from_device(xd, x, single, H.realified)
    return _from_device(_matvec_device(H, xd), x, single, H.realified)


def hss_matvec(H, x):
    return H.matvec(x)
