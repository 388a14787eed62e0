"""Batched 1-D HSS storage of the compressed path's large factor blocks.

The reference keeps the F^-1 and E blocks of boxes with more than `k_cut`
skeleton points in a 1-D HSS form over the skeleton's curve ordering
(`hss1d/core.py` Hss1dMatrix: leaf diagonal blocks, nested interpolation
blocks, sibling blocks; `hss1d/build.py:51-191` compress_from_entries;
`hss1d/ops.py` matvec), one Python object per box.  Here a whole quadtree
level is one batch: `nb` matrices of the same size n share one interval tree
(`hss1d/core.py:52-71` build_interval_tree: halving, with a forced cut at the
skeleton / residual boundary), and every tree level of every matrix is one
item of a batched kernel call:

* build (`compress`): level by level from the leaves, the row and the column
  ID of every node's off-diagonal block row / column (candidates: the node's
  points at a leaf, the children's skeletons above; ranks of the two IDs
  coupled per node as in the reference) run as ONE vief_id_batched call per
  tree level; sibling blocks are sub-blocks of the matrix at the skeletons;
* apply (`matvec`): up sweep x^ = V^T x, sibling products, down sweep
  y^ = U y^_parent, leaf blocks -- one or two batched GEMMs (GEMVs for a
  single vector) per tree level, all items of all matrices at once.

Layout: item (matrix b, node i) of tree level l has index b * 2^l + i.  A
parent's candidate list is its two children's skeleton slots, each padded to
the child level's largest rank (zero columns in the ID input, zero rows in
U / V), so the children's coefficient vectors are the parent's input as they
lie in memory: no per-item pointer arithmetic above the leaves.

The matrices are given dense (the factorization forms F^-1 and E with batched
Gauss-Jordan / GEMMs, which is what the B200 is fast at) and are compressed
for storage; the reference builds them matrix-free (`solver_compressed.py:
313-424`) because dense blocks are what it cannot afford.  Everything numeric
runs in the library's kernels (ID, GEMM); torch indexing only gathers
sub-blocks.
"""

import numpy as np
import torch

from . import _lib

_F64 = torch.float64


def interval_tree(n, leaf_size, align=None):
    """Perfect binary tree of index intervals over [0, n): `depth` levels below
    the root, level l holding 2^l intervals (lo, hi) in order.  Intervals are
    halved (ceil first, hss1d/core.py:52-71); `align` (0 < align < n) forces the
    root cut there.  The depth is the smallest for which every leaf has at most
    leaf_size points."""
    levels = [np.array([[0, n]], dtype=np.int64)]
    while (levels[-1][:, 1] - levels[-1][:, 0]).max() > leaf_size or (
            align and len(levels) == 1 and 0 < align < n):
        cur = levels[-1]
        mid = cur[:, 0] + (cur[:, 1] - cur[:, 0] + 1) // 2
        if len(levels) == 1 and align and 0 < align < n:
            mid = np.array([align], dtype=np.int64)
        nxt = np.empty((2 * len(cur), 2), dtype=np.int64)
        nxt[0::2, 0], nxt[0::2, 1] = cur[:, 0], mid
        nxt[1::2, 0], nxt[1::2, 1] = mid, cur[:, 1]
        levels.append(nxt)
    return levels


def _i32(a, dev):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)


def _mm(A, sA, lda, tA, X, sx, ldx, Y, sy, ldy, M, K, batch, r, alpha=1.0, beta=0.0, Mb=None,
        Kb=None, xptr=None, yptr=None):
    """Y_b = alpha op(A_b) X_b + beta Y_b for r right-hand sides (vectors are
    (r, ld) row blocks: column-major M x r with leading dimension ld)."""
    if batch <= 0 or M <= 0:
        return
    if r == 1:
        _lib.gemv(A, None if xptr is not None else X, None if yptr is not None else Y, M=M, K=K,
                  lda=lda, sA=sA, sx=sx, sy=sy, tA=tA, alpha=alpha, beta=beta, batch=batch, Mb=Mb,
                  Kb=Kb, xptr=xptr, yptr=yptr)
    else:
        _lib.gemm(A, None if xptr is not None else X, None if yptr is not None else Y, M=M, N=r,
                  K=K, lda=lda, ldb=ldx, ldc=ldy, sA=sA, sB=sx, sC=sy, tA=tA, alpha=alpha,
                  beta=beta, batch=batch, Mb=Mb, Kb=Kb, Bptr=xptr, Cptr=yptr)


class _HLevel:
    """Generators of one tree level (all matrices): U, V (cnt, kmax, m) stored
    column-major m x k per item; k (cnt) ranks; B12/B21 of the level's nodes'
    CHILDREN (cnt, kc, kc); leaves: D (cnt, ms, ms)."""
    __slots__ = ("cnt", "m", "kmax", "k", "k_d", "U", "V", "B12", "B21", "D", "size_d", "off")


class Hss1dBatch:
    """`nb` n x n matrices in 1-D HSS form (see the module docstring)."""

    def __init__(self, nb, n, levels, dev):
        self.nb, self.n, self.dev = nb, n, dev
        self.tree = levels
        self.depth = len(levels) - 1
        self.lv = [None] * (self.depth + 1)
        self.dense = None          # depth 0: the matrices themselves

    # -- construction ------------------------------------------------------
    @staticmethod
    def from_dense(Ad, n):
        """The matrices kept as they are (a depth-0 tree: one dense block each)."""
        H = Hss1dBatch(Ad.shape[0], n, [np.array([[0, n]], dtype=np.int64)], Ad.device)
        H.dense = Ad[:, :n, :n].contiguous()
        return H

    @staticmethod
    def compress(Ad, n, eps, leaf_size=32, align=None, seed=0, max_items=32768):
        """Ad: (nb, ld, ld) device tensor, item b column-major (Ad[b, c, r] =
        A_b(r, c)), the leading n x n part is used.  `eps`: relative ID
        tolerance of every off-diagonal block row / column."""
        from . import solver_dense as sd
        dev = Ad.device
        nb = Ad.shape[0]
        tree = interval_tree(n, leaf_size, align)
        H = Hss1dBatch(nb, n, tree, dev)
        D = H.depth
        if D == 0:
            H.dense = Ad[:, :n, :n].contiguous()
            return H
        bidx = torch.arange(nb, device=dev)
        sib = {}
        rsk = csk = None           # (nb, nodes, kmax) skeleton positions of the level below
        kprev = None               # (nb, nodes) ranks of the level below
        for l in range(D, 0, -1):
            iv = tree[l]
            nodes = len(iv)
            sizes = iv[:, 1] - iv[:, 0]
            L = H.lv[l] = _HLevel()
            L.cnt = nb * nodes
            if l == D:             # candidates: the node's own points
                m = int(sizes.max())
                j = np.arange(m)[None, :]
                cand = torch.as_tensor(np.clip(np.minimum(iv[:, :1] + j, iv[:, 1:] - 1), 0, n - 1),
                                       device=dev)
                cmask = torch.as_tensor(j < sizes[:, None], device=dev)
                candR = candC = cand[None].expand(nb, nodes, m)
                maskR = maskC = cmask[None].expand(nb, nodes, m)
            else:                  # the children's skeleton slots (padded to their kmax)
                kc = rsk.shape[2]
                m = 2 * kc
                candR = rsk.reshape(nb, nodes, m)
                candC = csk.reshape(nb, nodes, m)
                live = (torch.arange(kc, device=dev)[None, None, :] < kprev[:, :, None])
                maskR = maskC = live.reshape(nb, nodes, m)
            L.m = m
            # complement of every node's interval (padded to the longest)
            pmax = int((n - sizes).max())
            ldA = pmax + (pmax & 1)
            comp = np.zeros((nodes, pmax), dtype=np.int64)
            cval = np.zeros((nodes, pmax), dtype=bool)
            for i, (lo, hi) in enumerate(iv):
                p = n - (hi - lo)
                comp[i, :lo] = np.arange(lo)
                comp[i, lo:p] = np.arange(hi, n)
                cval[i, :p] = True
            comp_d = torch.as_tensor(comp, device=dev)
            cval_d = torch.as_tensor(cval, device=dev)
            pv_node = (n - sizes).astype(np.int32)
            # boxes per ID call: item count and workspace bounds
            per_box = 2 * nodes
            chunk = max(1, min(nb, max_items // per_box, (1 << 27) // max(1, per_box * m * ldA)))
            ks, perms_r, perms_c, Ts_r, Ts_c = [], [], [], [], []
            for b0 in range(0, nb, chunk):
                b1 = min(nb, b0 + chunk)
                nbc = b1 - b0
                cnt2 = 2 * nbc * nodes
                X = torch.zeros((nbc, nodes, 2, m, ldA), dtype=_F64, device=dev)
                bb = bidx[b0:b1, None, None, None]
                cR = candR[b0:b1, :, :, None]
                cC = candC[b0:b1, :, :, None]
                cp = comp_d[None, :, None, :]
                msk = cval_d[None, :, None, :]
                # row ID item: columns = candidate rows, X[j, t] = A(cand[j], comp[t])
                X[:, :, 0, :, :pmax] = Ad[bb, cp, cR] * (maskR[b0:b1, :, :, None] & msk)
                # column ID item: X[j, t] = A(comp[t], cand[j])
                X[:, :, 1, :, :pmax] = Ad[bb, cC, cp] * (maskC[b0:b1, :, :, None] & msk)
                pv = _i32(np.repeat(np.tile(pv_node, nbc), 2), dev)
                mv = torch.full((cnt2,), m, dtype=torch.int32, device=dev)
                rank = torch.zeros(cnt2, dtype=torch.int32, device=dev)
                perm = torch.zeros((cnt2, m), dtype=torch.int32, device=dev)
                T = torch.zeros((cnt2, m, m), dtype=_F64, device=dev)
                sd._id_batched(dev, X, m * ldA, ldA, pv, mv, pmax, m, cnt2, 2, float(eps), rank,
                               perm, T, int(seed) * 7919 + l * 131 + b0, 0)
                del X
                ks.append(rank[0::2].clone())
                perms_r.append(perm[0::2].long())
                perms_c.append(perm[1::2].long())
                Ts_r.append(T[0::2])
                Ts_c.append(T[1::2])
                del T
            k = torch.cat(ks)
            kmax = max(int(k.max()), 1)
            L.kmax, L.k_d = kmax, k.contiguous()
            L.k = k.cpu().numpy()
            L.U = _interp_store(torch.cat(perms_r), torch.cat(Ts_r), k, kmax, m)
            L.V = _interp_store(torch.cat(perms_c), torch.cat(Ts_c), k, kmax, m)
            del Ts_r, Ts_c
            # skeleton positions (padded with the node's first candidate; masked by k)
            pr = torch.cat(perms_r)[:, :kmax]
            pc = torch.cat(perms_c)[:, :kmax]
            rsk = candR.reshape(L.cnt, m).gather(1, pr).reshape(nb, nodes, kmax)
            csk = candC.reshape(L.cnt, m).gather(1, pc).reshape(nb, nodes, kmax)
            kprev = k.reshape(nb, nodes)
            # sibling blocks of the parents (level l - 1): sub-blocks at the skeletons
            live = torch.arange(kmax, device=dev)[None, None, :] < kprev[:, :, None]
            r1, r2 = rsk[:, 0::2], rsk[:, 1::2]          # (nb, nodes/2, kmax)
            c1, c2 = csk[:, 0::2], csk[:, 1::2]
            l1, l2 = live[:, 0::2], live[:, 1::2]
            bb = bidx[:, None, None, None]
            # B12[c, r] = A(rsk1[r], csk2[c]);  B21[c, r] = A(rsk2[r], csk1[c])
            B12 = Ad[bb, c2[:, :, :, None], r1[:, :, None, :]] * (l2[:, :, :, None] & l1[:, :, None, :])
            B21 = Ad[bb, c1[:, :, :, None], r2[:, :, None, :]] * (l1[:, :, :, None] & l2[:, :, None, :])
            sib[l - 1] = (B12.reshape(-1, kmax, kmax).contiguous(),
                          B21.reshape(-1, kmax, kmax).contiguous())
            L.D = L.size_d = L.off = None
            if l == D:             # leaf diagonal blocks
                ms = m
                j = np.arange(ms)
                pos = torch.as_tensor(np.clip(iv[:, :1] + j[None, :], 0, n - 1), device=dev)
                val = torch.as_tensor(j[None, :] < sizes[:, None], device=dev)
                Dd = Ad[bidx[:, None, None, None], pos[None, :, :, None], pos[None, :, None, :]]
                Dd = Dd * (val[None, :, :, None] & val[None, :, None, :])
                L.D = Dd.reshape(-1, ms, ms).contiguous()
                L.size_d = _i32(np.tile(sizes, nb), dev)
                L.off = (np.arange(nb, dtype=np.int64)[:, None] * n + iv[None, :, 0]).reshape(-1)
        R = H.lv[0] = _HLevel()   # the root only holds its children's sibling blocks
        R.cnt, R.m, R.kmax, R.k, R.k_d, R.U, R.V, R.D = nb, 2 * H.lv[1].kmax, 0, None, None, None, None, None
        for l in range(0, D + 1):
            H.lv[l].B12, H.lv[l].B21 = sib.get(l, (None, None))
        return H

    # -- queries -------------------------------------------------------------
    def nbytes(self):
        """Bytes of the stored generators (as allocated, padding included)."""
        if self.dense is not None:
            return self.dense.numel() * 8
        tot = 0
        for L in self.lv:
            for name in ("U", "V", "B12", "B21", "D"):
                t = getattr(L, name, None)
                if t is not None:
                    tot += t.numel() * t.element_size()
        return tot

    def max_rank(self):
        return max((int(L.kmax) for L in self.lv[1:]), default=0)

    # -- apply ---------------------------------------------------------------
    def matvec(self, X, Y=None, alpha=1.0, beta=0.0, trans=False):
        """Y = alpha A X + beta Y (or A^T X) for all matrices: X, Y are (r, nb * n)
        device tensors (matrix b's vector at columns b*n .. b*n+n-1)."""
        from .solver_dense import _ptrs
        nb, n, dev = self.nb, self.n, self.dev
        r = X.shape[0]
        ldx = X.shape[1]
        if Y is None:
            Y = torch.zeros_like(X)
            beta = 0.0
        if self.dense is not None:
            _mm(self.dense, n * n, n, 1 if trans else 0, X, n, ldx, Y, n, Y.shape[1], n, n, nb, r,
                alpha, beta)
            return Y
        D = self.depth
        lv = self.lv
        # A^T: the roles of (U, V) and of (B12, B21) swap, D is applied transposed
        Vn, Un = ("U", "V") if trans else ("V", "U")
        xh = [None] * (D + 1)
        L = lv[D]
        ms = L.D.shape[1]
        xp = _ptrs(X, L.off, dev)
        xh[D] = torch.zeros((r, L.cnt * L.kmax), dtype=_F64, device=dev)
        _mm(getattr(L, Vn), L.kmax * L.m, L.m, 1, None, 0, ldx, xh[D], L.kmax, L.cnt * L.kmax,
            L.kmax, L.m, L.cnt, r, Mb=L.k_d, Kb=L.size_d, xptr=xp)
        for l in range(D - 1, 0, -1):
            L, C = lv[l], lv[l + 1]
            xh[l] = torch.zeros((r, L.cnt * L.kmax), dtype=_F64, device=dev)
            _mm(getattr(L, Vn), L.kmax * L.m, L.m, 1, xh[l + 1], L.m, C.cnt * C.kmax, xh[l], L.kmax,
                L.cnt * L.kmax, L.kmax, L.m, L.cnt, r, Mb=L.k_d)
        yh = None
        for l in range(0, D):
            L, C = lv[l], lv[l + 1]
            kc = C.kmax
            yc = torch.zeros((r, C.cnt * kc), dtype=_F64, device=dev)
            if l >= 1:
                _mm(getattr(L, Un), L.kmax * L.m, L.m, 0, yh, L.kmax, L.cnt * L.kmax, yc, 2 * kc,
                    C.cnt * kc, 2 * kc, L.kmax, L.cnt, r, Kb=L.k_d)
            b12, b21, tb = (L.B21, L.B12, 1) if trans else (L.B12, L.B21, 0)
            x1, x2 = _lib.ptr(xh[l + 1]), _lib.ptr(xh[l + 1]) + 8 * kc
            y1, y2 = _lib.ptr(yc), _lib.ptr(yc) + 8 * kc
            npar = C.cnt // 2
            _mm(b12, kc * kc, kc, tb, x2, 2 * kc, C.cnt * kc, y1, 2 * kc, C.cnt * kc, kc, kc, npar, r,
                1.0, 1.0)
            _mm(b21, kc * kc, kc, tb, x1, 2 * kc, C.cnt * kc, y2, 2 * kc, C.cnt * kc, kc, kc, npar, r,
                1.0, 1.0)
            yh = yc
        L = lv[D]
        yp = _ptrs(Y, L.off, dev)
        ldy = Y.shape[1]
        _mm(L.D, ms * ms, ms, 1 if trans else 0, None, 0, ldx, None, 0, ldy, ms, ms, L.cnt, r,
            alpha, beta, Mb=L.size_d, Kb=L.size_d, xptr=xp, yptr=yp)
        _mm(getattr(L, Un), L.kmax * L.m, L.m, 0, yh, L.kmax, L.cnt * L.kmax, None, 0, ldy, L.m,
            L.kmax, L.cnt, r, alpha, 1.0, Mb=L.size_d, Kb=L.k_d, yptr=yp)
        return Y

    def to_dense(self):
        """(nb, n, n) column-major dense matrices (tests, small n)."""
        nb, n = self.nb, self.n
        eye = torch.eye(n, dtype=_F64, device=self.dev).repeat(1, nb).contiguous()  # (n, nb*n)
        Y = self.matvec(eye)                    # row j: column j of every A_b
        return Y.reshape(n, nb, n).permute(1, 0, 2).contiguous()


def _interp_store(perm, T, k, kmax, m):
    """Dense interpolation blocks from the ID output: item = P [I_k ; T^T]
    (m x k), stored (cnt, kmax, m) column-major.  perm (cnt, m) pivot order,
    T (cnt, m, m) with T[it, c, r] = T(r, c) (k x (m - k)), k (cnt)."""
    cnt = perm.shape[0]
    dev = perm.device
    q = torch.arange(m, device=dev)[None, :]                 # pivot-order position
    kk = k.long()[:, None]
    # W[it, j, q]: row j of [I | T] in pivot order
    idx = (q - kk).clamp_(0, m - 1)                          # column of T for q >= k
    G = T.gather(1, idx[:, :, None].expand(cnt, m, kmax))    # G[it, q, j] = T(j, q - k)
    jj = torch.arange(kmax, device=dev)[None, None, :]
    G = torch.where(q[:, :, None] >= kk[:, :, None], G, (q[:, :, None] == jj).to(_F64))
    G = G * (jj < kk[:, :, None])                            # rows j >= k unused
    W = G.transpose(1, 2).contiguous()                       # (cnt, kmax, m) in pivot order
    out = torch.zeros((cnt, kmax, m), dtype=_F64, device=dev)
    out.scatter_(2, perm[:, None, :].expand(cnt, kmax, m), W)
    return out
