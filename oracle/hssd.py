"""CPU ORACLE — test infrastructure only, never the product path.

A NumPy/SciPy restatement of the reference's dense-block recursive
skeletonization (HSS-D) path: the `vief` package under
/root/reference/pkg/src/vief.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s CPU-baseline / `--impl reference` legs may import this module.

The restatement is procedural (arrays + dicts keyed by box id) rather than the
reference's class layout; every function names the reference lines it follows.
The dense linear algebra the reference delegates to LAPACK is delegated to the
same third-party routines here:

    scipy.linalg.qr(pivoting=True)  -> LAPACK ?geqp3      (dense_core.py:80)
    scipy.linalg.solve_triangular   -> LAPACK ?trtrs/?trsm (dense_core.py:98)
    scipy.linalg.lu_factor/lu_solve -> LAPACK ?getrf/?getrs (dense_core.py:224,
                                                          solver_dense.py:309-367)

(scipy-openblas 0.3.30 in this image; the reference pins none,
pyproject.toml:10-13).  Parity pins: tests/golden/*.npz, produced by
tests/golden/make_golden.py from the reference itself.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field

import numpy as np
import scipy.linalg as sla

TWO_PI = 2.0 * np.pi
# closed-form mean of log|y| over the unit-side square cell: log h + C_CELL
C_CELL = -1.5 + np.pi / 4.0 - 0.5 * math.log(2.0)
LOG_H2_CONST = -1.3105329258137919          # _quad_constants.py:8


# ---------------------------------------------------------------------------
# grid + fields (kernels.py:34-63, 143-169)

def lattice(n_side):
    """(int coords (N,2), points (N,2), h) of the cell-centred grid on [-1,1]^2;
    linear index iy*n+ix (kernels.py:145,157-166)."""
    lin = np.arange(n_side * n_side)
    ic = np.column_stack([lin % n_side, lin // n_side]).astype(np.int64)
    h = 2.0 / n_side
    return ic, -1.0 + (ic + 0.5) * h, h


def field_values(name, params, xy):
    """Field presets (kernels.py:41-57) plus the harness bump used for the
    BASELINE configs: 1 + 0.5 exp(-|x|^2/w) * scale-free, times `scale`."""
    x, y = xy[..., 0], xy[..., 1]
    p = dict(params)
    if name == "one":
        return np.ones_like(x)
    if name == "gaussian_bump":
        return 1.0 + 0.5 * np.exp(-((x - 0.3) ** 2) - (y - 0.6) ** 2)
    if name == "centre_bump":
        w = p.get("width", 0.08)
        amp = p.get("amp", 0.5)
        base = p.get("base", 1.0)
        return p.get("scale", 1.0) * (base + amp * np.exp(-(x * x + y * y) / w))
    if name in ("tanh_box", "tanh_box_sqrt"):
        d, edge, scale = p["d"], p["eps_edge"], p.get("scale", 1.0)
        v = (0.25 * scale * (1.0 + np.tanh(d * (1.0 - edge - np.abs(x))))
             * (1.0 + np.tanh(d * (1.0 - edge - np.abs(y)))))
        return np.sqrt(v) if name == "tanh_box_sqrt" else v
    raise ValueError(name)


def kernel_table(family, k, h, qmax):
    """K(h*sqrt(q)) for q = 0..qmax, entry 0 unused (kernels.py:106-117,239-247).
    The reference grows its table lazily; entries are elementwise in q, so the
    values do not depend on the growth history."""
    q = np.arange(1, qmax + 1)
    r = h * np.sqrt(q)
    cplx = family == "helmholtz2d"
    out = np.empty(qmax + 1, dtype=np.complex128 if cplx else np.float64)
    out[0] = 0.0
    if family == "laplace2d":
        out[1:] = np.log(r) / (2.0 * np.pi)
    elif family == "helmholtz2d":
        from scipy.special import hankel1
        out[1:] = -0.25j * hankel1(0, k * r)
    elif family == "yukawa2d":
        from scipy.special import k0
        out[1:] = k0(k * r) / (2.0 * np.pi)
    else:
        out[1:] = 1.0 / (4.0 * np.pi * r)
    return out


def diagonal_corr(family, k, h, quad):
    """corr0 of A_ii = a_i + h^2 b_i c_i corr0 (kernels.py:196-203); 'cell' is the
    harness closed-form cell integral of (1/2pi) log r."""
    if quad == "none":
        return 0.0
    if quad == "cell":
        assert family == "laplace2d"
        return (np.log(h) + C_CELL) / (2.0 * np.pi)
    if family == "laplace3d_sl":
        return 3.9002649200601773 / (4.0 * np.pi * h)
    if family == "laplace2d":
        p0, ksm0 = 1.0 / (2.0 * np.pi), 0.0
    elif family == "helmholtz2d":
        lg = np.log(k / 2.0) + 0.5772156649015329
        p0, ksm0 = 1.0 / (2.0 * np.pi), lg / (2.0 * np.pi) - 0.25j
    else:
        lg = np.log(k / 2.0) + 0.5772156649015329
        p0, ksm0 = -1.0 / (2.0 * np.pi), -lg / (2.0 * np.pi)
    return p0 * (1.0 * np.log(h) + LOG_H2_CONST) + ksm0


@dataclass
class Problem:
    """Everything the entry oracle needs: lattice, fields, kernel table."""
    n_side: int
    family: str = "laplace2d"
    k: float = 0.0
    a: tuple = ("one", ())
    b: tuple = ("one", ())
    c: tuple = ("one", ())
    quad: str = "none"
    ic: np.ndarray = dc_field(init=False)
    h: float = dc_field(init=False)

    def __post_init__(self):
        self.ic, xy, self.h = lattice(self.n_side)
        self.av = field_values(*self.a, xy)
        self.bv = field_values(*self.b, xy)
        self.cv = field_values(*self.c, xy)
        self.symmetric = self.b == self.c
        self.dtype = np.complex128 if self.family == "helmholtz2d" else np.float64
        self.corr = diagonal_corr(self.family, self.k, self.h, self.quad)
        # largest squared offset between a grid point and anything within 3
        # rings outside the domain
        ext = self.n_side + 6
        self.table = kernel_table(self.family, self.k, self.h, 2 * ext * ext)


# ---------------------------------------------------------------------------
# entries (kernels.py:249-298)

def _q2(pc, qc):
    d = pc[:, None, :] - qc[None, :, :]
    return d[..., 0] ** 2 + d[..., 1] ** 2


def entries(P, I, J):
    """A[I, J] incl. the diagonal rule (kernels.py:258-275): value
    (K*h^2)*(b_i c_j); coincident entries a_i + h^2 b_i c_i corr."""
    I = np.asarray(I, np.int64)
    J = np.asarray(J, np.int64)
    q2 = _q2(P.ic[I], P.ic[J])
    out = P.table[q2] * (P.h * P.h)
    out *= np.multiply.outer(P.bv[I], P.cv[J])
    ii, jj = np.nonzero(I[:, None] == J[None, :])
    if ii.size:
        g = I[ii]
        out[ii, jj] = P.av[g] + P.h * P.h * P.bv[g] * P.cv[g] * P.corr
    return out


def proxy_src(P, I, Z):
    """h^2 b_i K(x_i, z) (kernels.py:292-298): (K*b)*h^2."""
    I = np.asarray(I, np.int64)
    v = P.table[_q2(P.ic[I], Z)]
    v *= P.bv[I][:, None]
    v *= P.h * P.h
    return v


def proxy_tgt(P, Z, J):
    """h^2 K(z, x_j) c_j (kernels.py:285-290): (K*c)*h^2."""
    J = np.asarray(J, np.int64)
    v = P.table[_q2(Z, P.ic[J])]
    v *= P.cv[J][None, :]
    v *= P.h * P.h
    return v


# ---------------------------------------------------------------------------
# tree + geometry (tree.py:105-138, 275-311; solver_dense.py:24-34)

@dataclass
class Tree:
    n_side: int
    rect: np.ndarray      # (nbox, 4) x0, x1, y0, y1
    level: np.ndarray
    parent: np.ndarray
    kids: np.ndarray      # (nbox, 2), -1 for leaves
    levels: list

    @property
    def depth(self):
        return len(self.levels) - 1

    def is_leaf(self, b):
        return self.kids[b, 0] < 0

    def fine_to_coarse(self):
        for lv in range(self.depth, -1, -1):
            yield from self.levels[lv]

    def coarse_to_fine(self):
        for lv in range(self.depth + 1):
            yield from self.levels[lv]

    def owned(self, b):
        x0, x1, y0, y1 = self.rect[b]
        return (np.arange(y0, y1)[:, None] * self.n_side + np.arange(x0, x1)[None, :]).ravel()


def make_tree(n_side, n_max):
    """Breadth-first alternating bisection, x cut at even levels, cut at
    lo + extent//2 (tree.py:59-61,105-138).  Raises ValueError where the
    reference raises ConfigError."""
    if n_max < 4:
        raise ValueError("leaf size must be at least 4 points")
    if n_side * n_side < n_max:
        raise ValueError("grid smaller than one leaf")
    rect = [(0, n_side, 0, n_side)]
    level, parent, kids = [0], [-1], [[-1, -1]]
    levels = [[0]]
    front = [0]
    npts = lambda r: (r[1] - r[0]) * (r[3] - r[2])
    while any(npts(rect[b]) > n_max for b in front):
        nxt = []
        for b in front:
            if npts(rect[b]) <= n_max:
                raise ValueError("uneven tree")
            x0, x1, y0, y1 = rect[b]
            if level[b] % 2 == 0:
                c = x0 + (x1 - x0) // 2
                halves = ((x0, c, y0, y1), (c, x1, y0, y1))
            else:
                c = y0 + (y1 - y0) // 2
                halves = ((x0, x1, y0, c), (x0, x1, c, y1))
            for i, r in enumerate(halves):
                rect.append(r)
                level.append(level[b] + 1)
                parent.append(b)
                kids.append([-1, -1])
                kids[b][i] = len(rect) - 1
                nxt.append(len(rect) - 1)
        levels.append(list(nxt))
        front = nxt
    return Tree(n_side, np.array(rect, np.int64), np.array(level, np.int64),
                np.array(parent, np.int64), np.array(kids, np.int64), levels)


def ring_walk(w, h):
    """Perimeter cells of a w x h rectangle, CCW from (0,0) (tree.py:301-311)."""
    if w == 1:
        return np.column_stack([np.zeros(h, np.int64), np.arange(h)])
    if h == 1:
        return np.column_stack([np.arange(w), np.zeros(w, np.int64)])
    xs = np.concatenate([np.arange(w - 1), np.full(h - 1, w - 1),
                         np.arange(w - 1, 0, -1), np.zeros(h - 1, np.int64)])
    ys = np.concatenate([np.zeros(w - 1, np.int64), np.arange(h - 1),
                         np.full(w - 1, h - 1), np.arange(h - 1, 0, -1)])
    return np.column_stack([xs, ys]).astype(np.int64)


def proxy_ring(rect, layers):
    """`layers` rings outside the box merged by (walk fraction, ring)
    (tree.py:275-298; no budget on the HSS-D path)."""
    x0, x1, y0, y1 = rect
    cs, ts, js = [], [], []
    for j in range(1, layers + 1):
        r = ring_walk(x1 - x0 + 2 * j, y1 - y0 + 2 * j) + np.array([x0 - j, y0 - j])
        cs.append(r)
        ts.append(np.arange(len(r)) / max(len(r), 1))
        js.append(np.full(len(r), j))
    order = np.lexsort((np.concatenate(js), np.concatenate(ts)))
    return np.concatenate(cs)[order]


def near_field(rect, n_side, pad):
    """Grid points of the clipped pad-dilation minus the box, row-major
    (solver_dense.py:24-34)."""
    x0, x1, y0, y1 = rect
    X0, X1 = max(x0 - pad, 0), min(x1 + pad, n_side)
    Y0, Y1 = max(y0 - pad, 0), min(y1 + pad, n_side)
    yy, xx = np.mgrid[Y0:Y1, X0:X1]
    keep = ~((xx >= x0) & (xx < x1) & (yy >= y0) & (yy < y1))
    return (yy[keep] * n_side + xx[keep]).astype(np.int64)


def proxy_layers(eps, family="laplace2d", k=0.0, layers=0, proxy_layers=0):
    """SolverOptions.resolved_proxy_layers (config.py:26-40)."""
    if proxy_layers:
        return proxy_layers
    if layers:
        return layers
    if family == "helmholtz2d":
        kappa = k / (2.0 * 3.141592653589793)
        if kappa <= 8.0:
            return 2
        if kappa <= 32.0:
            return 3
        raise ValueError("kappa > 32")
    return 1 if eps >= 1e-5 else 2


# ---------------------------------------------------------------------------
# dense core (dense_core.py:67-100, 222-230)

@dataclass
class ColumnID:
    perm: np.ndarray      # pivot order (skeleton first)
    k: int
    T: np.ndarray         # k x (n-k)
    err: float


def column_id(A, eps, min_rank=0):
    """Pivoted-QR column ID: k = first j with |R_jj| <= eps|R_00| (0 when
    R_00 = 0), raised to min(min_rank, min(A.shape)); T = R11^-1 R12
    (dense_core.py:67-100)."""
    m, n = A.shape
    if m == 0 or n == 0:
        return ColumnID(np.arange(n), 0, np.zeros((0, n), A.dtype), 0.0)
    _, R, piv = sla.qr(np.ascontiguousarray(A), mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    top = d[0]
    cut = eps * top
    if top == 0.0 or top <= cut:
        k = 0
    else:
        hit = np.flatnonzero(d <= cut)
        k = int(hit[0]) if hit.size else d.size
    k = max(k, min(min_rank, m, n))
    if k == 0:
        return ColumnID(piv, 0, np.zeros((0, n), A.dtype), float(top))
    T = (np.zeros((k, 0), A.dtype) if k == n
         else sla.solve_triangular(R[:k, :k], R[:k, k:]))
    return ColumnID(piv, k, T, float(d[k]) if k < d.size else 0.0)


class Singular(Exception):
    def __init__(self, where, pivot):
        self.where, self.pivot = where, pivot
        super().__init__(f"singular factor at {where} (pivot magnitude {pivot:.3e})")


def lu_checked(A, where):
    """Partial-pivot LU + pivot-ratio singularity test (dense_core.py:222-230)."""
    lu, piv = sla.lu_factor(A, check_finite=False)
    d = np.abs(np.diag(lu))
    if d.size:
        dmax = d.max()
        if dmax == 0.0 or d.min() <= 1e-300 or d.min() / dmax < np.finfo(float).eps ** 2:
            raise Singular(where, float(d.min()))
    return lu, piv


def interp_L(f, dtype):
    """Pi^T [I; T^T] (m x k) (solver_dense.py:82-86)."""
    m = f.perm.size
    out = np.zeros((m, f.k), dtype)
    out[f.perm[:f.k], np.arange(f.k)] = 1.0
    out[f.perm[f.k:]] = f.T.T
    return out


def interp_R_apply(f, x):
    """[I T] Pi x (solver_dense.py:71-73)."""
    return x[f.perm[:f.k]] + f.T @ x[f.perm[f.k:]]


def interp_L_apply(f, w):
    """Pi^T [I; T^T] w (solver_dense.py:75-80)."""
    out = np.empty((f.perm.size,) + w.shape[1:], np.result_type(f.T.dtype, w.dtype))
    out[f.perm[:f.k]] = w
    out[f.perm[f.k:]] = f.T.T @ w
    return out


# ---------------------------------------------------------------------------
# HSS-D compression / inversion / apply (solver_dense.py:234-372)

@dataclass
class Compressed:
    P: Problem
    tree: Tree
    D: dict
    B: dict
    Lf: dict
    Rf: dict
    rskel: dict
    cskel: dict

    def rows(self, b):
        if self.tree.is_leaf(b):
            return self.tree.owned(b)
        c1, c2 = self.tree.kids[b]
        return np.concatenate([self.rskel[c1], self.rskel[c2]])

    def cols(self, b):
        if self.tree.is_leaf(b):
            return self.tree.owned(b)
        c1, c2 = self.tree.kids[b]
        return np.concatenate([self.cskel[c1], self.cskel[c2]])

    def nbytes(self):
        t = sum(d.nbytes for d in self.D.values())
        t += sum(x.nbytes + y.nbytes for x, y in self.B.values())
        t += sum(f.T.nbytes for f in self.Lf.values())
        t += sum(f.T.nbytes for b, f in self.Rf.items() if f is not self.Lf.get(b))
        return t


def compress(P, tree, eps, pad, boxes=None, H=None):
    """Fine-to-coarse proxy-reduced skeletonization (solver_dense.py:234-272).
    `boxes` (fine-to-coarse order) restricts the sweep to a subtree, adding to
    an existing `H` (used by the distributed tests)."""
    H = H or Compressed(P, tree, {}, {}, {}, {}, {}, {})
    for b in (tree.fine_to_coarse() if boxes is None else boxes):
        rows = H.rows(b)
        if tree.is_leaf(b):
            H.D[b] = entries(P, rows, rows)
        else:
            c1, c2 = tree.kids[b]
            H.B[b] = (entries(P, H.rskel[c1], H.cskel[c2]),
                      entries(P, H.rskel[c2], H.cskel[c1]))
        if b == 0:
            continue
        cols = rows if P.symmetric else H.cols(b)
        zp = proxy_ring(tree.rect[b], pad)
        near = near_field(tree.rect[b], P.n_side, pad)
        rb_t = np.vstack([proxy_src(P, rows, zp).T, entries(P, rows, near).T])
        fr = column_id(rb_t, eps)
        if P.symmetric:
            fc = fr
        else:
            cb = np.vstack([proxy_tgt(P, zp, cols), entries(P, near, cols)])
            fc = column_id(cb, eps, min_rank=fr.k)
            if fc.k > fr.k:
                fr = column_id(rb_t, eps, min_rank=fc.k)
        H.Lf[b] = fr
        H.Rf[b] = fr if P.symmetric else fc
        H.rskel[b] = rows[fr.perm[:fr.k]]
        H.cskel[b] = cols[H.Rf[b].perm[:H.Rf[b].k]]
    return H


@dataclass
class Inverse:
    H: Compressed
    Flu: dict
    E: dict

    def nbytes(self):
        t = sum(lu.nbytes for lu, _ in self.Flu.values())
        t += sum(e.nbytes for e in self.E.values())
        t += sum(f.T.nbytes for f in self.H.Lf.values())
        t += sum(f.T.nbytes for b, f in self.H.Rf.items() if f is not self.H.Lf.get(b))
        return t


def invert(H, boxes=None, inv=None):
    """F = D | [[E1,B12],[B21,E2]]; LU(F); E = (R F^-1 L)^-1
    (solver_dense.py:332-368); `boxes` restricts to a subtree."""
    tree, dt = H.tree, H.P.dtype
    inv = inv or Inverse(H, {}, {})
    for b in (tree.fine_to_coarse() if boxes is None else boxes):
        if tree.is_leaf(b):
            F = np.array(H.D[b], dtype=dt)
        else:
            c1, c2 = tree.kids[b]
            F = np.block([[inv.E[c1], H.B[b][0]], [H.B[b][1], inv.E[c2]]]).astype(dt)
        inv.Flu[b] = lu_checked(F, f"box {b} level {tree.level[b]}")
        if b == 0:
            continue
        W = sla.lu_solve(inv.Flu[b], interp_L(H.Lf[b], dt), check_finite=False)
        G = interp_R_apply(H.Rf[b], W)
        glu = lu_checked(G, f"E of box {b}")
        inv.E[b] = sla.lu_solve(glu, np.eye(G.shape[0], dtype=dt), check_finite=False)
    return inv


def apply_up(inv, f2, boxes, ups, uin):
    """Up sweep over `boxes` (fine to coarse): phi = F^-1 u, ups = E R phi
    (solver_dense.py:303-310)."""
    H, tree = inv.H, inv.H.tree
    for b in boxes:
        u = f2[tree.owned(b)] if tree.is_leaf(b) else np.vstack([ups[c] for c in tree.kids[b]])
        uin[b] = u
        if b == 0:
            continue
        phi = sla.lu_solve(inv.Flu[b], u, check_finite=False)
        ups[b] = inv.E[b] @ interp_R_apply(H.Rf[b], phi)


def apply_down(inv, boxes, ups, uin, dn, out):
    """Down sweep over `boxes` (coarse to fine) (solver_dense.py:312-328)."""
    H, tree = inv.H, inv.H.tree
    for b in boxes:
        u = uin[b]
        if b == 0:
            res = sla.lu_solve(inv.Flu[0], u, check_finite=False)
        else:
            nu = u - interp_L_apply(H.Lf[b], ups[b])
            if dn.get(b) is not None:
                nu += interp_L_apply(H.Lf[b], inv.E[b] @ dn[b])
            res = sla.lu_solve(inv.Flu[b], nu, check_finite=False)
        if tree.is_leaf(b):
            out[tree.owned(b)] = res
        else:
            c1, c2 = tree.kids[b]
            k1 = inv.E[c1].shape[0]
            dn[c1], dn[c2] = res[:k1], res[k1:]


def apply_inverse(inv, f):
    """Up (fine->coarse) then down (coarse->fine) sweeps
    (solver_dense.py:293-329)."""
    H, tree = inv.H, inv.H.tree
    f = np.asarray(f, dtype=np.result_type(H.P.dtype, np.asarray(f).dtype))
    single = f.ndim == 1
    f2 = f[:, None] if single else f
    out = np.zeros_like(f2)
    ups, uin = {}, {}
    apply_up(inv, f2, list(tree.fine_to_coarse()), ups, uin)
    apply_down(inv, list(tree.coarse_to_fine()), ups, uin, {0: None}, out)
    return out[:, 0] if single else out


def matvec(H, x):
    """Forward compressed operator (solver_dense.py:143-178)."""
    tree = H.tree
    x = np.asarray(x, dtype=np.result_type(H.P.dtype, np.asarray(x).dtype))
    single = x.ndim == 1
    x2 = x[:, None] if single else x
    out = np.zeros_like(x2)
    phi = {}
    for b in tree.fine_to_coarse():
        if b == 0:
            continue
        w = x2[tree.owned(b)] if tree.is_leaf(b) else np.vstack([phi[c] for c in tree.kids[b]])
        phi[b] = interp_R_apply(H.Rf[b], w)
    wdn = {}
    for b in tree.coarse_to_fine():
        if tree.is_leaf(b):
            continue
        c1, c2 = tree.kids[b]
        w1 = H.B[b][0] @ phi[c2]
        w2 = H.B[b][1] @ phi[c1]
        if b in wdn:
            t = interp_L_apply(H.Lf[b], wdn[b])
            k1 = H.Rf[c1].k
            w1, w2 = w1 + t[:k1], w2 + t[k1:]
        wdn[c1], wdn[c2] = w1, w2
    for b in range(len(tree.rect)):
        if not tree.is_leaf(b):
            continue
        idx = tree.owned(b)
        r = H.D[b] @ x2[idx]
        if b in wdn:
            r += interp_L_apply(H.Lf[b], wdn[b])
        out[idx] = r
    return out[:, 0] if single else out


def dense_matrix(P):
    """Full A (small N only)."""
    idx = np.arange(P.n_side * P.n_side)
    return entries(P, idx, idx)


def solve(P, n_max, eps, f, pad=None):
    """Tree + compress + invert + apply; returns (x, H, inv)."""
    tree = make_tree(P.n_side, n_max)
    pad = pad or proxy_layers(eps, P.family, P.k)
    H = compress(P, tree, eps, pad)
    inv = invert(H)
    return apply_inverse(inv, f), H, inv


# ---------------------------------------------------------------------------
# compressed path with a-priori skeletons, dense blocks
# (tree.py:141-269 annotate_skeletons; solver_compressed.py:223-266
#  _interp_lowrank at full rank; 437-483 _dense_factors / _dense_E_from_lu;
#  560-577 dense root).  Restated as the dense oracle the reference's own
#  tests use (test_solver_compressed.py:88-126 dense_box_F): T from
#  lstsq(K(Z, X_sk), K(Z, X_rs)) with the field scalings.

def _ring_dist(dx, dy, w, h):
    return np.minimum(np.minimum(dx, w - 1 - dx), np.minimum(dy, h - 1 - dy))


def _walk_order(idx, rect, n_side):
    """Band points by (t on own ring, ring, dx, dy) (tree.py:148-180)."""
    x0, x1, y0, y1 = (int(v) for v in rect)
    w, h = x1 - x0, y1 - y0
    dx, dy = idx % n_side - x0, idx // n_side - y0
    r = _ring_dist(dx, dy, w, h)
    rw, rh, lx, ly = w - 2 * r, h - 2 * r, dx - r, dy - r
    pos = np.where(ly == 0, lx, np.where(
        lx == rw - 1, rw - 1 + ly, np.where(
            ly == rh - 1, 2 * (rw - 1) + (rh - 1) - lx,
            2 * (rw - 1) + 2 * (rh - 1) - ly)))
    per = np.maximum(2 * (rw - 1) + 2 * (rh - 1), 1)
    return idx[np.lexsort((dy, dx, r, pos / per))]


def annotate(tree, layers):
    """{box: (sk, rs, work_perm)} fine to coarse (tree.py:198-269; no
    support mask, no interior retention)."""
    n = tree.n_side
    out = {}
    for b in tree.fine_to_coarse():
        if tree.is_leaf(b):
            full = tree.owned(b)
        else:
            c1, c2 = tree.kids[b]
            full = np.concatenate([out[c1][0], out[c2][0]])
        x0, x1, y0, y1 = (int(v) for v in tree.rect[b])
        dx, dy = full % n - x0, full // n - y0
        band = _ring_dist(dx, dy, x1 - x0, y1 - y0) < layers
        sk = _walk_order(full[band], tree.rect[b], n)
        rs = full[~band]
        rdx, rdy = rs % n - x0, rs // n - y0
        rs = rs[np.lexsort((rdx, rdy) if tree.level[b] % 2 == 0 else (rdy, rdx))]
        where = {g: i for i, g in enumerate(full.tolist())}
        perm = np.array([where[g] for g in np.concatenate([sk, rs]).tolist()], np.int64)
        out[b] = (sk, rs, perm)
    return out


def compress_apriori(P, tree, layers):
    """A Compressed object whose skeletons are the a-priori bands and whose
    interpolations are the proxy least-squares fits; invert() / apply_inverse()
    then give the compressed path's solution with dense blocks."""
    ann = annotate(tree, layers)
    H = Compressed(P, tree, {}, {}, {}, {}, {}, {})
    for b in tree.fine_to_coarse():
        rows = H.rows(b)
        if tree.is_leaf(b):
            H.D[b] = entries(P, rows, rows)
        else:
            c1, c2 = tree.kids[b]
            H.B[b] = (entries(P, H.rskel[c1], H.cskel[c2]),
                      entries(P, H.rskel[c2], H.cskel[c1]))
        if b == 0:
            continue
        sk, rs, perm = ann[b]
        zp = proxy_ring(tree.rect[b], layers)
        k = sk.size
        if rs.size:
            t_up = sla.lstsq(proxy_tgt(P, zp, sk), proxy_tgt(P, zp, rs))[0]
            t_dn = sla.lstsq(proxy_src(P, sk, zp).T, proxy_src(P, rs, zp).T)[0]
        else:
            t_up = t_dn = np.zeros((k, 0))
        H.Lf[b] = ColumnID(perm, k, t_dn, 0.0)
        H.Rf[b] = ColumnID(perm, k, t_up, 0.0)
        H.rskel[b] = H.cskel[b] = sk
    return H, ann


def solve_apriori(P, n_max, layers, f):
    """Tree + a-priori compression + invert + apply; returns (x, H, inv)."""
    tree = make_tree(P.n_side, n_max)
    H, _ = compress_apriori(P, tree, layers)
    inv = invert(H)
    return apply_inverse(inv, f), H, inv
