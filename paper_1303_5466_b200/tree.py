"""Binary box tree over the grid and proxy rings (host integer planning).

Mirrors the reference's tree.py for the HSS-D path: `build_tree`
(tree.py:105-138), `BoxTree.owned_indices` (tree.py:97-102) and
`proxy_points` / `_ring_cells` (tree.py:275-311).  The tree is built one
level at a time with array operations (breadth-first ids, so children of the
j-th box of a level are boxes 2j, 2j+1 of the next level); the per-level
rectangle arrays are what the device planner consumes.  The a-priori
skeleton choice of the compressed path (`annotate_skeletons`,
tree.py:141-269) fills per-box skeleton / residual splits on the host.
"""

import numpy as np

from .errors import ConfigError


class BoxNode:
    __slots__ = ("idx", "level", "parent", "children", "x0", "x1", "y0", "y1",
                 "full_idx", "sk_idx", "rs_idx", "work_perm", "n_interior_sk")

    def __init__(self, idx, level, parent, x0, x1, y0, y1):
        self.idx, self.level, self.parent = idx, level, parent
        self.children = None
        self.full_idx = self.sk_idx = self.rs_idx = self.work_perm = None
        self.n_interior_sk = 0
        self.x0, self.x1, self.y0, self.y1 = x0, x1, y0, y1

    @property
    def is_leaf(self):
        return self.children is None

    @property
    def width(self):
        return self.x1 - self.x0

    @property
    def height(self):
        return self.y1 - self.y0

    @property
    def npoints(self):
        return self.width * self.height

    @property
    def shape_key(self):
        return (self.width, self.height)

    def split_axis(self):
        return "x" if self.level % 2 == 0 else "y"

    def __repr__(self):
        return f"Box({self.idx}, lvl={self.level}, [{self.x0},{self.x1})x[{self.y0},{self.y1}))"


_OWNED_CACHE = {}


class BoxTree:
    """Nodes in breadth-first order plus per-level arrays.

    rects[l]: (n_l, 4) int64 array of (x0, x1, y0, y1) of level l's boxes,
    ids[l]: their node ids (contiguous: 2^l - 1 ... for a full binary tree)."""

    def __init__(self, grid, n_max):
        self.grid = grid
        self.n_max = n_max
        self._nodes = None
        self._levels = None
        self.rects = []
        self.ids = []
        self.parents = []
        self.layers = 0

    # The node objects and id lists mirror the reference's API; the solver only
    # reads the per-level arrays, so they are materialised on first use.
    @property
    def nodes(self):
        if self._nodes is None:
            nodes = []
            for lv, (r, ids_l, par) in enumerate(zip(self.rects, self.ids, self.parents)):
                for i, row, p in zip(ids_l.tolist(), r.tolist(), par.tolist()):
                    nodes.append(BoxNode(i, lv, p, row[0], row[1], row[2], row[3]))
            for lv in range(1, len(self.ids)):
                kid = self.ids[lv].tolist()
                for j, pid in enumerate(self.ids[lv - 1].tolist()):
                    nodes[pid].children = (kid[2 * j], kid[2 * j + 1])
            self._nodes = nodes
        return self._nodes

    @property
    def levels(self):
        if self._levels is None:
            self._levels = [ids_l.tolist() for ids_l in self.ids]
        return self._levels

    @property
    def depth(self):
        return len(self.ids) - 1

    @property
    def root(self):
        return self.nodes[0]

    def leaves(self):
        return [b for b in self.nodes if b.is_leaf]

    def boxes_fine_to_coarse(self):
        for lv in range(self.depth, -1, -1):
            for i in self.levels[lv]:
                yield self.nodes[i]

    def boxes_coarse_to_fine(self):
        for lv in range(self.depth + 1):
            for i in self.levels[lv]:
                yield self.nodes[i]

    def owned_indices(self, box):
        n = self.grid.n_side
        return (np.arange(box.y0, box.y1)[:, None] * n + np.arange(box.x0, box.x1)[None, :]).ravel()

    def owned_level(self, lv):
        """(n_l, w*h) int64 owned indices of every box of level `lv`; memoised
        per (grid side, leaf size, level) -- trees are deterministic."""
        key = (self.grid.n_side, self.n_max, lv)
        out = _OWNED_CACHE.get(key)
        if out is None:
            out = self._owned_level(lv)
            out.setflags(write=False)
            if len(_OWNED_CACHE) > 64:
                _OWNED_CACHE.clear()
            _OWNED_CACHE[key] = out
        return out

    def _owned_level(self, lv):
        """(n_l, w*h) int64 owned indices of every box of level `lv` (all boxes
        of the leaf level share one shape for the trees build_tree accepts,
        otherwise rows are padded with -1)."""
        r = self.rects[lv]
        w = r[:, 1] - r[:, 0]
        h = r[:, 3] - r[:, 2]
        npts = (w * h).max()
        t = np.arange(npts)[None, :]
        wv = w[:, None]
        out = (r[:, 2:3] + t // wv) * self.grid.n_side + (r[:, 0:1] + t % wv)
        out[t >= (w * h)[:, None]] = -1
        return out


def build_tree(grid, n_max):
    """Alternating bisection (x at even levels, cut at lo + extent//2) until
    every leaf holds <= n_max points (tree.py:105-138)."""
    if n_max < 4:
        raise ConfigError("leaf size must be at least 4 points")
    if grid.n < n_max:
        raise ConfigError("grid smaller than one leaf")
    tree = BoxTree(grid, n_max)
    rect = np.array([[0, grid.n_side, 0, grid.n_side]], dtype=np.int64)
    ids = np.array([0])
    rects, idss, parents = [rect], [ids], [np.array([-1])]
    while True:
        npts = (rect[:, 1] - rect[:, 0]) * (rect[:, 3] - rect[:, 2])
        big = npts > n_max
        if not big.any():
            break
        if not big.all():
            raise ConfigError("uneven tree: box sizes at one level straddle the leaf size")
        lv = len(rects) - 1
        kids = np.repeat(rect, 2, axis=0)
        if lv % 2 == 0:
            cut = rect[:, 0] + (rect[:, 1] - rect[:, 0]) // 2
            kids[0::2, 1] = cut
            kids[1::2, 0] = cut
        else:
            cut = rect[:, 2] + (rect[:, 3] - rect[:, 2]) // 2
            kids[0::2, 3] = cut
            kids[1::2, 2] = cut
        start = ids[-1] + 1
        kid_ids = start + np.arange(kids.shape[0])
        parents.append(np.repeat(ids, 2))
        rect, ids = kids, kid_ids
        rects.append(rect)
        idss.append(ids)
    tree.rects = rects
    tree.ids = idss
    tree.parents = parents
    return tree


def _ring_cells(w, h):
    """Perimeter of a w x h rectangle walked CCW from (0, 0) (tree.py:301-311)."""
    if w == 1:
        return np.column_stack([np.zeros(h, np.int64), np.arange(h)])
    if h == 1:
        return np.column_stack([np.arange(w), np.zeros(w, np.int64)])
    xs = np.concatenate([np.arange(w - 1), np.full(h - 1, w - 1),
                         np.arange(w - 1, 0, -1), np.zeros(h - 1, np.int64)])
    ys = np.concatenate([np.zeros(w - 1, np.int64), np.arange(h - 1),
                         np.full(w - 1, h - 1), np.arange(h - 1, 0, -1)])
    return np.column_stack([xs, ys]).astype(np.int64)


def proxy_points(box, layers, budget=None):
    """`layers` lattice rings just outside the box, merged by walk fraction
    then ring (tree.py:275-298); optional uniform decimation to `budget`."""
    cs, ts, js = [], [], []
    for j in range(1, layers + 1):
        ring = _ring_cells(box.width + 2 * j, box.height + 2 * j)
        ring += np.array([box.x0 - j, box.y0 - j])
        cs.append(ring)
        ts.append(np.arange(len(ring)) / max(len(ring), 1))
        js.append(np.full(len(ring), j))
    order = np.lexsort((np.concatenate(js), np.concatenate(ts)))
    out = np.concatenate(cs)[order]
    if budget is not None and budget < len(out):
        out = out[np.linspace(0, len(out), budget, endpoint=False).astype(np.int64)]
    return out


def proxy_count(w, h, layers):
    """Number of proxy points of a w x h box (sum of ring lengths)."""
    tot = 0
    for j in range(1, layers + 1):
        W, H = w + 2 * j, h + 2 * j
        tot += H if W == 1 else W if H == 1 else 2 * (W - 1) + 2 * (H - 1)
    return tot


def proxy_count_v(w, h, layers):
    """Vectorised proxy_count over arrays of box widths/heights."""
    w = np.asarray(w, dtype=np.int64)
    h = np.asarray(h, dtype=np.int64)
    tot = np.zeros(w.shape, dtype=np.int64)
    for j in range(1, layers + 1):
        W, H = w + 2 * j, h + 2 * j
        tot += np.where(W == 1, H, np.where(H == 1, W, 2 * (W - 1) + 2 * (H - 1)))
    return tot


def near_count(rects, n_side, pad):
    """Vectorised size of the clipped pad-dilation minus the box
    (solver_dense.py:24-34)."""
    x0, x1, y0, y1 = rects.T
    X0, X1 = np.maximum(x0 - pad, 0), np.minimum(x1 + pad, n_side)
    Y0, Y1 = np.maximum(y0 - pad, 0), np.minimum(y1 + pad, n_side)
    return (X1 - X0) * (Y1 - Y0) - (x1 - x0) * (y1 - y0)


def near_field_indices(box, grid, pad):
    """Host version of solver_dense.py:24-34 (tests / API)."""
    n = grid.n_side
    X0, X1 = max(box.x0 - pad, 0), min(box.x1 + pad, n)
    Y0, Y1 = max(box.y0 - pad, 0), min(box.y1 + pad, n)
    yy, xx = np.mgrid[Y0:Y1, X0:X1]
    keep = ~((xx >= box.x0) & (xx < box.x1) & (yy >= box.y0) & (yy < box.y1))
    return (yy[keep] * n + xx[keep]).astype(np.int64)


# ---------------------------------------------------------------------------
# a-priori skeletons of the compressed path (tree.py:141-269)

def ring_of(dx, dy, w, h):
    """Distance of box-local cell (dx, dy) to the box boundary (tree.py:143-145)."""
    return np.minimum(np.minimum(dx, w - 1 - dx), np.minimum(dy, h - 1 - dy))


def walk_key(dx, dy, w, h):
    """(t, ring): t = CCW position of the cell on its own ring, from that
    ring's lower-left corner, over the ring length (tree.py:148-167)."""
    dx = np.asarray(dx, dtype=np.int64)
    dy = np.asarray(dy, dtype=np.int64)
    r = ring_of(dx, dy, w, h)
    rw, rh = w - 2 * r, h - 2 * r
    lx, ly = dx - r, dy - r
    pos = np.select([ly == 0, lx == rw - 1, ly == rh - 1],
                    [lx, (rw - 1) + ly, (rw - 1) + (rh - 1) + (rw - 1 - lx)],
                    2 * (rw - 1) + (rh - 1) + (rh - 1 - ly))
    per = np.maximum(2 * (rw - 1) + 2 * (rh - 1), 1)
    return pos / per, r


def order_boundary_cyclic(indices, box, grid):
    """Band points by (t, ring, dx, dy) (tree.py:170-180)."""
    indices = np.asarray(indices, dtype=np.int64)
    if indices.size == 0:
        return indices
    n = grid.n_side
    dx, dy = indices % n - box.x0, indices // n - box.y0
    t, r = walk_key(dx, dy, box.width, box.height)
    return indices[np.lexsort((dy, dx, r, t))]


def order_interface(indices, box, grid):
    """Interior points along the children's interface (tree.py:183-195)."""
    indices = np.asarray(indices, dtype=np.int64)
    if indices.size == 0:
        return indices
    n = grid.n_side
    dx, dy = indices % n - box.x0, indices // n - box.y0
    keys = (dx, dy) if box.split_axis() == "x" else (dy, dx)
    return indices[np.lexsort(keys)]


def boundary_layer_split(box, layers, grid, candidates=None, support_mask=None):
    """(sk, rs): candidates within `layers` of the box boundary vs the rest;
    points outside `support_mask` never become skeletons (tree.py:198-218)."""
    n = grid.n_side
    if candidates is None:
        candidates = (np.arange(box.y0, box.y1)[:, None] * n
                      + np.arange(box.x0, box.x1)[None, :]).ravel()
    candidates = np.asarray(candidates, dtype=np.int64)
    dx, dy = candidates % n - box.x0, candidates // n - box.y0
    band = ring_of(dx, dy, box.width, box.height) < layers
    if support_mask is not None:
        band &= np.asarray(support_mask)[candidates]
    return (order_boundary_cyclic(candidates[band], box, grid),
            order_interface(candidates[~band], box, grid))


def interface_interior_subset(rs_idx, box, grid, k_wave, points_per_wavelength):
    """Residual points kept as skeletons for oscillatory kernels: a sublattice
    at the requested density per wavelength (tree.py:221-234)."""
    if rs_idx.size == 0:
        return np.zeros(0, dtype=bool)
    cells = (2.0 * np.pi / k_wave) / grid.h
    stride = max(1, int(np.floor(cells / points_per_wavelength)))
    if stride <= 1:
        return np.ones(rs_idx.size, dtype=bool)
    n = grid.n_side
    return (rs_idx % n % stride == 0) & (rs_idx // n % stride == 0)


def annotate_skeletons(tree, layers, support_mask=None, k_wave=None, points_per_wavelength=0.0):
    """A-priori skeleton / residual split of every box, fine to coarse
    (tree.py:237-269): a leaf splits its owned points, a parent the
    concatenation of its children's skeletons, against its own boundary band
    of width `layers`.  `work_perm` maps [sk, rs] onto positions in that
    concatenation (`full_idx`).  Levels whose boxes share one shape (every
    level of a power-of-two grid) are split with 2-D array operations; the
    per-level arrays are kept in `tree.ann_levels[lv]` = (k, work_perm) for
    the device planner."""
    tree.layers = layers
    keep_interior = k_wave is not None and points_per_wavelength > 0
    nodes = tree.nodes
    tree.ann_levels = {}
    n = tree.grid.n_side
    for lv in range(tree.depth, -1, -1):
        ids = tree.ids[lv]
        rects = tree.rects[lv]
        w, h = rects[:, 1] - rects[:, 0], rects[:, 3] - rects[:, 2]
        uniform = (support_mask is None and not keep_interior
                   and (w == w[0]).all() and (h == h[0]).all())
        if lv == tree.depth:
            full = [tree.owned_indices(nodes[i]) for i in ids.tolist()] if not uniform else \
                tree.owned_level(lv)
        else:
            kid = tree.ids[lv + 1]
            full = [np.concatenate([nodes[a].sk_idx, nodes[b].sk_idx])
                    for a, b in zip(kid[0::2].tolist(), kid[1::2].tolist())]
            uniform = uniform and len({f.size for f in full}) == 1
            if uniform:
                full = np.stack(full)
        if uniform:
            _annotate_level_uniform(tree, lv, np.asarray(full), layers)
            continue
        for j, i in enumerate(ids.tolist()):
            box = nodes[i]
            box.full_idx = np.asarray(full[j], dtype=np.int64)
            sk, rs = boundary_layer_split(box, layers, tree.grid, candidates=box.full_idx,
                                          support_mask=support_mask)
            box.n_interior_sk = 0
            if keep_interior and not box.is_leaf and rs.size:
                keep = interface_interior_subset(rs, box, tree.grid, k_wave,
                                                 points_per_wavelength)
                extra = rs[keep]
                rs = rs[~keep]
                sk = np.concatenate([sk, extra])
                box.n_interior_sk = extra.size
            box.sk_idx, box.rs_idx = sk, rs
            # full_idx has distinct entries: position of each [sk, rs] point in it
            srt = np.argsort(box.full_idx, kind="stable")
            order = np.concatenate([sk, rs])
            box.work_perm = srt[np.searchsorted(box.full_idx, order, sorter=srt)].astype(np.int64)
        k = np.array([nodes[i].sk_idx.size for i in ids.tolist()], np.int64)
        m = max(nodes[i].full_idx.size for i in ids.tolist())
        perm = np.zeros((len(ids), m), np.int64)
        for j, i in enumerate(ids.tolist()):
            perm[j, :nodes[i].work_perm.size] = nodes[i].work_perm
        tree.ann_levels[lv] = (k, perm)
    return tree


def _annotate_level_uniform(tree, lv, full, layers):
    """One level of annotate_skeletons for boxes of one shape: the band mask
    has the same count in every row (translation of one box), so the splits
    are (nb, k) / (nb, r) arrays ordered with a row-wise lexsort."""
    n = tree.grid.n_side
    rects = tree.rects[lv]
    x0, y0 = rects[:, 0:1], rects[:, 2:3]
    w, h = int(rects[0, 1] - rects[0, 0]), int(rects[0, 3] - rects[0, 2])
    dx, dy = full % n - x0, full // n - y0
    if (dx == dx[0]).all() and (dy == dy[0]).all():
        # every box is a translate of the first (true by induction for trees
        # of one box shape per level): split the first, reuse the permutation
        dx, dy = dx[:1], dy[:1]
    band = ring_of(dx, dy, w, h) < layers
    m = full.shape[1]
    nb = dx.shape[0]
    k = int(band[0].sum())
    pos = np.broadcast_to(np.arange(m), (nb, m))
    bpos = pos[band].reshape(nb, k)
    rpos = pos[~band].reshape(nb, m - k)
    take = lambda a, p: np.take_along_axis(a, p, axis=1)  # noqa: E731
    if k:
        bdx, bdy = take(dx, bpos), take(dy, bpos)
        t, r = walk_key(bdx, bdy, w, h)
        bpos = take(bpos, np.lexsort((bdy, bdx, r, t), axis=-1))
    if m - k:
        rdx, rdy = take(dx, rpos), take(dy, rpos)
        keys = (rdx, rdy) if lv % 2 == 0 else (rdy, rdx)
        rpos = take(rpos, np.lexsort(keys, axis=-1))
    perm = np.concatenate([bpos, rpos], axis=1)
    if nb < full.shape[0]:
        perm = np.broadcast_to(perm, full.shape)
    nb = full.shape[0]
    ordered = take(full, perm)
    nodes = tree.nodes
    for j, i in enumerate(tree.ids[lv].tolist()):
        box = nodes[i]
        box.full_idx = full[j]
        box.sk_idx = ordered[j, :k]
        box.rs_idx = ordered[j, k:]
        box.work_perm = perm[j]
        box.n_interior_sk = 0
    tree.ann_levels[lv] = (np.full(nb, k, np.int64), perm)
