"""Binary box tree over the grid and proxy rings (host integer planning).

Mirrors the reference's tree.py for the HSS-D path: `build_tree`
(tree.py:105-138), `BoxTree.owned_indices` (tree.py:97-102) and
`proxy_points` / `_ring_cells` (tree.py:275-311).  The tree is built one
level at a time with array operations (breadth-first ids, so children of the
j-th box of a level are boxes 2j, 2j+1 of the next level); the per-level
rectangle arrays are what the device planner consumes.  The a-priori
skeleton machinery of the O(N) path (tree.py:141-269) is out of scope.
"""

import numpy as np

from .errors import ConfigError


class BoxNode:
    __slots__ = ("idx", "level", "parent", "children", "x0", "x1", "y0", "y1")

    def __init__(self, idx, level, parent, x0, x1, y0, y1):
        self.idx, self.level, self.parent = idx, level, parent
        self.children = None
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
