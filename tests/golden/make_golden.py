"""Generate the golden parity fixtures by running the REFERENCE implementation.

Runs only in the build container (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs tests/golden/*.npz.  Nothing here is imported by the product or by
GPU tests at run time; the GPU box only reads the committed .npz files.
The BASELINE configs are expressed in reference objects exactly as SURVEY.md
Appendix A.2 recommends: a frozen `Field` subclass for the centre bump and a
`QuadratureCorrection` subclass for the closed-form cell-integral diagonal.
"""
import hashlib
import math
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from vief import Grid, KernelSpec, PLAIN, H4, SolverOptions, build_tree, make_field  # noqa: E402
from vief.kernels import Field, QuadratureCorrection, assemble_dense, get_assembler  # noqa: E402
from vief.tree import proxy_points  # noqa: E402
from vief.solver_dense import compress_outer, invert_dense_block, _near_field_indices  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
C_CELL = -1.5 + math.pi / 4.0 - 0.5 * math.log(2.0)


@dataclass(frozen=True)
class CentreBump(Field):
    """scale * (1 + 0.5 exp(-|x|^2/0.08)) on [-1,1]^2 == BASELINE's
    1 + 0.5 exp(-|x'-(.5,.5)|^2/0.02) on [0,1]^2."""

    def __call__(self, xy):
        xy = np.asarray(xy, dtype=float)
        x, y = xy[..., 0], xy[..., 1]
        p = dict(self.params)
        return p.get("scale", 1.0) * (p.get("base", 1.0) + p.get("amp", 0.5)
                                      * np.exp(-(x * x + y * y) / p.get("width", 0.08)))


@dataclass(frozen=True)
class CellQuad(QuadratureCorrection):
    """A_ii = a_i + h^2 b_i c_i (1/2pi)(log h + c_cell)."""

    def diagonal_term(self, spec, h):
        return (np.log(h) + C_CELL) / (2.0 * np.pi)


def bump(scale=1.0):
    return CentreBump("centre_bump", tuple(sorted(dict(scale=scale).items())))


CELL = CellQuad("none")


def tree_arrays(tree):
    nodes = tree.nodes
    rect = np.array([(b.x0, b.x1, b.y0, b.y1) for b in nodes], np.int32)
    level = np.array([b.level for b in nodes], np.int32)
    parent = np.array([b.parent for b in nodes], np.int32)
    kids = np.array([b.children if b.children else (-1, -1) for b in nodes], np.int32)
    return dict(rect=rect, level=level, parent=parent, kids=kids)


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(np.asarray(a, np.int64)).tobytes())
        h.update(b"|")
    return h.hexdigest()


def gen_trees():
    out = {}
    for n, nmax in ((7, 49), (14, 49), (28, 49), (18, 81), (9, 25), (30, 64), (128, 64), (64, 64)):
        t = tree_arrays(build_tree(Grid(n), nmax))
        for k, v in t.items():
            out[f"t{n}_{nmax}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "trees.npz"), **out)


def gen_geometry():
    """proxy rings + near fields, every box of two trees (pads 1..3), plus
    digests for the 128^2 / 1024^2-shaped trees."""
    out = {}
    for n, nmax in ((28, 49), (18, 81), (30, 64)):
        tree = build_tree(Grid(n), nmax)
        for pad in (1, 2, 3):
            for b in tree.nodes:
                out[f"p{n}_{pad}_{b.idx}"] = proxy_points(b, pad).astype(np.int32)
                out[f"n{n}_{pad}_{b.idx}"] = _near_field_indices(b, tree.grid, pad).astype(np.int32)
    for n, nmax in ((128, 64), (256, 64)):
        tree = build_tree(Grid(n), nmax)
        out[f"dig_proxy_{n}"] = np.frombuffer(
            digest([proxy_points(b, 2) for b in tree.nodes]).encode(), np.uint8)
        out[f"dig_near_{n}"] = np.frombuffer(
            digest([_near_field_indices(b, tree.grid, 2) for b in tree.nodes]).encode(), np.uint8)
    np.savez_compressed(os.path.join(OUT, "geometry.npz"), **out)


def gen_entries():
    out = {}
    specs = {
        "nti": KernelSpec("laplace2d", b_field=make_field("gaussian_bump"),
                          c_field=make_field("gaussian_bump")),
        "rows": KernelSpec("laplace2d", b_field=bump(math.pi / 2), c_field=make_field("one")),
        "helm": KernelSpec("helmholtz2d", k=2 * np.pi * 2),
        "yuk": KernelSpec("yukawa2d", k=3.0, b_field=make_field("gaussian_bump")),
    }
    quads = {"plain": PLAIN, "h4": H4, "cell": CELL}
    for sname, spec in specs.items():
        for qname, quad in quads.items():
            if qname == "cell" and spec.family != "laplace2d":
                continue
            for n in (4, 12):
                idx = np.arange(n * n)
                out[f"A_{sname}_{qname}_{n}"] = assemble_dense(spec, Grid(n), quad, idx, idx)
            asm = get_assembler(spec, Grid(12), quad)
            tree = build_tree(Grid(12), 36)
            box = tree.nodes[3]
            rows = tree.owned_indices(box)
            zp = proxy_points(box, 2)
            out[f"pc_{sname}_{qname}"] = asm.proxy_cols(rows, zp)
            out[f"pr_{sname}_{qname}"] = asm.proxy_rows(zp, rows)
    np.savez_compressed(os.path.join(OUT, "entries.npz"), **out)


def run_case(name, spec, n, leaf, eps, quad, nrhs, seed, store_skel=True):
    grid = Grid(n)
    opts = SolverOptions(eps=eps, leaf_size=leaf, k_cut=None)
    t0 = time.perf_counter()
    tree = build_tree(grid, leaf)
    H = compress_outer(spec, grid, tree, eps, opts, quad)
    t1 = time.perf_counter()
    inv = invert_dense_block(H)
    t2 = time.perf_counter()
    rng = np.random.default_rng(seed)
    if spec.is_complex:
        f = rng.standard_normal((grid.n, nrhs)) + 1j * rng.standard_normal((grid.n, nrhs))
    else:
        f = rng.standard_normal((grid.n, nrhs))
    x = inv.apply(f)
    t3 = time.perf_counter()
    hx = H.matvec(x)
    out = dict(f=f, x=x, hx=hx, nbytes_inv=np.int64(inv.nbytes()), nbytes_H=np.int64(H.nbytes()),
               times=np.array([t1 - t0, t2 - t1, t3 - t2]))
    nb = len(tree.nodes)
    out["rank"] = np.array([H.row_skel[i].size if i in H.row_skel else -1 for i in range(nb)], np.int32)
    if store_skel:
        out["row_skel"] = np.concatenate([H.row_skel.get(i, np.zeros(0, np.int64)) for i in range(nb)]).astype(np.int32)
        out["col_skel"] = np.concatenate([H.col_skel.get(i, np.zeros(0, np.int64)) for i in range(nb)]).astype(np.int32)
    if n <= 30:
        idx = np.arange(grid.n)
        A = assemble_dense(spec, grid, quad, idx, idx)
        out["x_dense"] = np.linalg.solve(A, f)
    np.savez_compressed(os.path.join(OUT, f"solve_{name}.npz"), **out)
    print(f"{name}: build {t1-t0:.2f}s factor {t2-t1:.2f}s apply {t3-t2:.2f}s "
          f"max rank {out['rank'].max()} nbytes {inv.nbytes()}")


def gen_solves():
    nti = KernelSpec("laplace2d", b_field=make_field("gaussian_bump"),
                     c_field=make_field("gaussian_bump"))
    rows = KernelSpec("laplace2d", b_field=make_field("gaussian_bump"), c_field=make_field("one"))
    run_case("nti28", nti, 28, 49, 1e-10, PLAIN, 3, 3)
    run_case("rows14", rows, 14, 49, 1e-10, PLAIN, 2, 5)
    run_case("rows30", rows, 30, 64, 1e-10, PLAIN, 2, 5)
    run_case("helm18", KernelSpec("helmholtz2d", k=2 * np.pi * 2), 18, 81, 1e-10, PLAIN, 2, 6)
    run_case("single7", nti, 7, 49, 1e-10, PLAIN, 1, 1)
    run_case("eps5_28", rows, 28, 49, 1e-5, H4, 2, 8)
    c1 = KernelSpec("laplace2d", b_field=bump(math.pi / 2), c_field=make_field("one"))
    run_case("c1_64", c1, 64, 64, 1e-10, CELL, 2, 0)
    run_case("c1_128", c1, 128, 64, 1e-10, CELL, 2, 0)
    if os.environ.get("GOLDEN_BIG"):
        run_case("c1_256", c1, 256, 64, 1e-10, CELL, 1, 0)


if __name__ == "__main__":
    gen_trees()
    gen_geometry()
    gen_entries()
    gen_solves()
