"""Reference solutions of config c1 at 256^2 and 512^2 (SURVEY.md §8(c) item 2:
side-by-side runs at 128^2..1024^2; 1024^2 is hours of reference CPU time and
is checked by residuals only).  Imports the reference from /root/reference
(build container only).  To keep the fixtures small the right-hand side is
NOT stored: it is np.random.default_rng(seed).standard_normal(N), regenerated
by the test; only the solution, the per-box ranks and nbytes are kept.

    OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_big.py [256 512]
"""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import CELL, OUT, bump  # noqa: E402  (also puts the reference on sys.path)
from vief import Grid, KernelSpec, SolverOptions, build_tree, make_field  # noqa: E402
from vief.solver_dense import compress_outer, invert_dense_block  # noqa: E402


def run(n, seed=0):
    spec = KernelSpec("laplace2d", b_field=bump(math.pi / 2), c_field=make_field("one"))
    grid = Grid(n)
    opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    t0 = time.perf_counter()
    tree = build_tree(grid, 64)
    H = compress_outer(spec, grid, tree, 1e-10, opts, CELL)
    t1 = time.perf_counter()
    inv = invert_dense_block(H)
    t2 = time.perf_counter()
    f = np.random.default_rng(seed).standard_normal(grid.n)
    x = inv.apply(f)
    t3 = time.perf_counter()
    nb = len(tree.nodes)
    rank = np.array([H.row_skel[i].size if i in H.row_skel else -1 for i in range(nb)], np.int32)
    np.savez_compressed(os.path.join(OUT, f"solve_c1_{n}.npz"), x=x, seed=np.int64(seed),
                        rank=rank, nbytes_inv=np.int64(inv.nbytes()),
                        times=np.array([t1 - t0, t2 - t1, t3 - t2]))
    print(f"c1_{n}: compress {t1-t0:.1f}s invert {t2-t1:.1f}s apply {t3-t2:.2f}s "
          f"max rank {rank.max()} nbytes {inv.nbytes()}", flush=True)


if __name__ == "__main__":
    for n in [int(a) for a in sys.argv[1:]] or [256, 512]:
        run(n)
