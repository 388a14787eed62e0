"""One sequential factorization of the bench problem (c4 operator) with NVTX
ranges around every level's phases, for ncu filtering
(`--nvtx --nvtx-include "id_L01/"` etc.):

    blocks_Lxx   K1 entry generation of D/B blocks       (_compress_level_blocks)
    id_Lxx       proxy/near sources, K1 ID matrices, K2 ID (_compress_level_id)
    finv_Lxx     F^-1 (Gauss-Jordan / block elimination)  (_invert_level_F)
    wgec_Lxx     W, G, E = G^-1, C                        (_invert_level_rest)

    python tools/ncu_levels.py [--n 1024]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
a = ap.parse_args()


def ranged(tag, fn):
    def wrap(*args, **kw):
        L = next(x for x in args if isinstance(x, sd._Level))
        torch.cuda.nvtx.range_push(f"{tag}_L{L.lv:02d}")
        try:
            return fn(*args, **kw)
        finally:
            torch.cuda.nvtx.range_pop()
    return wrap


sd._compress_level_blocks = ranged("blocks", sd._compress_level_blocks)
sd._compress_level_id = ranged("id", sd._compress_level_id)
sd._invert_level_F = ranged("finv", sd._invert_level_F)
sd._invert_level_rest = ranged("wgec", sd._invert_level_rest)

spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                  c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
H = sd.compress_outer(spec, grid, build_tree(grid, 64), 1e-10, opts, CELL)
inv = sd.invert_dense_block(H)
torch.cuda.synchronize()
print("ok", [(L.lv, int(L.kmax)) for L in H.levels if L.lv > 0][:4])
