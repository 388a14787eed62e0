"""Time DenseBlockInverse.apply on the bench problem after one factorization:
256 RHS and 1 RHS, CUDA events; reports the root's storage form."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field
from paper_1303_5466_b200 import solver_dense as sd
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=int, default=1024); a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
H = sd.compress_outer(spec, grid, build_tree(grid, 64), 1e-10, opts, CELL)
inv = sd.invert_dense_block(H)
print("root block form:", getattr(H.levels[0], "rb", None) is not None,
      "refined:", [L.lv for L in H.levels if getattr(L, "refine", False)])
for r in (256, 1):
    F = torch.randn((grid.n, r), dtype=torch.float64, device="cuda")
    inv.apply(F)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); inv.apply(F); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"apply nrhs={r}: {['%.1f' % t for t in ts]} ms")
