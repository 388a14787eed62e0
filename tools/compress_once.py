"""One compress_outer (the ID stage) of the n^2 benchmark problem, for ncu
captures of individual ID kernels (filter with -k / --launch-skip)."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                  c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
H = sd.compress_outer(spec, grid, build_tree(grid, 64), 1e-10, opts, CELL)
torch.cuda.synchronize()
print("ok", {L.lv: int(L.kmax) for L in H.levels if L.lv})
