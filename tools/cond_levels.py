"""Per-level conditioning estimate (pivot spread of the F eliminations) and
refinement flags of the bench problem (c4 operator) at --n."""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field
from paper_1303_5466_b200 import solver_dense as sd
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=int, default=512); a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(a.n)
H, inv = sd.factorize(spec, grid, build_tree(grid, 64), 1e-10, SolverOptions(eps=1e-10, leaf_size=64, k_cut=None), CELL)
for L in H.levels:
    print(f"L{L.lv:02d} nb={L.nb} pivot spread {getattr(L, 'cond_est', float('nan')):.3e} refine={getattr(L, 'refine', None)}")
