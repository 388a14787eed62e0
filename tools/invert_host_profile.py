"""Host-side profile (cProfile) of the sequential invert_dense_block at 1024^2:
where the Python time of the inversion stage goes (the GPU phases of levels
13/14 sum to ~19/13 ms while their wall time is 57/40 ms).

    python tools/invert_host_profile.py [--n 1024]
"""
import argparse, cProfile, math, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, CELL
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
tree = build_tree(grid, 64)
for rep in range(2):
    H = sd.compress_outer(spec, grid, tree, 1e-10, opts, CELL)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    inv = sd.invert_dense_block(H)
    pr.disable()
    t1 = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"rep {rep}: invert host {t1 * 1e3:.1f} ms, with sync {(time.perf_counter() - t) * 1e3:.1f} ms")
    del inv, H
    torch.cuda.empty_cache()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
