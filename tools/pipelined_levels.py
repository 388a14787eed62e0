"""Per-level time of the compression (main) stream inside the PIPELINED
factor_solve of the bench problem (StageTimer marks on the main stream), next
to the same marks of a back-to-back compress_outer: shows how much the ID
chain stretches when the inversion / sweep streams share the GPU.

    python tools/pipelined_levels.py [--n 1024] [--nrhs 256] [--reps 2]
"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, CELL
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
F = torch.randn(grid.n, a.nrhs, dtype=torch.float64, device="cuda")
for rep in range(a.reps + 1):
    sd.TIMER = sd.StageTimer() if rep else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    H, inv, X = sd.factor_solve(spec, grid, build_tree(grid, 64), 1e-10, opts, F, CELL)
    e1.record()
    torch.cuda.synchronize()
    if rep:
        r = sd.TIMER.report()
        sd.TIMER = None
        tot = sum(ms for t, ms in r if t.startswith("compress:"))
        print(f"rep {rep}: step {e0.elapsed_time(e1):.1f} ms, compression stream {tot:.1f} ms, "
              f"tail {e0.elapsed_time(e1) - tot:.1f} ms")
        print("   " + "  ".join(f"{t.split(':')[1]}:{ms:.0f}" for t, ms in r if t.startswith("compress:")))
    del H, inv, X
