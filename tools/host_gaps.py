"""Host-side time of the compression loop outside vief_id_batched, per level,
in the pipelined factor_solve (wall clock around the Python stages: the ID
chain is the critical path, so host time between two levels' ID calls
extends the step).

    python tools/host_gaps.py [--n 1024]
"""
import argparse, math, os, sys, time
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
F = torch.randn(grid.n, 256, dtype=torch.float64, device="cuda")
T = {}


def wrap(name):
    orig = getattr(sd, name)

    def f(*args, **kw):
        t = time.perf_counter()
        r = orig(*args, **kw)
        T.setdefault(name, []).append(time.perf_counter() - t)
        return r
    setattr(sd, name, f)


for nm in ("_compress_level_blocks", "_compress_level_id", "_id_batched", "_level_sources"):
    wrap(nm)
for rep in range(3):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = build_tree(grid, 64)
    t1 = time.perf_counter()
    H, inv, X = sd.factor_solve(spec, grid, tree, 1e-10, opts, F, CELL)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {rep}: build_tree {1e3*(t1-t0):.1f} ms, factor_solve host {1e3*(t2-t1):.1f} ms, + sync {1e3*(t3-t2):.1f} ms")
    for nm, v in T.items():
        print(f"  {nm:24s} total {1e3*sum(v):7.1f} ms   per level: " + " ".join(f"{1e3*x:.1f}" for x in v))
    del H, inv, X
