"""Per-level stage timings of the B200 HSS-D factor/solve (CUDA events)."""
import argparse, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, CELL
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
for rep in range(a.reps):
    sd.TIMER = sd.StageTimer()
    torch.cuda.synchronize(); t0 = time.time()
    tree = build_tree(grid, 64)
    H = sd.compress_outer(spec, grid, tree, 1e-10, opts, CELL)
    inv = sd.invert_dense_block(H)
    torch.cuda.synchronize(); t1 = time.time()
    rep_ = sd.TIMER.report()
    sd.TIMER = None
    f = torch.randn(a.n * a.n, a.nrhs, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t2 = time.time()
    x = inv.apply(f)
    torch.cuda.synchronize(); t3 = time.time()
    print(f"n={a.n}: factor {t1-t0:.3f}s  solve(nrhs={a.nrhs}) {t3-t2:.4f}s  mem {torch.cuda.max_memory_allocated()/1e9:.1f} GB", flush=True)
    for tag, ms in rep_:
        print(f"  {tag:>14s} {ms:9.2f} ms")
    ks = {L.lv: (L.nb, int(L.mmax), int(getattr(L, 'kmax', 0))) for L in H.levels}
    print("  levels (nb, mmax, kmax):", ks)
    r = x[:, 0] if x.dim() > 1 else x
    del H, inv, x, f
    torch.cuda.empty_cache()
if os.environ.get("VF_PROF"):
    from paper_1303_5466_b200 import _lib
    _lib.prof_enable(True)
    tree = build_tree(grid, 64)
    torch.cuda.synchronize(); t0 = time.time()
    H = sd.compress_outer(spec, grid, tree, 1e-10, opts, CELL)
    inv = sd.invert_dense_block(H)
    torch.cuda.synchronize(); t1 = time.time()
    _lib.prof_prefix("")
    _lib.prof_mark("solve1")
    x = inv.apply(torch.randn(grid.n, 1, dtype=torch.float64, device="cuda"))
    _lib.prof_mark("solve256")
    x = inv.apply(torch.randn(grid.n, 256, dtype=torch.float64, device="cuda"))
    _lib.prof_flush()
    print(f"profiled factor {t1-t0:.3f}s")
    print(_lib.prof_report())
