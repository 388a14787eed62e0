"""Per-level timing of the batched ID (vief_id_batched) inside one
compress_outer of the bench problem: every _id_batched call is bracketed by
CUDA events on the library stream (the call itself synchronises), and the
level's rank sum / skeleton digest are printed so two builds or two settings
can be compared (A/B of ID kernels on the real matrices).

    python tools/id_levels.py [--n 1024] [--reps 2]
"""
import argparse, hashlib, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, CELL, _lib
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
rows = []
orig = sd._id_batched


def timed(dev, A, sA, ldA, pv, mv, maxp, mm, count, g, eps, rank, perm, T, seed, forced, *args, **kw):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    orig(dev, A, sA, ldA, pv, mv, maxp, mm, count, g, eps, rank, perm, T, seed, forced, *args, **kw)
    e1.record()
    torch.cuda.synchronize()
    r = rank.cpu().numpy()
    dig = hashlib.sha1(perm.cpu().numpy().tobytes()).hexdigest()[:10]
    rows.append((count, maxp, mm, e0.elapsed_time(e1), int(r.sum()), dig))


sd._id_batched = timed
for rep in range(a.reps):
    rows.clear()
    torch.cuda.synchronize()
    H = sd.compress_outer(spec, grid, build_tree(grid, 64), 1e-10, opts, CELL)
    torch.cuda.synchronize()
    tot = sum(r[3] for r in rows)
    print(f"rep {rep}: ID total {tot:.1f} ms")
    for count, maxp, mm, ms, ks, dig in rows:
        print(f"  count {count:6d}  p {maxp:5d}  m {mm:5d}  {ms:8.2f} ms  sum k {ks:9d}  perm {dig}")
    del H
    torch.cuda.empty_cache()
