"""The compressed path (finite k_cut: a-priori skeletons, proxy least-squares
interpolation) timed like bench.py's step on the c4 workload: build_tree +
annotate_skeletons + factor + 256-RHS solve (factor_solve, apriori) at 1024^2,
CUDA events, W warm-up + K timed steps; true residual of 4 RHS columns through
the exact FFT operator.  Prints one JSON line.
Usage: python tools/compressed_bench.py [--n 1024] [--nrhs 256] [--steps 3] [--warmup 3]"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1303_5466_b200 import (CELL, Grid, KernelSpec, SolverOptions, build_tree,  # noqa: E402
                                  make_field)
from paper_1303_5466_b200 import solver_dense as sd  # noqa: E402
from paper_1303_5466_b200.tree import annotate_skeletons  # noqa: E402
from paper_1303_5466_b200.verify import true_residual  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=256)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
n, N = a.n, a.n * a.n
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                  c_field=make_field("one"))
grid = Grid(n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=64)
layers = opts.resolved_layers(spec)
F = torch.randn((N, a.nrhs), dtype=torch.float64, device="cuda",
                generator=torch.Generator(device="cuda").manual_seed(1234))


def step():
    tree = build_tree(grid, 64)
    annotate_skeletons(tree, layers)
    return sd.factor_solve(spec, grid, tree, 1e-10, opts, F, CELL, apriori=layers)


for _ in range(a.warmup):
    out = step()
    del out
times = []
for _ in range(a.steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    H, inv, X = step()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / 1e3)
    if len(times) < a.steps:
        del H, inv, X
res = true_residual(spec, grid, CELL, F[:, :4].cpu().numpy(), X[:, :4].cpu().numpy()
                    if hasattr(X, "cpu") else X[:, :4])
t = sum(times) / len(times)
print(json.dumps({"path": "compressed (k_cut=64, a-priori skeletons, dense blocks)",
                  "metric": "factor & solve unknowns/sec", "value": N / t, "unit": "unknowns/s",
                  "s_per_step": t, "steps": a.steps, "warmup": a.warmup, "n_side": n,
                  "nrhs": a.nrhs, "true_residual_max": float(max(res)),
                  "factor_bytes": int(inv.nbytes()), "times": times}))
