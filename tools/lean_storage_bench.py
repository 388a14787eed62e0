"""ID path (k_cut = None, the headline path) at the bench problem with dense vs
lean factor storage (invert_dense_block(storage=)): factor bytes, peak
allocation, sequential factor time, solve times, residual.

    python tools/lean_storage_bench.py [--n 1024] [--nrhs 256]
"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1303_5466_b200 as P
from paper_1303_5466_b200 import solver_dense as sd
from paper_1303_5466_b200.verify import FFTOperator

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=256)
a = ap.parse_args()
spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                    c_field=P.make_field("one"))
grid = P.Grid(a.n)
opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
F = torch.randn(grid.n, a.nrhs, dtype=torch.float64, device="cuda")
f1 = F[:, :1].contiguous()
op = FFTOperator(spec, grid, P.CELL, "cuda")
out = {"n_side": a.n, "N": grid.n, "nrhs": a.nrhs}


def t():
    torch.cuda.synchronize()
    return time.time()


for storage in ("dense", "lean", "dense", "lean"):
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    t0 = t()
    H = sd.compress_outer(spec, grid, P.build_tree(grid, 64), 1e-10, opts, P.CELL)
    t1 = t()
    inv = sd.invert_dense_block(H, free_source=True, storage=storage)
    t2 = t()
    inv.apply(f1)
    t3 = t()
    x1 = inv.apply(f1)
    t4 = t()
    X = inv.apply(F)
    t5 = t()
    X = inv.apply(F)
    t6 = t()
    res = float(((F[:, :4] - op.matvec(X[:, :4])).norm(dim=0) / F[:, :4].norm(dim=0)).max())
    out[storage] = {"compress_s": t1 - t0, "invert_s": t2 - t1, "solve1_s": t4 - t3,
                    f"solve{a.nrhs}_s": t6 - t5, "factor_bytes": inv.nbytes(),
                    "reference_layout_bytes": inv.nbytes_reference_layout() if storage == "dense" else None,
                    "peak_alloc": torch.cuda.max_memory_allocated(), "true_residual_fft": res}
    del H, inv, X, x1
print(json.dumps(out))
