"""One batched Gauss-Jordan inversion (vief_inv_batched) of `batch` random
n x n matrices (diagonally weighted), timed; for ncu captures of the GJ
kernels (filter with -k / --launch-skip).

python tools/gj_case.py [--n 6136] [--batch 2] [--reps 3]
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=6136)
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
_lib.require_cuda()
n, b = a.n, a.batch
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn((b, n, n), dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
A0 += 4.0 * torch.eye(n, dtype=torch.float64, device="cuda")
for r in range(a.reps):
    A = A0.clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pmin, pmax = _lib.inv_batched(A, n * n, n, n, b)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"n={n} batch={b}: {dt*1e3:.2f} ms  {2.0*n**3*b/dt/1e12:.2f} TF/s (2n^3)", flush=True)
I = torch.eye(n, dtype=torch.float64, device="cuda")
# A holds the inverse of A0 stored column-major per item: check A0^T-layout consistency
err = max(float(torch.linalg.norm(A0[i].t() @ A[i].t() - I) / n ** 0.5) for i in range(b))
print("inverse residual", err)
