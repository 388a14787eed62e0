"""HBM bandwidth of the library's batched notrans GEMV (the 1-RHS solve sweeps)
on the per-level factor shapes of the 1024^2 problem, vs torch (cuBLAS) bmm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import _lib

_lib.require_cuda()


def bench(M, K, batch, reps=20):
    A = torch.randn(batch, K, M, dtype=torch.float64, device="cuda")  # column-major M x K
    x = torch.randn(batch, K, dtype=torch.float64, device="cuda")
    y = torch.zeros(batch, M, dtype=torch.float64, device="cuda")
    f = lambda: _lib.gemv(A, x, y, M=M, K=K, lda=M, sA=M * K, sx=K, sy=M, alpha=1.0, beta=0.0,
                          batch=batch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = torch.bmm(A.transpose(1, 2), x.unsqueeze(2)).squeeze(2)
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    g = lambda: torch.bmm(A.transpose(1, 2), x.unsqueeze(2))
    for _ in range(3):
        g()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g()
    e1.record()
    torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / reps
    gb = 8.0 * M * K * batch / 1e9
    print(f"M={M:6d} K={K:6d} batch={batch:6d} ({gb:6.2f} GB): ours {gb / ms * 1e3:7.1f} GB/s "
          f"({ms:7.3f} ms)  torch {gb / ms2 * 1e3:7.1f} GB/s  err {err:.1e}", flush=True)


# level shapes at 1024^2: (m, k) per level, 2^l boxes
for M, K, b in [(8176, 8176, 2), (6136, 8176, 2), (8176, 6136, 2), (6136, 6136, 2),
                (6128, 6128, 4), (4100, 6128, 8), (4096, 4096, 16), (2048, 2048, 64),
                (1024, 1024, 256), (512, 512, 1024), (256, 256, 4096), (128, 128, 8192),
                (64, 64, 16384), (60, 64, 16384), (12272, 12272, 1)]:
    bench(M, K, b)
