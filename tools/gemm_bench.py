"""Throughput of the library's DMMA GEMM vs cuBLAS (torch) on FP64 shapes that
occur in the factorization."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import _lib
_lib.require_cuda()

def bench(M, N, K, batch=1, tA=0, tB=0, beta=1.0):
    A = torch.randn(batch, M if tA else K, K if tA else M, dtype=torch.float64, device="cuda")
    B = torch.randn(batch, K if tB else N, N if tB else K, dtype=torch.float64, device="cuda")
    C = torch.randn(batch, N, M, dtype=torch.float64, device="cuda")
    f = lambda: _lib.gemm(A, B, C, M=M, N=N, K=K, lda=A.shape[2], ldb=B.shape[2], ldc=M,
                          sA=A[0].numel(), sB=B[0].numel(), sC=C[0].numel(), tA=tA, tB=tB,
                          alpha=-1.0, beta=beta, batch=batch)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    # cublas reference
    At = A.transpose(1, 2) if not tA else A
    Bt = B.transpose(1, 2) if not tB else B
    g = lambda: torch.baddbmm(C.transpose(1, 2), At, Bt, alpha=-1.0, beta=beta)
    for _ in range(3): g()
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): g()
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / 10
    fl = 2.0 * M * N * K * batch
    print(f"M={M:6d} N={N:6d} K={K:6d} b={batch:5d} tA={tA} tB={tB}: ours {fl/ms/1e9:7.2f} TF ({ms:8.3f} ms)  cublas {fl/ms2/1e9:7.2f} TF", flush=True)

import sys as _s
if len(_s.argv) > 1 and _s.argv[1] == "hss":
    bench(12272, 12016, 256)                    # GJ outer update at the 1024^2 root
    bench(8208, 8000, 256, batch=4)             # ID delayed update, level 1
    bench(32, 8000, 8208, batch=4, tA=1, beta=0.0)  # ID W = Q^T A, level 1
    bench(3104, 2000, 128, batch=64)            # ID update, level 5
    bench(32, 2000, 3104, batch=64, tA=1, beta=0.0)
    bench(3000, 2744, 256, batch=32)            # GJ outer, level 5
    bench(544, 368, 64, batch=2048)             # ID update, level 10
    bench(40, 32, 8208, batch=4, beta=0.0)      # sketch Z = Omega Q
    bench(8192, 8192, 8192)
    _s.exit(0)
bench(8192, 8192, 8192)
bench(8192, 8192, 128)
bench(12272, 12272, 32)
bench(8192, 8192, 64)
bench(64, 64, 64, batch=16384)
bench(368, 368, 32, batch=1024)
bench(32, 8000, 8208, batch=4, tA=1)
bench(8208, 8000, 32, batch=4)
bench(1024, 2040, 3000, batch=4)
