"""Representative DMMA GEMM launches for an ncu --set full capture: the
Gauss-Jordan outer update at the 1024^2 root (12272 x 12144 x 128, beta=1)
and the ID delayed trailing update at level 1 (4 x 8208 x 8000 x 128)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import _lib
_lib.require_cuda()
n = 12272
A = torch.randn(128, n, dtype=torch.float64, device="cuda")       # X (n x 128) col-major
B = torch.randn(n, 128, dtype=torch.float64, device="cuda")       # R (128 x n) col-major
C = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.gemm(A, B, C, M=n, N=n - 128, K=128, lda=n, ldb=128, ldc=n, alpha=1.0, beta=1.0)
p, m = 8208, 8000
Q = torch.randn(4, 128, p, dtype=torch.float64, device="cuda")
W = torch.randn(4, m, 128, dtype=torch.float64, device="cuda")
Am = torch.randn(4, m, p, dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.gemm(Q, W, Am, M=p, N=m, K=128, lda=p, ldb=128, ldc=p, sA=128 * p, sB=m * 128,
              sC=m * p, alpha=-1.0, beta=1.0, batch=4)
torch.cuda.synchronize()
print("ok")
