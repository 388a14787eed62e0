"""One large square DGEMM launch (mainloop efficiency) for an ncu capture."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import _lib
_lib.require_cuda()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else n
A = torch.randn(k, n, dtype=torch.float64, device="cuda")
B = torch.randn(n, k, dtype=torch.float64, device="cuda")
C = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    _lib.gemm(A, B, C, M=n, N=n, K=k, lda=n, ldb=k, ldc=n, alpha=1.0, beta=1.0)
torch.cuda.synchronize()
print("ok")
