import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import _lib
for n in (3, 49):
    A = torch.zeros(1, n, n, dtype=torch.float64, device="cuda")
    A[0, 0, 0] = 1.0
    pmin, pmax = _lib.inv_batched(A, n * n, n, n, 1)
    torch.cuda.synchronize()
    print(n, float(pmin[0]), float(pmax[0]), flush=True)
A = torch.zeros(1, 49, 49, dtype=torch.float64, device="cuda")
pmin, pmax = _lib.inv_batched(A, 49 * 49, 49, 49, 1)
torch.cuda.synchronize()
print("zero", float(pmin[0]), float(pmax[0]))
