import sys, os, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1303_5466_b200 import _lib
n = 12272
A0 = torch.randn(1, n, n, dtype=torch.float64, device="cuda") + 4 * torch.eye(n, dtype=torch.float64, device="cuda")
s2 = torch.cuda.Stream()
for name, st in [("default", torch.cuda.current_stream()), ("side", s2), ("default", torch.cuda.current_stream()), ("side", s2)]:
    A = A0.clone()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t = time.perf_counter()
        _lib.inv_batched(A, n * n, n, n, 1)
        th = time.perf_counter() - t
        e1.record()
    torch.cuda.synchronize()
    print(name, f"gpu {e0.elapsed_time(e1):.1f} ms  host enqueue {th*1e3:.1f} ms")
