"""A/B timing of the panel kernels inside batched GJ inversion and the ID
(VF_PANEL=cl|rr selects the implementation; the profiler splits phases)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1303_5466_b200 import _lib
from paper_1303_5466_b200.dense_core import interp_decomp_batched

ap = argparse.ArgumentParser()
ap.add_argument("--inv", default="64x16384,250x4096,500x1024,1000x256,3000x16,6000x2,12000x1")
ap.add_argument("--id", default="160x64x16384,288x180x8192,800x496x1024,2080x1520x128,8208x8176x4")
a = ap.parse_args()
_lib.require_cuda()
_lib.prof_enable(True)
g = torch.Generator(device="cuda").manual_seed(0)
for spec in a.inv.split(","):
    if not spec: continue
    n, b = map(int, spec.split("x"))
    A0 = torch.randn(b, n, n, dtype=torch.float64, device="cuda", generator=g)
    A0 += 4 * torch.eye(n, dtype=torch.float64, device="cuda")
    for rep in range(2):
        A = A0.clone()
        _lib.prof_prefix(f"inv{n}x{b}.")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.inv_batched(A, n * n, n, n, b)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            fl = 2.0 * n ** 3 * b
            print(f"inv {n}x{b}: {e0.elapsed_time(e1):.2f} ms  {fl / e0.elapsed_time(e1) / 1e9:.2f} TF/s")
    err = (torch.linalg.inv(A0[:2]) - A[:2]).abs().max().item() / A[:2].abs().max().item()
    print(f"  inverse check (first 2): max rel err {err:.2e}")
    torch.cuda.synchronize()
    del A, A0
import ctypes
for spec in a.id.split(","):
    if not spec: continue
    p, m, c = map(int, spec.split("x"))
    k = min(p, m) * 3 // 4
    U = torch.randn(p, k, dtype=torch.float64, device="cuda", generator=g)
    V = torch.randn(k, m, dtype=torch.float64, device="cuda", generator=g)
    V *= torch.logspace(0, -14, k, dtype=torch.float64, device="cuda")[:, None]
    M = (U @ V).t().contiguous()              # column-major p x m (ld = p)
    del U, V
    ldA = p + (p & 1)
    A0 = torch.zeros((c, m, ldA), dtype=torch.float64, device="cuda")
    A0[:, :, :p] = M
    del M
    pv = torch.full((c,), p, dtype=torch.int32, device="cuda")
    mv = torch.full((c,), m, dtype=torch.int32, device="cuda")
    for rep in range(2):
        A = A0.clone()
        rank = torch.zeros(c, dtype=torch.int32, device="cuda")
        perm = torch.zeros((c, m), dtype=torch.int32, device="cuda")
        T = torch.zeros((c, m, m), dtype=torch.float64, device="cuda")
        d = _lib.IdDesc(_lib.ptr(A), m * ldA, ldA, _lib.ptr(pv), _lib.ptr(mv), p, m, c, 2, 1e-10,
                        _lib.ptr(rank), _lib.ptr(perm), _lib.ptr(T), m * m, m, 0,
                        int(os.environ.get("VF_FB", "1")))
        _lib.prof_prefix(f"id{p}x{m}x{c}.")
        _lib.call("vief_id_batched", ctypes.byref(d), _lib.stream_handle())
        torch.cuda.synchronize()
        del A, T
    del A0
_lib.prof_prefix("")
print(_lib.prof_report())
