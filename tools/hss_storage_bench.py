"""Compressed path (finite k_cut) with dense vs 1-D HSS block storage at the
bench problem: factor bytes, conversion time, solve times, agreement.

    python tools/hss_storage_bench.py [--n 1024] [--nrhs 256]
"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1303_5466_b200 as P
from paper_1303_5466_b200 import compressed_store
from paper_1303_5466_b200.solver_compressed import compress_inverse

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=256)
a = ap.parse_args()
spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                    c_field=P.make_field("one"))
grid = P.Grid(a.n)
opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=64)


def timed(fn):
    torch.cuda.synchronize()
    t = time.time()
    out = fn()
    torch.cuda.synchronize()
    return out, time.time() - t


F = torch.randn(grid.n, a.nrhs, dtype=torch.float64, device="cuda")
f1 = F[:, :1].contiguous()
inv, t_fac = timed(lambda: compress_inverse(spec, grid, eps=1e-10, opts=opts, quad=P.CELL))
inv, t_fac = timed(lambda: compress_inverse(spec, grid, eps=1e-10, opts=opts, quad=P.CELL))
D = inv.factors
nd = D.nbytes()
D.apply(f1)
x1d, t1d = timed(lambda: D.apply(f1))
Xd, tRd = timed(lambda: D.apply(F))
torch.cuda.reset_peak_memory_stats()
nconv, t_conv = timed(lambda: compressed_store.compact(D))
nh = D.nbytes()
D.apply(f1)
x1h, t1h = timed(lambda: D.apply(f1))
Xh, tRh = timed(lambda: D.apply(F))
H = inv.dense_matvec_source
lv = {L.lv: dict(m=int(L.mmax), k=int(L.kmax), nb=int(L.nb),
                 dense_MB=round(compressed_store.level_dense_bytes(L) / 1e6, 1),
                 hss_MB=round(compressed_store.hss_bytes(L) / 1e6, 1),
                 ranks_Finv=[int(x.kmax) for x in L.hss[0].lv[1:]],
                 ranks_E=[int(x.kmax) for x in L.hss[1].lv[1:]])
      for L in H.levels if L is not None and getattr(L, "hss", None) is not None}
print(json.dumps({
    "n_side": a.n, "N": grid.n, "nrhs": a.nrhs, "factor_s": t_fac, "convert_s": t_conv,
    "levels_converted": nconv, "factor_bytes_dense": nd, "factor_bytes_hss1d": nh,
    "solve1_s": {"dense": t1d, "hss1d": t1h}, f"solve{a.nrhs}_s": {"dense": tRd, "hss1d": tRh},
    "rel_diff_1": float((x1h - x1d).norm() / x1d.norm()),
    f"rel_diff_{a.nrhs}": float((Xh - Xd).norm() / Xd.norm()),
    "levels": lv}))
