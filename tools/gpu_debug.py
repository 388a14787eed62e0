"""Quick end-to-end debug run (not a test)."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, PLAIN, CELL
from paper_1303_5466_b200.solver_dense import compress_outer, invert_dense_block
from paper_1303_5466_b200.kernels import assemble_dense

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

def case(name, spec, n, leaf, eps, quad, force=0):
    gold = np.load(os.path.join(G, f"solve_{name}.npz"))
    grid = Grid(n)
    opts = SolverOptions(eps=eps, leaf_size=leaf, k_cut=None)
    torch.cuda.synchronize(); t0 = time.time()
    tree = build_tree(grid, leaf)
    from paper_1303_5466_b200 import solver_dense as sd
    H = sd.Hss2dMatrix.__new__(sd.Hss2dMatrix)
    H = compress_outer(spec, grid, tree, eps, opts, quad) if not force else None
    torch.cuda.synchronize(); t1 = time.time()
    inv = invert_dense_block(H)
    torch.cuda.synchronize(); t2 = time.time()
    f = gold["f"]
    x = inv.apply(f)
    torch.cuda.synchronize(); t3 = time.time()
    xr = gold["x"]
    err = np.linalg.norm(x - xr) / np.linalg.norm(xr)
    res = np.linalg.norm(f - H.matvec(x)) / np.linalg.norm(f)
    ranks = np.array([H.levels[0].k[0] if False else 0])
    rk = {int(i): int(L.k[j]) for L in H.levels if L.lv > 0 for j, i in enumerate(L.ids)}
    gr = gold["rank"]
    dr = np.array([rk[i] - gr[i] for i in rk] or [0])
    print(f"{name}: compress {t1-t0:.3f}s invert {t2-t1:.3f}s apply {t3-t2:.3f}s "
          f"relerr vs ref {err:.2e} resid {res:.2e} rank diff min {dr.min()} max {dr.max()} "
          f"nbytes {inv.nbytes_reference_layout()} vs ref {int(gold['nbytes_inv'])}", flush=True)
    if "x_dense" in gold.files:
        e2 = np.linalg.norm(x - gold["x_dense"]) / np.linalg.norm(gold["x_dense"])
        print(f"   vs dense solve {e2:.2e}")

nti = KernelSpec("laplace2d", b_field=make_field("gaussian_bump"), c_field=make_field("gaussian_bump"))
rows = KernelSpec("laplace2d", b_field=make_field("gaussian_bump"), c_field=make_field("one"))
import math
c1 = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
case("single7", nti, 7, 49, 1e-10, PLAIN)
case("nti28", nti, 28, 49, 1e-10, PLAIN)
case("rows14", rows, 14, 49, 1e-10, PLAIN)
case("rows30", rows, 30, 64, 1e-10, PLAIN)
case("c1_64", c1, 64, 64, 1e-10, CELL)
case("c1_128", c1, 128, 64, 1e-10, CELL)
