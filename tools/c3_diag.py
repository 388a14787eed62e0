"""Config c3 (Helmholtz kappa = 40, 256^2, tol 1e-8) accuracy diagnostics:
E = ||f - H x|| / ||f|| of the one-shot inverse and after residual
correction, with the non-leaf F inverted by block elimination (default) or by
a Gauss-Jordan inverse of the assembled F (--noblock), and the E/G condition
per level.

    python tools/c3_diag.py [--noblock] [--n 256]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1303_5466_b200 as P
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--noblock", action="store_true")
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--steps", type=int, default=None)
ap.add_argument("--cond", type=float, default=None)
a = ap.parse_args()
if a.steps is not None:
    sd._REFINE_STEPS = a.steps
if a.cond is not None:
    sd._REFINE_COND = a.cond

if a.noblock:
    orig = sd._invert_level_F

    def no_block(inv, L, checks=None):
        C1 = inv.H.levels[L.lv + 1] if L.lv + 1 < len(inv.H.levels) else None
        if C1 is not None:
            C1.Gkeep = None
        return orig(inv, L, checks)
    sd._invert_level_F = no_block

spec = P.KernelSpec("helmholtz2d", k=20.0,
                    b_field=P.make_field("centre_bump", scale=-400.0, base=0.0, amp=1.0, width=0.09),
                    c_field=P.make_field("one"))
grid = P.Grid(a.n)
opts = P.SolverOptions(eps=a.tol, leaf_size=64, k_cut=None)
tree = P.build_tree(grid, 64)
H = sd.compress_outer(spec, grid, tree, a.tol, opts, P.PLAIN)
inv = sd.invert_dense_block(H)
f = np.exp(1j * 20.0 * (grid.points()[:, 0] + 1.0))
x = inv.apply(f)
es = []
for r in range(3):
    es.append(float(np.linalg.norm(f - H.matvec(x)) / np.linalg.norm(f)))
    x = x + inv.apply(f - H.matvec(x))
print(f"n={a.n} noblock={a.noblock} steps={sd._REFINE_STEPS} cond={sd._REFINE_COND:.0e}: "
      f"E per round {['%.2e' % e for e in es]}; refined levels "
      f"{[L.lv for L in H.levels if getattr(L, 'refine', False)]}")
for L in H.levels[1:]:
    E = getattr(L, "E", None)
    if E is None:
        continue
    nE = [float(torch.linalg.matrix_norm(E[b, :int(L.k[b]), :int(L.k[b])], 2)) for b in range(min(L.nb, 64))]
    print(f"L{L.lv:02d} nb={L.nb} kmax={int(L.kmax)} max||E||_2={max(nE):.2e} "
          f"pivot spread {getattr(L, 'cond_est', float('nan')):.2e}")
# realified skeletons: fraction of skeleton unknowns (2 point + component)
# whose partner component is not a skeleton unknown, per level
for L in H.levels[1:]:
    tot = unp = 0
    for i in L.ids[:64]:
        s = np.asarray(H.row_skel[int(i)])
        tot += s.size
        unp += np.setdiff1d(s ^ 1, s).size
    print(f"L{L.lv:02d} unpaired skeleton fraction {unp / max(tot, 1):.3f}")
