"""Time the compressed (finite k_cut, a-priori skeleton) path on the B200:
factor + 1-RHS solve at the given sizes, with the true residual (FFT operator)
and the per-stage split.  Usage: python tools/compressed_run.py 256 512 1024"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1303_5466_b200 as P  # noqa: E402
from paper_1303_5466_b200.solver_compressed import compress_inverse  # noqa: E402
from paper_1303_5466_b200.verify import true_residual  # noqa: E402

spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
for n in [int(a) for a in sys.argv[1:]] or [256]:
    grid = P.Grid(n)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=64)
    f = np.random.default_rng(0).standard_normal(grid.n)
    for rep in range(2):
        tree = P.build_tree(grid, 64)
        t0 = time.perf_counter()
        from paper_1303_5466_b200.tree import annotate_skeletons
        annotate_skeletons(tree, opts.resolved_layers(spec))
        t1 = time.perf_counter()
        inv = compress_inverse(spec, grid, tree=tree, eps=1e-10, opts=opts)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        x = inv.apply(f)
        t3 = time.perf_counter()
        res = true_residual(spec, grid, P.PLAIN, f, x)
        H = inv.dense_matvec_source
        kmax = max(int(L.k.max()) for L in H.levels if L is not None and hasattr(L, "k"))
        print(f"n={n} rep={rep} annotate {t1 - t0:.3f} s factor {t2 - t1:.3f} s "
              f"solve(1 rhs, host) {t3 - t2:.3f} s  N/(annot+factor) "
              f"{grid.n / (t2 - t0):.4g} unknowns/s  true residual {res:.2e}  max k {kmax}  "
              f"factor bytes {inv.nbytes() / 1e9:.2f} GB", flush=True)
        del inv, H, x
        torch.cuda.empty_cache()
