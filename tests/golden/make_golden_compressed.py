"""Golden fixtures for the compressed (finite k_cut) path, made by running the
REFERENCE implementation (build container only; needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_compressed.py

Writes tests/golden/compressed.npz:
  * ann_<n>_<leaf>_<layers>_{sk,rs,perm,nsk,nrs}: annotate_skeletons output
    (tree.py:237-269) for every box in breadth-first order, concatenated;
  * solve_<case>_{f,x,nbytes}: compress_inverse(k_cut finite).apply(f)
    (solver_compressed.py:514-591) for the cases below.
"""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from vief import Grid, KernelSpec, SolverOptions, build_tree, make_field  # noqa: E402
from vief.solver_compressed import compress_inverse  # noqa: E402
from vief.tree import annotate_skeletons  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

BUMP = make_field("gaussian_bump")
ONE = make_field("one")
CASES = {
    # name: (n, leaf, k_cut, b, c, ti_mode, rhs seed)
    "nti28_k8": (28, 49, 8, BUMP, BUMP, False, 1),
    "nti28_k64": (28, 49, 64, BUMP, BUMP, False, 1),
    "nonsym28_k8": (28, 49, 8, BUMP, ONE, False, 5),
    "ti28_k8": (28, 49, 8, ONE, ONE, True, 3),
    "nti56_k64": (56, 49, 64, BUMP, BUMP, False, 7),
    "nonsym64_leaf64": (64, 64, 64, BUMP, ONE, False, 0),
}


def main():
    out = {}
    for n, leaf, layers in [(28, 49, 2), (56, 49, 2), (32, 64, 2), (64, 64, 1)]:
        tree = build_tree(Grid(n), leaf)
        annotate_skeletons(tree, layers)
        key = f"ann_{n}_{leaf}_{layers}"
        out[key + "_sk"] = np.concatenate([b.sk_idx for b in tree.nodes])
        out[key + "_rs"] = np.concatenate([b.rs_idx for b in tree.nodes])
        out[key + "_perm"] = np.concatenate([b.work_perm for b in tree.nodes])
        out[key + "_nsk"] = np.array([b.sk_idx.size for b in tree.nodes])
        out[key + "_nrs"] = np.array([b.rs_idx.size for b in tree.nodes])
    # oscillatory retention (tree.py:221-234): kappa >= 16, stride 3 at 64^2
    tree = build_tree(Grid(64), 64)
    annotate_skeletons(tree, 3, k_wave=101.0, points_per_wavelength=0.5)
    key = "ann_64_64_3_kw101"
    out[key + "_sk"] = np.concatenate([b.sk_idx for b in tree.nodes])
    out[key + "_rs"] = np.concatenate([b.rs_idx for b in tree.nodes])
    out[key + "_perm"] = np.concatenate([b.work_perm for b in tree.nodes])
    out[key + "_nsk"] = np.array([b.sk_idx.size for b in tree.nodes])
    out[key + "_nrs"] = np.array([b.rs_idx.size for b in tree.nodes])
    out[key + "_nint"] = np.array([b.n_interior_sk for b in tree.nodes])
    # complex: test_solver_compressed.py:243-253 (k = 4 pi, 18^2, leaf 81, k_cut 16)
    spec = KernelSpec("helmholtz2d", k=4 * np.pi)
    grid = Grid(18)
    inv = compress_inverse(spec, grid, eps=1e-10,
                           opts=SolverOptions(eps=1e-10, leaf_size=81, k_cut=16))
    rng = np.random.default_rng(4)
    f = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    out["solve_helm18_f"] = f
    out["solve_helm18_x"] = inv.apply(f)
    for name, (n, leaf, k_cut, b, c, ti, seed) in CASES.items():
        spec = KernelSpec("laplace2d", b_field=b, c_field=c)
        grid = Grid(n)
        opts = SolverOptions(eps=1e-10, leaf_size=leaf, k_cut=k_cut)
        inv = compress_inverse(spec, grid, eps=1e-10, opts=opts, ti_mode=ti)
        f = np.random.default_rng(seed).standard_normal(grid.n)
        out[f"solve_{name}_f"] = f
        out[f"solve_{name}_x"] = inv.apply(f)
        out[f"solve_{name}_nbytes"] = np.array(inv.nbytes())
        print(name, "nbytes", inv.nbytes(), flush=True)
    np.savez_compressed(os.path.join(OUT, "compressed.npz"), **out)


if __name__ == "__main__":
    main()
