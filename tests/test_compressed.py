"""Compressed (finite k_cut) path, CPU side: the a-priori skeleton split
(tree.annotate_skeletons) pinned bit-exact to the reference's
(tests/golden/compressed.npz from make_golden_compressed.py), and the CPU
oracle's a-priori solve (oracle/hssd.py compress_apriori) pinned to the
reference's compressed solutions.  The reference stores the large blocks in
eps-accurate 1-D HSS form, so solutions agree to ~eps * cond, not bitwise:
the tolerance is 1e-8 relative (the reference's own residual bar,
test_solver_compressed.py:187-200)."""
import os

import numpy as np
import pytest

G = os.path.join(os.path.dirname(__file__), "golden")
GOLD = np.load(os.path.join(G, "compressed.npz"))
ANN = [(28, 49, 2), (56, 49, 2), (32, 64, 2), (64, 64, 1)]
CASES = {  # name: (n, leaf, b field, c field)
    "nti28_k8": (28, 49, "gaussian_bump", "gaussian_bump"),
    "nti28_k64": (28, 49, "gaussian_bump", "gaussian_bump"),
    "nonsym28_k8": (28, 49, "gaussian_bump", "one"),
    "ti28_k8": (28, 49, "one", "one"),
    "nti56_k64": (56, 49, "gaussian_bump", "gaussian_bump"),
    "nonsym64_leaf64": (64, 64, "gaussian_bump", "one"),
}


def _split(key):
    nsk, nrs = GOLD[key + "_nsk"], GOLD[key + "_nrs"]
    osk = np.concatenate([[0], np.cumsum(nsk)])
    ors = np.concatenate([[0], np.cumsum(nrs)])
    op = np.concatenate([[0], np.cumsum(nsk + nrs)])
    for b in range(nsk.size):
        yield (b, GOLD[key + "_sk"][osk[b]:osk[b + 1]], GOLD[key + "_rs"][ors[b]:ors[b + 1]],
               GOLD[key + "_perm"][op[b]:op[b + 1]])


@pytest.mark.parametrize("n,leaf,layers", ANN)
def test_annotate_skeletons_matches_reference(n, leaf, layers):
    from paper_1303_5466_b200 import Grid, build_tree
    from paper_1303_5466_b200.tree import annotate_skeletons
    tree = build_tree(Grid(n), leaf)
    annotate_skeletons(tree, layers)
    for b, sk, rs, perm in _split(f"ann_{n}_{leaf}_{layers}"):
        node = tree.nodes[b]
        np.testing.assert_array_equal(node.sk_idx, sk)
        np.testing.assert_array_equal(node.rs_idx, rs)
        np.testing.assert_array_equal(node.work_perm, perm)
        np.testing.assert_array_equal(np.concatenate([sk, rs]), node.full_idx[perm])


@pytest.mark.parametrize("n,leaf,layers", ANN)
def test_oracle_annotate_matches_reference(n, leaf, layers):
    import oracle.hssd as O
    ann = O.annotate(O.make_tree(n, leaf), layers)
    for b, sk, rs, perm in _split(f"ann_{n}_{leaf}_{layers}"):
        np.testing.assert_array_equal(ann[b][0], sk)
        np.testing.assert_array_equal(ann[b][1], rs)
        np.testing.assert_array_equal(ann[b][2], perm)


def test_annotate_interior_retention_matches_reference():
    """Oscillatory kernels keep an interface sublattice (tree.py:221-234)."""
    from paper_1303_5466_b200 import Grid, build_tree
    from paper_1303_5466_b200.tree import annotate_skeletons
    tree = build_tree(Grid(64), 64)
    annotate_skeletons(tree, 3, k_wave=101.0, points_per_wavelength=0.5)
    key = "ann_64_64_3_kw101"
    for b, sk, rs, perm in _split(key):
        node = tree.nodes[b]
        np.testing.assert_array_equal(node.sk_idx, sk)
        np.testing.assert_array_equal(node.rs_idx, rs)
        np.testing.assert_array_equal(node.work_perm, perm)
    np.testing.assert_array_equal([nd.n_interior_sk for nd in tree.nodes], GOLD[key + "_nint"])
    assert GOLD[key + "_nint"].max() > 0


def test_support_mask_drops_skeletons():
    from paper_1303_5466_b200 import Grid, build_tree
    from paper_1303_5466_b200.tree import annotate_skeletons
    grid = Grid(28)
    mask = np.ones(grid.n, bool)
    mask[::3] = False
    tree = annotate_skeletons(build_tree(grid, 49), 2, support_mask=mask)
    for node in tree.nodes:
        assert mask[node.sk_idx].all()
        assert np.array_equal(np.sort(np.concatenate([node.sk_idx, node.rs_idx])),
                              np.sort(node.full_idx))


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_apriori_solve_matches_reference(name):
    import oracle.hssd as O
    n, leaf, b, c = CASES[name]
    P = O.Problem(n, "laplace2d", 0.0, ("one", ()), (b, ()), (c, ()), "none")
    f = GOLD[f"solve_{name}_f"]
    x, _, _ = O.solve_apriori(P, leaf, 2, f)
    xr = GOLD[f"solve_{name}_x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-8
    A = O.dense_matrix(P)
    assert np.linalg.norm(A @ x - f) / np.linalg.norm(f) <= 1e-8


def test_ti_mode_rejects_nti_spec():
    from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, make_field
    from paper_1303_5466_b200.errors import ConfigError
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    spec = KernelSpec("laplace2d", b_field=make_field("gaussian_bump"),
                      c_field=make_field("gaussian_bump"))
    with pytest.raises(ConfigError):
        compress_inverse(spec, Grid(28), eps=1e-10, opts=SolverOptions(), ti_mode=True)
