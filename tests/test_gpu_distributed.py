"""Subtree-sharded factor/solve on one B200 (all shards emulated in this
process, the same phase code that runs one-process-per-GPU over NCCL):
solutions agree with the single-GPU path and with the reference."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_shards_match_reference(world):
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.distributed import ShardedInverse
    g = np.load(os.path.join(G, "solve_c1_128.npz"))
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                        c_field=P.make_field("one"))
    grid = P.Grid(128)
    tree = P.build_tree(grid, 64)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    inv = ShardedInverse(spec, grid, tree, 1e-10, opts, P.CELL, world, emulate=True)
    x = inv.apply(g["f"])
    assert np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]) <= 1e-9


def test_emulated_shards_equal_single_gpu():
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200 import solver_dense as sd
    from paper_1303_5466_b200.distributed import ShardedInverse
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(64)
    tree = P.build_tree(grid, 64)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)  # ID skeletons (HSS-D)
    ref = sd.invert_dense_block(sd.compress_outer(spec, grid, tree, 1e-10, opts))
    f = np.random.default_rng(3).standard_normal((grid.n, 3))
    xr = ref.apply(f)
    for world in (2, 4):
        x = ShardedInverse(spec, grid, tree, 1e-10, opts, P.PLAIN, world, emulate=True).apply(f)
        # same per-box arithmetic; the sketch seeds are per level, so skeletons agree
        assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)


def test_emulated_shards_compressed_path():
    """Finite k_cut (a-priori skeletons) through the sharded phases: same
    arithmetic per box as the single-GPU compressed path, and the reference's
    compressed solution (tests/golden/compressed.npz)."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.distributed import ShardedInverse
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    gold = np.load(os.path.join(G, "compressed.npz"))
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(64)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=64)
    f = gold["solve_nonsym64_leaf64_f"]
    xr = compress_inverse(spec, grid, eps=1e-10, opts=opts).apply(f)
    for world in (2, 4):
        tree = P.build_tree(grid, 64)
        x = ShardedInverse(spec, grid, tree, 1e-10, opts, P.PLAIN, world, emulate=True).apply(f)
        assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)
        xg = gold["solve_nonsym64_leaf64_x"]
        assert np.linalg.norm(x - xg) / np.linalg.norm(xg) <= 1e-8


def test_emulated_shards_helmholtz_interior_retention():
    """Helmholtz above the oscillatory threshold (kappa = k / 2pi >= 16): the
    sharded path annotates the same a-priori skeletons as compress_inverse
    (interface-interior retention included, solver_compressed.py:536-542), so
    it reproduces the single-GPU compressed solve."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.distributed import ShardedInverse
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    k = 2 * np.pi * 17.0
    spec = P.KernelSpec("helmholtz2d", k=k, b_field=P.make_field("gaussian_bump"),
                        c_field=P.make_field("one"))
    grid = P.Grid(64)
    opts = P.SolverOptions(eps=1e-8, leaf_size=64, k_cut=64)
    assert opts.keep_interface_interior(spec)
    tree1 = P.build_tree(grid, 64)
    inv1 = compress_inverse(spec, grid, tree=tree1, eps=1e-8, opts=opts)
    f = np.exp(1j * k * (grid.points()[:, 0] + 1.0))
    xr = inv1.apply(f)
    tree2 = P.build_tree(grid, 64)
    x = ShardedInverse(spec, grid, tree2, 1e-8, opts, P.PLAIN, 2, emulate=True).apply(f)
    for a, b in zip(tree1.nodes, tree2.nodes):
        assert np.array_equal(a.sk_idx, b.sk_idx)
    assert np.linalg.norm(x - xr) <= 1e-11 * np.linalg.norm(xr)
