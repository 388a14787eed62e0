"""Batched 1-D HSS storage (paper_1303_5466_b200/hss1d.py) against the dense
matrices it compresses: the reference's hss1d contracts (`test_hss1d.py`:
densify / matvec agree with the entry oracle to the build tolerance; the
transposed apply; block-diagonal alignment) on kernel matrices over a closed
curve, which is what the compressed path stores (E and F^-1 over a box's
boundary ordering)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _curve_matrices(nb, n, seed, shift=0.0):
    """nb nonsymmetric n x n matrices: log kernel between points of a closed
    curve (1-D ordering), row / column weights, a dominant diagonal."""
    rng = np.random.default_rng(seed)
    out = []
    for b in range(nb):
        t = np.sort(rng.uniform(0, 2 * np.pi, n))
        a, c = 1.0 + 0.3 * rng.uniform(), 0.6 + 0.3 * rng.uniform()
        x = np.stack([a * np.cos(t) + shift, c * np.sin(t)], 1)
        d = np.linalg.norm(x[:, None, :] - x[None, :, :], axis=2)
        np.fill_diagonal(d, 1.0)
        K = np.log(d) / (2 * np.pi)
        w1 = 1.0 + 0.5 * np.sin(3 * t)
        w2 = 1.0 + 0.4 * np.cos(2 * t + 0.3)
        A = (w1[:, None] * K * w2[None, :]) * (2 * np.pi / n) + np.diag(1.0 + 0.1 * rng.uniform(size=n))
        out.append(A)
    return np.stack(out)


def _to_dev(A):
    # library layout: item b column-major, Ad[b, c, r] = A_b(r, c)
    return torch.from_numpy(np.ascontiguousarray(A.transpose(0, 2, 1))).cuda()


@pytest.mark.parametrize("nb,n,leaf,align", [(3, 700, 32, None), (2, 517, 32, 390), (1, 1200, 64, 800),
                                             (4, 40, 64, None), (2, 90, 32, 64)])
def test_compress_matvec_matches_dense(nb, n, leaf, align):
    from paper_1303_5466_b200.hss1d import Hss1dBatch
    A = _curve_matrices(nb, n, seed=n)
    H = Hss1dBatch.compress(_to_dev(A), n, 1e-10, leaf_size=leaf, align=align)
    rng = np.random.default_rng(1)
    for r in (1, 5):
        X = rng.standard_normal((nb, n, r))
        Xd = torch.from_numpy(np.ascontiguousarray(X.transpose(2, 0, 1).reshape(r, nb * n))).cuda()
        Y = H.matvec(Xd).cpu().numpy().reshape(r, nb, n).transpose(1, 2, 0)
        ref = A @ X
        assert np.linalg.norm(Y - ref) <= 1e-8 * np.linalg.norm(ref)
        Yt = H.matvec(Xd, trans=True).cpu().numpy().reshape(r, nb, n).transpose(1, 2, 0)
        reft = A.transpose(0, 2, 1) @ X
        assert np.linalg.norm(Yt - reft) <= 1e-8 * np.linalg.norm(reft)
    # accumulate form: Y = alpha A X + beta Y
    X = rng.standard_normal((nb, n, 3))
    Xd = torch.from_numpy(np.ascontiguousarray(X.transpose(2, 0, 1).reshape(3, nb * n))).cuda()
    Y0 = rng.standard_normal((3, nb * n))
    Yd = torch.from_numpy(Y0.copy()).cuda()
    H.matvec(Xd, Yd, alpha=-2.0, beta=1.0)
    ref = Y0.reshape(3, nb, n).transpose(1, 2, 0) - 2.0 * (A @ X)
    got = Yd.cpu().numpy().reshape(3, nb, n).transpose(1, 2, 0)
    assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)


def test_densify_and_memory():
    from paper_1303_5466_b200.hss1d import Hss1dBatch
    nb, n = 2, 1500
    A = _curve_matrices(nb, n, seed=7)
    H = Hss1dBatch.compress(_to_dev(A), n, 1e-10, leaf_size=32)
    Ad = H.to_dense().cpu().numpy().transpose(0, 2, 1)
    assert np.abs(Ad - A).max() <= 1e-8 * np.abs(A).max()
    assert H.depth >= 5 and H.max_rank() <= 64
    assert H.nbytes() < 0.5 * A.nbytes            # O(n k) storage against n^2
    # a looser tolerance gives smaller ranks
    H2 = Hss1dBatch.compress(_to_dev(A), n, 1e-5, leaf_size=32)
    assert H2.max_rank() < H.max_rank() and H2.nbytes() < H.nbytes()


def test_block_diagonal_alignment_keeps_zero_blocks():
    """A block-diagonal matrix cut at `align` has rank-0 root siblings
    (hss1d/core.py:52-71 align: cross blocks stay exactly zero)."""
    from paper_1303_5466_b200.hss1d import Hss1dBatch
    n, cut = 300, 180
    A = _curve_matrices(1, n, seed=3)
    A[0, :cut, cut:] = 0.0
    A[0, cut:, :cut] = 0.0
    H = Hss1dBatch.compress(_to_dev(A), n, 1e-10, leaf_size=32, align=cut)
    assert int(H.lv[1].k.max()) == 0
    X = np.random.default_rng(0).standard_normal((n, 2))
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    Y = H.matvec(Xd).cpu().numpy().T
    assert np.linalg.norm(Y - A[0] @ X) <= 1e-9 * np.linalg.norm(A[0] @ X)


# -- the compressed path with 1-D HSS block storage ---------------------------

def _problem(n, leaf, b="gaussian_bump", c="one", **kw):
    import paper_1303_5466_b200 as P
    spec = P.KernelSpec("laplace2d", b_field=P.make_field(b), c_field=P.make_field(c))
    grid = P.Grid(n)
    opts = P.SolverOptions(eps=1e-10, leaf_size=leaf, k_cut=64, **kw)
    return P, spec, grid, opts


@pytest.mark.parametrize("n,leaf,force", [(128, 64, True), (192, 64, True), (128, 64, False)])
def test_hss1d_storage_matches_dense_storage(n, leaf, force):
    """The reference's storage for boxes above k_cut (solver_compressed.py:
    490-511): F^-1 and E in 1-D HSS form (forced here: at these sizes the forms
    are larger than the blocks) or as lean dense blocks, the sweeps applying
    T_up / T_dn -- solves like the dense storage of the same factors for one
    and for several right-hand sides; the residual meets the reference's bar
    (test_solver_compressed.py:187-266: <= 1e-8)."""
    from paper_1303_5466_b200 import compressed_store
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    from paper_1303_5466_b200.verify import FFTOperator
    P, spec, grid, opts = _problem(n, leaf)
    dense = compress_inverse(spec, grid, eps=1e-10, opts=opts)
    if force:
        hss = compress_inverse(spec, grid, eps=1e-10, opts=opts)
        assert compressed_store.compact(hss.factors, force_hss=True) >= 4
    else:   # the option: every level above k_cut goes lean at this size
        hss = compress_inverse(spec, grid, eps=1e-10, opts=opts.with_(block_storage="hss1d"))
        H = hss.dense_matvec_source
        assert hss.hss_levels == 0
        assert sum(getattr(L, "hss_kind", None) == "lean" for L in H.levels) >= 5
        assert hss.nbytes() < 0.7 * dense.nbytes()
    rng = np.random.default_rng(3)
    f1 = rng.standard_normal(grid.n)
    F = rng.standard_normal((grid.n, 6))
    for f in (f1, F):
        xd, xh = dense.apply(f), hss.apply(f)
        assert xh.shape == f.shape
        assert np.linalg.norm(xh - xd) <= 1e-8 * np.linalg.norm(xd)
    op = FFTOperator(spec, grid, P.PLAIN, "cuda")
    X = torch.from_numpy(hss.apply(F)).cuda()
    R = torch.from_numpy(F).cuda() - op.matvec(X)
    assert float(R.norm() / np.linalg.norm(F)) <= 1e-8
    # deterministic: same object, same input, same bits (test_solver_dense.py:108-112)
    np.testing.assert_array_equal(hss.apply(f1), hss.apply(f1))


def test_hss1d_storage_matches_reference_compressed_solution():
    """Against the reference's own compressed solve (which stores these blocks
    in 1-D HSS form too): tests/golden/compressed.npz."""
    import os
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "compressed.npz"))
    P, spec, grid, opts = _problem(64, 64)
    # k_cut below the top boxes' skeleton sizes so that levels convert at this size
    # (at this size the forms are larger than the dense blocks: tried for every size)
    from paper_1303_5466_b200 import compressed_store
    inv = compress_inverse(spec, grid, eps=1e-10, opts=opts.with_(k_cut=32))
    assert compressed_store.compact(inv.factors, force_hss=True) >= 2
    f = gold["solve_nonsym64_leaf64_f"]
    xr = gold["solve_nonsym64_leaf64_x"]
    x = inv.apply(f)
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-8


def test_hss1d_factor_views_densify():
    """factor_of(box) on a converted level returns the blocks densified from
    the HSS forms: equal to the dense storage's blocks to the tolerance."""
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    P, spec, grid, opts = _problem(64, 64)
    dense = compress_inverse(spec, grid, eps=1e-10, opts=opts.with_(k_cut=32))
    from paper_1303_5466_b200 import compressed_store
    hss = compress_inverse(spec, grid, eps=1e-10, opts=opts.with_(k_cut=32))
    assert compressed_store.compact(hss.factors, force_hss=True) >= 2
    box = dense.tree.nodes[1]
    fd, fh = dense.factor_of(box), hss.factor_of(hss.tree.nodes[1])
    assert np.abs(fd.E - fh.E).max() <= 1e-8 * np.abs(fd.E).max()
    assert np.abs(fd.Finv - fh.Finv).max() <= 1e-8 * np.abs(fd.Finv).max()


def test_sequential_inversion_compacts_level_by_level():
    """invert_dense_block(storage="hss1d") converts a level as soon as its
    parent is factored (the low-memory schedule); same solution."""
    import paper_1303_5466_b200.solver_dense as sd
    from paper_1303_5466_b200.solver_compressed import ensure_apriori_skeletons
    from paper_1303_5466_b200.tree import build_tree
    P, spec, grid, opts = _problem(128, 64)
    f = np.random.default_rng(8).standard_normal(grid.n)
    sols = []
    for storage, on_demand in (("dense", False), ("hss1d", False), ("hss1d", True)):
        tree = build_tree(grid, 64)
        layers = ensure_apriori_skeletons(spec, tree, opts)
        H = sd.Hss2dMatrix(spec, grid, tree, 1e-10, opts, P.PLAIN)
        H.apriori = layers
        if on_demand:   # each level compressed just before its inversion, sources freed after
            inv = sd.invert_dense_block(H, storage=storage, compress=True, free_source=True)
            assert all(getattr(L, "D", None) is None and getattr(L, "B12", None) is None
                       for L in H.levels if L is not None and not getattr(L, "refine", False))
        else:
            sd.compress_levels(H)
            inv = sd.invert_dense_block(H, storage=storage)
        if storage == "hss1d":
            assert sum(getattr(L, "hss", None) is not None for L in H.levels) >= 1
        sols.append(inv.apply(f))
    assert np.linalg.norm(sols[1] - sols[0]) <= 1e-8 * np.linalg.norm(sols[0])
    assert np.array_equal(sols[2], sols[1])   # same arithmetic, a different schedule


def test_on_demand_compression_on_the_id_path():
    """invert_dense_block(compress=True) on the pivoted-ID path (k_cut = None):
    bitwise the solution of compress_outer + invert_dense_block."""
    import paper_1303_5466_b200 as P
    import paper_1303_5466_b200.solver_dense as sd
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(128)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    tree = P.build_tree(grid, 64)
    f = np.random.default_rng(3).standard_normal(grid.n)
    x0 = sd.invert_dense_block(sd.compress_outer(spec, grid, tree, 1e-10, opts)).apply(f)
    H = sd.Hss2dMatrix(spec, grid, tree, 1e-10, opts, P.PLAIN)
    x1 = sd.invert_dense_block(H, compress=True, free_source=True, storage="lean").apply(f)
    assert np.linalg.norm(x1 - x0) <= 1e-11 * np.linalg.norm(x0)


def test_hss1d_storage_at_512():
    """Where the forms pay off (m >= 1000): the top levels of a 512^2 grid
    go to HSS form, the others lean: the factor bytes nearly halve, same solution."""
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    P, spec, grid, opts = _problem(512, 64)
    f = np.random.default_rng(4).standard_normal((grid.n, 3))
    dense = compress_inverse(spec, grid, eps=1e-10, opts=opts)
    xd = dense.apply(f)
    nd = dense.nbytes()
    del dense
    torch.cuda.empty_cache()
    hss = compress_inverse(spec, grid, eps=1e-10, opts=opts.with_(block_storage="hss1d"))
    assert hss.hss_levels >= 3
    assert hss.nbytes() < 0.6 * nd
    xh = hss.apply(f)
    assert np.linalg.norm(xh - xd) <= 1e-8 * np.linalg.norm(xd)


@pytest.mark.parametrize("n,leaf,b,c", [(64, 64, "gaussian_bump", "one"), (128, 64, "gaussian_bump", "gaussian_bump"),
                                        (30, 64, "gaussian_bump", "one")])
def test_lean_storage_on_the_id_path(n, leaf, b, c):
    """invert_dense_block(storage="lean") on the pivoted-ID path (k_cut = None:
    row / column skeletons in pivot order, ranks varying from box to box): the
    reference's own factor set (F, E, T: solver_dense.py:284-291) -- same
    solution as the dense storage, the reference layout's byte count."""
    import paper_1303_5466_b200 as P
    import paper_1303_5466_b200.solver_dense as sd
    spec = P.KernelSpec("laplace2d", b_field=P.make_field(b), c_field=P.make_field(c))
    grid = P.Grid(n)
    opts = P.SolverOptions(eps=1e-10, leaf_size=leaf, k_cut=None)
    rng = np.random.default_rng(6)
    F = rng.standard_normal((grid.n, 4))
    f1 = rng.standard_normal(grid.n)
    tree = P.build_tree(grid, leaf)
    dense = sd.invert_dense_block(sd.compress_outer(spec, grid, tree, 1e-10, opts))
    H = sd.compress_outer(spec, grid, tree, 1e-10, opts)
    lean = sd.invert_dense_block(H, storage="lean")
    kinds = [getattr(L, "hss_kind", None) for L in H.levels if L is not None and L.lv > 0]
    assert all(kd == "lean" for kd in kinds), kinds
    # (as allocated: boxes are padded to the largest of their level)
    assert abs(lean.nbytes() - dense.nbytes_reference_layout()) <= 0.08 * lean.nbytes()
    assert lean.nbytes() <= dense.nbytes()
    for f in (f1, F):
        xd, xl = dense.apply(f), lean.apply(f)
        assert np.linalg.norm(xl - xd) <= 1e-11 * np.linalg.norm(xd)
    v = rng.standard_normal(grid.n)
    assert np.linalg.norm(v - H.matvec(lean.apply(v))) <= 1e-9 * np.linalg.norm(v)
    i = int(H.tree.nodes[1].idx)
    assert np.abs(lean.E[i] - dense.E[i]).max() <= 1e-12 * np.abs(dense.E[i]).max()
    assert np.abs(lean.Finv[i] - dense.Finv[i]).max() <= 1e-12 * np.abs(dense.Finv[i]).max()


@pytest.mark.parametrize("mode", ["hss", "lean"])
def test_helmholtz_compressed_with_block_storage(mode):
    """Complex kernel (realified on the device): the converted storage solves
    like the dense one and meets the reference's residual bar
    (test_solver_compressed.py:243-253: <= 1e-7); the skeleton stays a set of
    grid points ((Re, Im) pairs stay adjacent in the [sk, rs] ordering)."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200 import compressed_store
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    spec = P.KernelSpec("helmholtz2d", k=4 * np.pi)
    grid = P.Grid(36)
    opts = P.SolverOptions(eps=1e-10, leaf_size=81, k_cut=16)
    dense = compress_inverse(spec, grid, eps=1e-10, opts=opts)
    conv = compress_inverse(spec, grid, eps=1e-10, opts=opts)
    if mode == "hss":
        assert compressed_store.compact(conv.factors, force_hss=True) >= 2
    else:
        compressed_store.compact(conv.factors, min_size=float("inf"))
        kinds = [getattr(L, "hss_kind", None) for L in conv.dense_matvec_source.levels if L is not None]
        assert kinds.count("lean") >= 2
    rng = np.random.default_rng(12)
    f = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    xd, xc = dense.apply(f), conv.apply(f)
    assert xc.dtype == np.complex128
    assert np.linalg.norm(xc - xd) <= 1e-8 * np.linalg.norm(xd)
    A = P.assemble_dense(spec, grid, P.PLAIN, np.arange(grid.n), np.arange(grid.n))
    assert np.linalg.norm(A @ xc - f) / np.linalg.norm(f) <= 1e-7


@pytest.mark.parametrize("k_cut,storage", [(None, "dense"), (64, "dense"), (64, "hss1d")])
def test_low_memory_option_same_solution(k_cut, storage):
    """SolverOptions(low_memory=True) (level-by-level compression + inversion,
    sources dropped, lean / 1-D HSS factors) through the public
    compress_inverse: the default schedule's solution and a true residual
    (FFT operator: H's blocks are gone) at the tolerance."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    from paper_1303_5466_b200.verify import FFTOperator
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(128)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=k_cut, block_storage=storage)
    f = np.random.default_rng(12).standard_normal((grid.n, 2))
    x0 = compress_inverse(spec, grid, eps=1e-10, opts=opts).apply(f)
    low = compress_inverse(spec, grid, eps=1e-10, opts=opts.with_(low_memory=True))
    x1 = low.apply(f)
    assert np.linalg.norm(x1 - x0) <= 1e-8 * np.linalg.norm(x0)
    assert low.nbytes() > 0
    op = FFTOperator(spec, grid, P.PLAIN, "cuda")
    X = torch.as_tensor(x1, device="cuda")
    F = torch.as_tensor(f, device="cuda")
    res = float(((F - op.matvec(X)).norm(dim=0) / F.norm(dim=0)).max())
    assert res <= (1e-9 if k_cut is None else 1e-6), res
