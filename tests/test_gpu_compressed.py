"""Compressed (finite k_cut) path on the B200: a-priori skeletons, proxy
least-squares interpolation (fixed-rank batched QR, vief_id_batched kfix) and
dense per-box factors.  Checked against the CPU oracle's a-priori solve on the
same inputs (same arithmetic, dense blocks: <= 1e-9 relative), against the
reference's compressed solutions (tests/golden/compressed.npz; the reference
keeps large blocks in eps-accurate 1-D HSS form: <= 1e-8 relative), and by the
reference's residual bar (test_solver_compressed.py:187-266: <= 1e-8)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")
CASES = {  # name: (n, leaf, k_cut, b field, c field, ti_mode)
    "nti28_k8": (28, 49, 8, "gaussian_bump", "gaussian_bump", False),
    "nti28_k64": (28, 49, 64, "gaussian_bump", "gaussian_bump", False),
    "nonsym28_k8": (28, 49, 8, "gaussian_bump", "one", False),
    "ti28_k8": (28, 49, 8, "one", "one", True),
    "nti56_k64": (56, 49, 64, "gaussian_bump", "gaussian_bump", False),
    "nonsym64_leaf64": (64, 64, 64, "gaussian_bump", "one", False),
}


def _solve(name, f=None):
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    n, leaf, k_cut, b, c, ti = CASES[name]
    spec = P.KernelSpec("laplace2d", b_field=P.make_field(b), c_field=P.make_field(c))
    grid = P.Grid(n)
    opts = P.SolverOptions(eps=1e-10, leaf_size=leaf, k_cut=k_cut)
    inv = compress_inverse(spec, grid, eps=1e-10, opts=opts, ti_mode=ti)
    return spec, grid, inv


@pytest.mark.parametrize("name", list(CASES))
def test_compressed_matches_reference_and_oracle(name):
    import oracle.hssd as O
    import paper_1303_5466_b200 as P
    gold = np.load(os.path.join(G, "compressed.npz"))
    spec, grid, inv = _solve(name)
    f = gold[f"solve_{name}_f"]
    x = inv.apply(f)
    assert x.shape == f.shape and x.dtype == np.float64
    xr = gold[f"solve_{name}_x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-8
    n, leaf, _, b, c, _ = CASES[name]
    Pr = O.Problem(n, "laplace2d", 0.0, ("one", ()), (b, ()), (c, ()), "none")
    xo, _, _ = O.solve_apriori(Pr, leaf, 2, f)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-9
    A = P.assemble_dense(spec, grid, P.PLAIN, np.arange(grid.n), np.arange(grid.n))
    assert np.linalg.norm(A @ x - f) / np.linalg.norm(f) <= 1e-8


def test_skeletons_are_the_apriori_bands():
    _, _, inv = _solve("nonsym28_k8")
    H = inv.dense_matvec_source
    for node in inv.tree.nodes[1:]:
        np.testing.assert_array_equal(H.row_skel[node.idx], node.sk_idx)
        np.testing.assert_array_equal(H.col_skel[node.idx], node.sk_idx)


def test_interp_least_squares_residual():
    """T_up / T_dn fit the proxy systems: box 1 to 1e-9
    (test_solver_compressed.py:29-44), every checked box as well as LAPACK's
    least-squares solution does (the fit error itself is ~1e-9 at level 2)."""
    import oracle.hssd as O
    import scipy.linalg as sla
    _, _, inv = _solve("nonsym28_k8")
    H = inv.dense_matvec_source
    Pr = O.Problem(28, "laplace2d", 0.0, ("one", ()), ("gaussian_bump", ()), ("one", ()),
                   "none")
    tree = inv.tree
    for bid in (1, 3, 7, 20):
        node = tree.nodes[bid]
        zp = O.proxy_ring(np.array([node.x0, node.x1, node.y0, node.y1]), 2)
        for f, sys_of in ((H.Rfac[bid], lambda I: O.proxy_tgt(Pr, zp, I)),
                          (H.Lfac[bid], lambda I: O.proxy_src(Pr, I, zp).T)):
            sk = node.full_idx[f.perm[:f.k]]
            rs = node.full_idx[f.perm[f.k:]]
            kzs, kzr = sys_of(sk), sys_of(rs)
            resid = np.linalg.norm(kzs @ f.T - kzr) / np.linalg.norm(kzr)
            best = np.linalg.norm(kzs @ sla.lstsq(kzs, kzr)[0] - kzr) / np.linalg.norm(kzr)
            assert resid <= 1.01 * best + 1e-13, (bid, resid, best)
            if bid == 1:
                assert resid <= 1e-9


def test_multiple_rhs_batch_matches_sequential():
    _, grid, inv = _solve("nti28_k64")
    F = np.random.default_rng(6).standard_normal((grid.n, 3))
    batch = inv.apply(F)
    np.testing.assert_array_equal(batch, inv.apply(F))
    for j in range(3):
        col = inv.apply(F[:, j])
        assert np.linalg.norm(batch[:, j] - col) <= 1e-13 * np.linalg.norm(col)


def test_compressed_c1_size_residual():
    """128^2, leaf 64, the c1 problem family on the compressed path: true
    residual through the exact FFT operator."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    from paper_1303_5466_b200.verify import true_residual
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"),
                        c_field=P.make_field("one"))
    grid = P.Grid(128)
    inv = compress_inverse(spec, grid, eps=1e-10,
                           opts=P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=64))
    f = np.random.default_rng(0).standard_normal(grid.n)
    x = inv.apply(f)
    assert true_residual(spec, grid, P.PLAIN, f, x) <= 1e-8


def test_helmholtz_compressed_matches_reference():
    """Complex kernel, realified on the device (test_solver_compressed.py:243-253:
    residual <= 1e-7), solution vs the reference's compressed one."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    gold = np.load(os.path.join(G, "compressed.npz"))
    spec = P.KernelSpec("helmholtz2d", k=4 * np.pi)
    grid = P.Grid(18)
    inv = compress_inverse(spec, grid, eps=1e-10,
                           opts=P.SolverOptions(eps=1e-10, leaf_size=81, k_cut=16))
    f = gold["solve_helm18_f"]
    x = inv.apply(f)
    assert x.dtype == np.complex128
    A = P.assemble_dense(spec, grid, P.PLAIN, np.arange(grid.n), np.arange(grid.n))
    assert np.linalg.norm(A @ x - f) / np.linalg.norm(f) <= 1e-7
    xr = gold["solve_helm18_x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-7


def _oracle_apriori(name):
    import oracle.hssd as O
    n, leaf, _, b, c, _ = CASES[name]
    Pr = O.Problem(n, "laplace2d", 0.0, ("one", ()), (b, ()), (c, ()), "none")
    tree = O.make_tree(n, leaf)
    H, ann = O.compress_apriori(Pr, tree, 2)
    return O, tree, H, ann, O.invert(H)


def test_build_e_matches_dense_oracle():
    """E = ([I T_up] F^-1 [I; T_dn^T])^-1 per box vs the dense oracle
    (test_solver_compressed.py:168-184: <= 1e-7; here <= 1e-8)."""
    _, _, inv = _solve("nonsym28_k8")
    O, tree, H, ann, oinv = _oracle_apriori("nonsym28_k8")
    for bid in (1, 3, 7, 20):
        fac = inv.factor_of(inv.tree.nodes[bid])
        assert fac.kind == ("leaf" if inv.tree.nodes[bid].is_leaf else "dense")
        assert fac.E.shape == (fac.k, fac.k)
        E = oinv.E[bid]
        # T comes from an ill-conditioned least-squares fit (LAPACK gelsd in the
        # oracle, Householder QR here): E agrees to ~1e-9, 100x inside the bar
        assert np.linalg.norm(fac.E - E) / np.linalg.norm(E) <= 1e-8
        assert fac.T_up.shape == fac.T_dn.shape == (fac.k, fac.r)


def test_apply_finv_matches_dense_oracle():
    """F^-1 on [sk, rs] vs the dense oracle F (test_solver_compressed.py:129-153),
    linearity, record count."""
    _, _, inv = _solve("nti28_k8")
    O, tree, H, ann, oinv = _oracle_apriori("nti28_k8")
    bid = 3
    fac = inv.factor_of(inv.tree.nodes[bid])
    c1, c2 = tree.kids[bid]
    F = np.block([[oinv.E[c1], H.B[bid][0]], [H.B[bid][1], oinv.E[c2]]])
    perm = ann[bid][2]
    Fd = F[np.ix_(perm, perm)]
    rng = np.random.default_rng(0)
    u = rng.standard_normal((Fd.shape[0], 3))
    got, ref = fac.apply_finv(u), np.linalg.solve(Fd, u)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-9
    u2 = rng.standard_normal(Fd.shape[0])
    lhs = fac.apply_finv((2.0 * u[:, 0] + u2)[:, None])
    rhs = 2.0 * fac.apply_finv(u[:, 0][:, None]) + fac.apply_finv(u2[:, None])
    assert np.linalg.norm(lhs - rhs) <= 1e-11 * np.linalg.norm(rhs)
    assert inv.record_count() == len(inv.tree.nodes)
    with pytest.raises(KeyError):
        inv.factor_of(inv.tree.nodes[0])


def test_ti_record_sharing_and_accuracy():
    """TI mode keeps one record per level (test_solver_compressed.py:216-234):
    same solution as per-box factors, factor memory one record per level."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    spec = P.KernelSpec("laplace2d")
    grid = P.Grid(28)
    opts = P.SolverOptions(eps=1e-10, k_cut=8)
    inv_ti = compress_inverse(spec, grid, eps=1e-10, opts=opts, ti_mode=True)
    inv_nti = compress_inverse(spec, grid, eps=1e-10, opts=opts, ti_mode=False)
    assert inv_ti.record_count() == inv_ti.tree.depth + 1
    assert inv_ti.nbytes() < inv_nti.nbytes() / 2   # reference: 2.6 MB vs 6.3 MB
    # the factorization itself ran on the first box of every level only (28^2
    # with leaf 64 is uniform): one record per level, no per-box F^-1 computed
    Hti = inv_ti.dense_matvec_source
    assert Hti.ti_share
    assert all(L.Finv.shape[0] == 1 for L in Hti.levels if L.lv > 0)
    A = P.assemble_dense(spec, grid, P.PLAIN, np.arange(grid.n), np.arange(grid.n))
    v = np.random.default_rng(3).standard_normal((grid.n, 2))
    x_ti, x_nti = inv_ti.apply(v), inv_nti.apply(v)
    assert np.linalg.norm(x_ti - x_nti) <= 1e-12 * np.linalg.norm(x_nti)
    r = np.linalg.norm(A @ x_ti - v) / np.linalg.norm(v)
    assert r <= 1e-8
    x1 = inv_ti.apply(v[:, 0])   # single RHS: the GEMV path with stride-0 factors
    assert np.linalg.norm(x1 - x_ti[:, 0]) <= 1e-13 * np.linalg.norm(x1)
    gold = np.load(os.path.join(G, "compressed.npz"))
    f = gold["solve_ti28_k8_f"]
    xg = gold["solve_ti28_k8_x"]
    assert np.linalg.norm(inv_ti.apply(f) - xg) / np.linalg.norm(xg) <= 1e-8


def test_ti_mode_512_memory():
    """512^2 TI problem: shared records make the factors small; true residual."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    from paper_1303_5466_b200.verify import true_residual
    spec = P.KernelSpec("laplace2d")
    grid = P.Grid(512)
    inv = compress_inverse(spec, grid, eps=1e-10,
                           opts=P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=64), ti_mode=True)
    assert inv.nbytes() < 2e9
    f = np.random.default_rng(0).standard_normal(grid.n)
    assert true_residual(spec, grid, P.PLAIN, f, inv.apply(f)) <= 1e-8


def test_ti_mode_ragged_grid_keeps_per_box_records():
    """Ragged boxes (Grid(30), leaf 64: 49/56/64-point leaves) are not
    translates of each other; TI mode must keep their per-box records instead
    of reading box 0's factors for every box."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    from paper_1303_5466_b200.solver_dense import _level_is_uniform
    spec = P.KernelSpec("laplace2d")
    grid = P.Grid(30)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=8)
    inv_ti = compress_inverse(spec, grid, eps=1e-10, opts=opts, ti_mode=True)
    inv_nti = compress_inverse(spec, grid, eps=1e-10, opts=opts, ti_mode=False)
    levels = [L for L in inv_ti.dense_matvec_source.levels if L is not None]
    assert any(not _level_is_uniform(L) for L in levels)
    for L in levels:
        assert getattr(L, "ti", False) == (L.nb >= 2 and _level_is_uniform(L))
    v = np.random.default_rng(4).standard_normal((grid.n, 2))
    x_ti, x_nti = inv_ti.apply(v), inv_nti.apply(v)
    assert np.linalg.norm(x_ti - x_nti) <= 1e-12 * np.linalg.norm(x_nti)
    A = P.assemble_dense(spec, grid, P.PLAIN, np.arange(grid.n), np.arange(grid.n))
    assert np.linalg.norm(A @ x_ti - v) / np.linalg.norm(v) <= 1e-8
