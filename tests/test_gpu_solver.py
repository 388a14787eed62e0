"""End-to-end HSS-D parity on the B200: the reference's own solver tests
(test_solver_dense.py) ported to this API, plus solutions compared with the
reference's (golden vectors from tests/golden/make_golden.py) on identical
seeded inputs.  Tolerances: relative error vs the reference <= 10*eps,
residuals <= 10*eps (BASELINE.json north star)."""
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def _api():
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200 import solver_dense as sd
    return P, sd


def laplace_nti():
    P, _ = _api()
    return P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"),
                        c_field=P.make_field("gaussian_bump"))


def setup(n_side, spec=None, eps=1e-10, leaf=49, quad=None):
    P, sd = _api()
    spec = spec or laplace_nti()
    grid = P.Grid(n_side)
    tree = P.build_tree(grid, leaf)
    opts = P.SolverOptions(eps=eps, leaf_size=leaf)
    H = sd.compress_outer(spec, grid, tree, eps, opts, quad or P.PLAIN)
    return spec, grid, tree, H


def dense_matrix(spec, grid, quad=None):
    P, _ = _api()
    return P.assemble_dense(spec, grid, quad or P.PLAIN, np.arange(grid.n), np.arange(grid.n))


# ---- ported from the reference's tests/test_solver_dense.py ----------------

def test_densify_small():
    spec, grid, tree, H = setup(14)
    A = dense_matrix(spec, grid)
    assert np.linalg.norm(H.densify() - A) / np.linalg.norm(A) <= 1e-9


def test_densify_784():
    spec, grid, tree, H = setup(28)
    A = dense_matrix(spec, grid)
    assert np.linalg.norm(H.densify() - A) / np.linalg.norm(A) <= 1e-9


def test_symmetric_shares_interp():
    spec, grid, tree, H = setup(28)
    for i in H.Lfac:
        assert H.Rfac[i] is H.Lfac[i]
    np.testing.assert_array_equal(H.row_skel[1], H.col_skel[1])


def test_matvec_against_dense():
    _, sd = _api()
    spec, grid, tree, H = setup(28)
    A = dense_matrix(spec, grid)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(grid.n)
    y = sd.hss_matvec(H, x)
    assert np.linalg.norm(y - A @ x) / np.linalg.norm(A @ x) <= 1e-9
    assert np.all(sd.hss_matvec(H, np.zeros(grid.n)) == 0)
    z = rng.standard_normal(grid.n)
    lhs = sd.hss_matvec(H, 2.0 * x - 3.0 * z)
    rhs = 2.0 * sd.hss_matvec(H, x) - 3.0 * sd.hss_matvec(H, z)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_skeleton_sizes_bounded():
    spec, grid, tree, H = setup(28)
    for box in tree.nodes:
        if box.idx:
            assert H.row_skel[box.idx].size <= H.work_rows(box).size


def test_single_leaf_tree_inverse():
    P, sd = _api()
    spec = laplace_nti()
    grid = P.Grid(7)
    tree = P.build_tree(grid, 49)
    H = sd.compress_outer(spec, grid, tree, 1e-10, P.SolverOptions())
    inv = sd.invert_dense_block(H)
    A = dense_matrix(spec, grid)
    f = np.random.default_rng(1).standard_normal(grid.n)
    x = sd.apply_inverse_dense_block(inv, f)
    assert np.linalg.norm(A @ x - f) / np.linalg.norm(f) <= 1e-12


def test_inverse_residual_784():
    _, sd = _api()
    spec, grid, tree, H = setup(28)
    inv = sd.invert_dense_block(H)
    rng = np.random.default_rng(2)
    worst = 0.0
    for _ in range(10):
        v = rng.standard_normal(grid.n)
        worst = max(worst, np.linalg.norm(v - H.matvec(inv.apply(v))) / np.linalg.norm(v))
    assert worst <= 1e-9


def test_inverse_against_dense_lu():
    _, sd = _api()
    spec, grid, tree, H = setup(28)
    inv = sd.invert_dense_block(H)
    A = dense_matrix(spec, grid)
    v = np.random.default_rng(3).standard_normal(grid.n)
    xd = np.linalg.solve(A, v)
    assert np.linalg.norm(inv.apply(v) - xd) / np.linalg.norm(xd) <= 1e-8


def test_apply_deterministic_bitwise():
    _, sd = _api()
    spec, grid, tree, H = setup(28)
    inv = sd.invert_dense_block(H)
    v = np.random.default_rng(4).standard_normal(grid.n)
    np.testing.assert_array_equal(inv.apply(v), inv.apply(v))


def test_nonsymmetric_kernel_roundtrip():
    P, sd = _api()
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(14)
    tree = P.build_tree(grid, 49)
    H = sd.compress_outer(spec, grid, tree, 1e-10, P.SolverOptions())
    A = dense_matrix(spec, grid)
    assert np.linalg.norm(H.densify() - A) / np.linalg.norm(A) <= 1e-9
    inv = sd.invert_dense_block(H)
    v = np.random.default_rng(5).standard_normal(grid.n)
    assert np.linalg.norm(A @ inv.apply(v) - v) / np.linalg.norm(v) <= 1e-8


def test_inverse_residual_3136():
    _, sd = _api()
    spec, grid, tree, H = setup(56)
    inv = sd.invert_dense_block(H)
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(10):
        v = rng.standard_normal(grid.n)
        worst = max(worst, np.linalg.norm(v - H.matvec(inv.apply(v))) / np.linalg.norm(v))
    assert worst <= 1e-9


def test_skeleton_scaling_slope():
    spec, grid, tree, H = setup(112, eps=1e-10)
    sizes = {}
    for box in tree.nodes:
        if box.idx == 0 or box.is_leaf:
            continue
        sizes.setdefault(box.level, []).append(H.row_skel[box.idx].size)
    levels = sorted(sizes)[:5]
    npts = [grid.n / 2 ** lv for lv in levels]
    kmax = [max(sizes[lv]) for lv in levels]
    slope = np.polyfit(np.log(npts), np.log(kmax), 1)[0]
    assert 0.4 <= slope <= 0.6, (dict(zip(levels, kmax)), slope)


def test_kcut_none_delegates_bitwise():
    P, sd = _api()
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    spec = laplace_nti()
    grid = P.Grid(28)
    tree = P.build_tree(grid, 49)
    opts = P.SolverOptions(eps=1e-10, k_cut=None)
    inv = compress_inverse(spec, grid, tree=tree, eps=1e-10, opts=opts)
    ref = sd.invert_dense_block(sd.compress_outer(spec, grid, tree, 1e-10, opts))
    v = np.random.default_rng(2).standard_normal(grid.n)
    np.testing.assert_array_equal(inv.apply(v), ref.apply(v))


@pytest.mark.parametrize("n_side,nrhs", [(28, 1), (64, 7)])
def test_factor_solve_matches_factorize_apply_bitwise(n_side, nrhs):
    """The pipelined factor_solve (up sweep overlapping the factorization) is
    the same computation as compress_outer + invert_dense_block + apply."""
    P, sd = _api()
    spec = laplace_nti()
    grid = P.Grid(n_side)
    tree = P.build_tree(grid, 49 if n_side == 28 else 64)
    opts = P.SolverOptions(eps=1e-10, k_cut=None)
    rng = np.random.default_rng(5)
    f = rng.standard_normal(grid.n) if nrhs == 1 else rng.standard_normal((grid.n, nrhs))
    H, inv, x = sd.factor_solve(spec, grid, tree, 1e-10, opts, f)
    ref = sd.invert_dense_block(sd.compress_outer(spec, grid, tree, 1e-10, opts))
    np.testing.assert_array_equal(x, ref.apply(f))
    np.testing.assert_array_equal(inv.apply(f), x)


def test_batch_vs_sequential_rhs():
    _, sd = _api()
    spec, grid, tree, H = setup(28)
    inv = sd.invert_dense_block(H)
    F = np.random.default_rng(9).standard_normal((grid.n, 5))
    Xb = inv.apply(F)
    Xs = np.column_stack([inv.apply(F[:, j]) for j in range(5)])
    assert np.linalg.norm(Xb - Xs) <= 1e-13 * np.linalg.norm(Xs)


def test_singular_factor_raises():
    P, sd = _api()
    from paper_1303_5466_b200.dense_core import dense_solve
    A = np.zeros((3, 3))
    A[0, 0] = 1.0
    with pytest.raises(P.SingularFactorError):
        dense_solve(A, np.eye(3))


def test_factor_singular_box_reports_where():
    # a = 0 and b = c = 0: the system matrix is identically zero -> leaf F singular
    P, sd = _api()
    spec = P.KernelSpec("laplace2d", a_field=P.make_field("tanh_box", d=1.0, eps_edge=5.0, scale=0.0),
                        b_field=P.make_field("tanh_box", d=1.0, eps_edge=5.0, scale=0.0),
                        c_field=P.make_field("tanh_box", d=1.0, eps_edge=5.0, scale=0.0))
    grid = P.Grid(7)
    tree = P.build_tree(grid, 49)
    H = sd.compress_outer(spec, grid, tree, 1e-10, P.SolverOptions())
    with pytest.raises(P.SingularFactorError) as ei:
        sd.invert_dense_block(H)
    assert ei.value.where.startswith("box ")


def test_factor_singular_leaf_in_a_deep_tree_reports_the_leaf():
    """Every leaf F singular in a three-level tree: the exception names a leaf
    box (the finest level is tested first), on the sequential and the
    pipelined factorization alike."""
    P, sd = _api()
    zero = P.make_field("tanh_box", d=1.0, eps_edge=5.0, scale=0.0)
    spec = P.KernelSpec("laplace2d", a_field=zero, b_field=zero, c_field=zero)
    grid = P.Grid(16)
    tree = P.build_tree(grid, 64)
    leaf_level = max(b.level for b in tree.nodes)
    assert leaf_level >= 2
    H = sd.compress_outer(spec, grid, tree, 1e-10, P.SolverOptions(leaf_size=64))
    with pytest.raises(P.SingularFactorError) as ei:
        sd.invert_dense_block(H)
    assert ei.value.where.startswith("box ") and ei.value.where.endswith(f"level {leaf_level}")
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    with pytest.raises(P.SingularFactorError) as ei:
        compress_inverse(spec, grid, eps=1e-10, opts=P.SolverOptions(leaf_size=64, k_cut=None))
    assert ei.value.where.endswith(f"level {leaf_level}")


# ---- parity with the reference's solutions (golden vectors) ----------------

def _case_spec(name):
    P, _ = _api()
    rows = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    c1 = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                      c_field=P.make_field("one"))
    return {
        "nti28": (laplace_nti(), 28, 49, 1e-10, P.PLAIN),
        "rows14": (rows, 14, 49, 1e-10, P.PLAIN),
        "rows30": (rows, 30, 64, 1e-10, P.PLAIN),
        "single7": (laplace_nti(), 7, 49, 1e-10, P.PLAIN),
        "eps5_28": (rows, 28, 49, 1e-5, P.H4),
        "c1_64": (c1, 64, 64, 1e-10, P.CELL),
        "c1_128": (c1, 128, 64, 1e-10, P.CELL),
    }[name]


@pytest.mark.parametrize("case", ["nti28", "rows14", "rows30", "single7", "eps5_28", "c1_64", "c1_128"])
def test_solution_matches_reference(case):
    P, sd = _api()
    spec, n, leaf, eps, quad = _case_spec(case)
    g = np.load(os.path.join(G, f"solve_{case}.npz"))
    grid = P.Grid(n)
    tree = P.build_tree(grid, leaf)
    H = sd.compress_outer(spec, grid, tree, eps, P.SolverOptions(eps=eps, leaf_size=leaf), quad)
    inv = sd.invert_dense_block(H)
    f = g["f"]
    x = inv.apply(f)
    xr = g["x"]
    tol = 10 * eps
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= tol
    # approximate residual E through the compressed operator (scattering.py:154-163)
    assert np.linalg.norm(f - H.matvec(x)) / np.linalg.norm(f) <= tol
    if "x_dense" in g.files:
        assert np.linalg.norm(x - g["x_dense"]) / np.linalg.norm(g["x_dense"]) <= max(tol, 1e-8)
    # skeleton sizes: diagnostic parity with the reference's LAPACK ranks
    rk = g["rank"]
    for b in tree.nodes:
        if b.idx:
            assert abs(H.row_skel[b.idx].size - rk[b.idx]) <= 5
    # storage accounting in the reference's layout within a few percent
    assert abs(inv.nbytes_reference_layout() - int(g["nbytes_inv"])) <= 0.02 * int(g["nbytes_inv"])


def test_torch_device_rhs_roundtrip():
    P, sd = _api()
    spec, grid, tree, H = setup(28)
    inv = sd.invert_dense_block(H)
    F = torch.randn(grid.n, 3, dtype=torch.float64, device="cuda")
    X = inv.apply(F)
    assert X.is_cuda and X.shape == F.shape
    r = (F - H.matvec(X)).norm() / F.norm()
    assert float(r) <= 1e-9


# ---- complex (helmholtz2d), factored in realified form ---------------------

def test_helmholtz_small_inverse():
    """Port of the reference's test_solver_dense.py:131-144."""
    P, sd = _api()
    k = 2 * np.pi * 2
    spec = P.KernelSpec("helmholtz2d", k=k)
    grid = P.Grid(18)
    tree = P.build_tree(grid, 81)
    H = sd.compress_outer(spec, grid, tree, 1e-10, P.SolverOptions())
    A = dense_matrix(spec, grid)
    assert np.linalg.norm(H.densify() - A) / np.linalg.norm(A) <= 1e-8
    inv = sd.invert_dense_block(H)
    rng = np.random.default_rng(6)
    v = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    x = inv.apply(v)
    assert x.dtype == np.complex128
    assert np.linalg.norm(A @ x - v) / np.linalg.norm(v) <= 1e-8


def test_helmholtz_matches_reference_solution():
    P, sd = _api()
    g = np.load(os.path.join(G, "solve_helm18.npz"))
    spec = P.KernelSpec("helmholtz2d", k=2 * np.pi * 2)
    grid = P.Grid(18)
    tree = P.build_tree(grid, 81)
    H = sd.compress_outer(spec, grid, tree, 1e-10, P.SolverOptions(eps=1e-10, leaf_size=81))
    inv = sd.invert_dense_block(H)
    x = inv.apply(g["f"])
    assert np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]) <= 1e-9
    assert np.linalg.norm(g["f"] - H.matvec(x)) / np.linalg.norm(g["f"]) <= 1e-9


@pytest.mark.parametrize("n", [256, 512])
def test_solution_matches_reference_large(n):
    """Config c1 at 256^2 / 512^2 side by side with the reference (SURVEY.md
    §8(c) item 2; fixtures from tests/golden/make_golden_big.py, RHS
    regenerated from its seed): relative error vs the reference's solution
    <= 10 eps, true residual (exact FFT operator) <= 10 eps, reference-layout
    storage within 2 %, per-level maximum skeleton sizes within 2 %."""
    P, sd = _api()
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    from paper_1303_5466_b200.verify import FFTOperator, true_residual
    path = os.path.join(G, f"solve_c1_{n}.npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {path} not generated")
    g = np.load(path)
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                        c_field=P.make_field("one"))
    grid = P.Grid(n)
    eps = 1e-10
    inv = compress_inverse(spec, grid, eps=eps,
                           opts=P.SolverOptions(eps=eps, leaf_size=64, k_cut=None), quad=P.CELL)
    f = np.random.default_rng(int(g["seed"])).standard_normal(grid.n)
    x = inv.apply(f)
    xr = g["x"]
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 10 * eps
    r = true_residual(spec, grid, P.CELL, f, x, FFTOperator(spec, grid, P.CELL, "cuda"))
    assert r <= 10 * eps, r
    H = inv.dense_matvec_source
    ref_nb = int(g["nbytes_inv"])
    assert abs(inv.dense_delegate.nbytes_reference_layout() - ref_nb) <= 0.02 * ref_nb
    rk = g["rank"]
    for L in H.levels[1:]:
        kref = max(int(rk[i]) for i in L.ids)
        assert abs(int(L.kmax) - kref) <= 0.02 * kref + 2, (L.lv, int(L.kmax), kref)


# ---- exact residual at sizes the dense oracle cannot reach (FFT operator) --

@pytest.mark.parametrize("n,nrhs", [(256, 1), (256, 4), (512, 2)])
def test_true_residual_fft_config_family(n, nrhs):
    """BASELINE config family (BUMP rows, cell diagonal, leaf 64, eps 1e-10):
    ||f - A x|| / ||f|| <= 10 eps with A applied exactly by FFT."""
    P, sd = _api()
    from paper_1303_5466_b200.verify import FFTOperator, true_residual
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                        c_field=P.make_field("one"))
    grid = P.Grid(n)
    eps = 1e-10
    opts = P.SolverOptions(eps=eps, leaf_size=64, k_cut=None)
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    inv = compress_inverse(spec, grid, eps=eps, opts=opts, quad=P.CELL)
    f = np.random.default_rng(n + nrhs).standard_normal((grid.n, nrhs) if nrhs > 1 else grid.n)
    x = inv.apply(f)
    r = true_residual(spec, grid, P.CELL, f, x, FFTOperator(spec, grid, P.CELL, "cuda"))
    assert np.all(np.asarray(r) <= 10 * eps), r


def test_true_residual_fft_helmholtz():
    """Lippmann-Schwinger (complex128 through the realified path) at 64^2."""
    P, sd = _api()
    from paper_1303_5466_b200.verify import true_residual
    spec = P.KernelSpec("helmholtz2d", k=20.0, b_field=P.make_field("gaussian_bump"),
                        c_field=P.make_field("one"))
    grid = P.Grid(64)
    eps = 1e-8
    from paper_1303_5466_b200.solver_compressed import compress_inverse
    inv = compress_inverse(spec, grid, eps=eps, opts=P.SolverOptions(eps=eps, leaf_size=64, k_cut=None),
                           quad=P.PLAIN)
    xy = grid.points()
    f = np.exp(1j * 20.0 * (xy[:, 0] + 1.0))
    x = inv.apply(f)
    assert np.iscomplexobj(x)
    assert true_residual(spec, grid, P.PLAIN, f, x) <= 10 * eps


def test_rhs_dtypes_follow_result_type():
    """Result dtype = np.result_type(spec.dtype, f.dtype) (solver_dense.py:296):
    a complex f on a real system is solved as its real and imaginary parts;
    integer / float32 inputs are promoted; nrhs = 0 returns an empty result."""
    P, sd = _api()
    spec, grid, tree, H = setup(28)
    inv = sd.invert_dense_block(H)
    rng = np.random.default_rng(9)
    a, b = rng.standard_normal((grid.n, 2)), rng.standard_normal((grid.n, 2))
    xc = inv.apply(a + 1j * b)
    assert xc.dtype == np.complex128 and xc.shape == (grid.n, 2)
    # same columns, solved in a wider batch: equal up to the GEMM's
    # N-dependent reduction schedule
    close = lambda x, y: np.testing.assert_allclose(x, y, rtol=0, atol=1e-13 * np.abs(y).max())
    close(xc.real, inv.apply(a))
    close(xc.imag, inv.apply(b))
    x1 = inv.apply(a[:, 0] + 1j * b[:, 0])
    assert x1.shape == (grid.n,) and x1.dtype == np.complex128
    close(x1.real, inv.apply(a[:, 0]))
    yc = H.matvec(a + 1j * b)
    close(yc.imag, H.matvec(b))
    xt = inv.apply(torch.as_tensor(a + 1j * b, device="cuda"))
    assert xt.is_complex() and xt.is_cuda
    np.testing.assert_array_equal(xt.cpu().numpy(), xc)
    ints = rng.integers(-5, 5, grid.n)
    xi = inv.apply(ints)
    assert xi.dtype == np.float64
    np.testing.assert_array_equal(xi, inv.apply(ints.astype(np.float64)))
    f32 = a[:, 0].astype(np.float32)
    np.testing.assert_array_equal(inv.apply(f32), inv.apply(f32.astype(np.float64)))
    e = inv.apply(np.zeros((grid.n, 0)))
    assert e.shape == (grid.n, 0) and e.dtype == np.float64
    assert H.matvec(np.zeros((grid.n, 0))).shape == (grid.n, 0)
    with pytest.raises(ValueError):
        inv.apply(np.zeros(grid.n + 1))


def test_spill_to_host_memory_solves_bitwise():
    """invert_dense_block(spill=_Spill(threshold_mb)) (the reference's _Spill
    tier, solver_dense.py:37-55): factor batches above the threshold live in
    pinned host memory and are streamed back level by level during the solve;
    the solution is bitwise the in-HBM one and HBM holds far less."""
    P, sd = _api()
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                        c_field=P.make_field("one"))
    grid = P.Grid(128)
    tree = P.build_tree(grid, 64)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    f = np.random.default_rng(5).standard_normal((grid.n, 3))
    H = sd.compress_outer(spec, grid, tree, 1e-10, opts, P.CELL)
    x_ref = sd.invert_dense_block(H).apply(f)
    x1_ref = sd.invert_dense_block(H).apply(f[:, 0])
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated()
    inv = sd.invert_dense_block(H, spill=sd._Spill(0))
    held = torch.cuda.memory_allocated() - base
    host = [getattr(L, n) for L in H.levels for n in ("Finv", "C", "E", "W")
            if isinstance(getattr(L, n, None), torch.Tensor)]
    assert host and all(not t.is_cuda and t.is_pinned() for t in host)
    assert held < 0.1 * inv.nbytes(), (held, inv.nbytes())
    np.testing.assert_array_equal(inv.apply(f), x_ref)
    np.testing.assert_array_equal(inv.apply(f[:, 0]), x1_ref)
    # threshold above every block: nothing moves
    inv2 = sd.invert_dense_block(H, spill=1e6)
    assert all(getattr(L, "Finv", None) is None or L.Finv.is_cuda for L in H.levels)
    np.testing.assert_array_equal(inv2.apply(f), x_ref)
