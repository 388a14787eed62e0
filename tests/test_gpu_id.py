"""ID (K2) contracts, ported from the reference's test_dense_core.py:20-77 and
run on BOTH device paths (shared-memory classical QRCP and the blocked
randomized path), plus parity with the oracle's LAPACK ID on kernel blocks."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PATHS = [False, True]


def reconstruct(A, f):
    return A[:, f.skeleton] @ f.right_matrix(A.dtype)


def planted(rng, m, n, sv):
    u, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))))
    v, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))))
    return (u * sv) @ v.T


@pytest.mark.parametrize("blocked", PATHS)
def test_id_identity_full_rank(blocked):
    from paper_1303_5466_b200.dense_core import interp_decomp
    f = interp_decomp(np.eye(3), 1e-10, force_blocked=blocked)
    assert f.rank == 3 and f.T.shape == (3, 0)


@pytest.mark.parametrize("blocked", PATHS)
def test_id_rank_one(blocked):
    from paper_1303_5466_b200.dense_core import interp_decomp
    rng = np.random.default_rng(1)
    A = np.outer(rng.standard_normal(20), rng.standard_normal(30))
    f = interp_decomp(A, 1e-10, force_blocked=blocked)
    assert f.rank == 1
    assert np.linalg.norm(A - reconstruct(A, f), 2) <= 1e-10 * np.linalg.norm(A, 2)


@pytest.mark.parametrize("blocked", PATHS)
def test_id_skeleton_columns_exact(blocked):
    from paper_1303_5466_b200.dense_core import interp_decomp
    rng = np.random.default_rng(2)
    A = planted(rng, 40, 50, np.geomspace(1, 1e-12, 40))
    f = interp_decomp(A, 1e-8, force_blocked=blocked)
    rec = reconstruct(A, f)
    np.testing.assert_allclose(rec[:, f.skeleton], A[:, f.skeleton], atol=1e-13)


@pytest.mark.parametrize("blocked", PATHS)
def test_id_error_vs_svd_planted_spectra(blocked):
    from paper_1303_5466_b200.dense_core import interp_decomp_batched
    rng = np.random.default_rng(3)
    mats, svs = [], []
    for _ in range(200):
        m, n = int(rng.integers(10, 60)), int(rng.integers(10, 60))
        decay = 10.0 ** -rng.uniform(0.1, 1.0)
        sv = decay ** np.arange(min(m, n))
        mats.append(planted(rng, m, n, sv))
        svs.append(sv)
    res = interp_decomp_batched(mats, 1e-6, force_blocked=blocked)
    worst = 0.0
    for A, sv, (perm, k, T) in zip(mats, svs, res):
        n = A.shape[1]
        if k == min(A.shape):
            continue
        R = np.zeros((k, n))
        R[np.arange(k), perm[:k]] = 1.0
        R[:, perm[k:]] = T
        err = np.linalg.norm(A - A[:, perm[:k]] @ R, 2)
        worst = max(worst, err / (10.0 * np.sqrt(1.0 + k * (n - k)) * sv[k]))
    assert worst <= 1.0


@pytest.mark.parametrize("blocked", PATHS)
def test_id_laplace_block_rank_near_svd(blocked):
    from paper_1303_5466_b200 import Grid, KernelSpec, PLAIN, assemble_dense
    from paper_1303_5466_b200.dense_core import interp_decomp
    grid = Grid(14)
    spec = KernelSpec("laplace2d")
    n = grid.n_side
    ix, iy = np.meshgrid(np.arange(7), np.arange(7), indexing="xy")
    box1 = (iy * n + ix).ravel()
    box2 = (iy * n + ix + 7).ravel()
    A = assemble_dense(spec, grid, PLAIN, box1, box2)
    f = interp_decomp(A, 1e-10, force_blocked=blocked)
    sv = np.linalg.svd(A, compute_uv=False)
    assert abs(f.rank - int(np.sum(sv > 1e-10 * sv[0]))) <= 5


@pytest.mark.parametrize("shape", [(300, 200), (500, 450), (160, 64), (1200, 900)])
def test_blocked_id_on_kernel_rows_vs_oracle(shape):
    """Proxy-style smooth kernel block: blocked-path rank within a few of the
    LAPACK ID's and reconstruction error at the tolerance."""
    import oracle.hssd as O
    from paper_1303_5466_b200.dense_core import interp_decomp_batched
    p, m = shape
    rng = np.random.default_rng(7)
    src = rng.uniform(-1, 1, (m, 2)) * 0.5
    th = np.linspace(0, 2 * np.pi, p, endpoint=False)
    tgt = np.column_stack([1.2 * np.cos(th), 1.2 * np.sin(th)]) + rng.normal(0, 0.05, (p, 2))
    r = np.hypot(*(tgt[:, None, :] - src[None, :, :]).transpose(2, 0, 1))
    A = np.log(r)
    eps = 1e-10
    ref = O.column_id(A, eps)
    (perm, k, T), = interp_decomp_batched([A], eps, force_blocked=True)
    R = np.zeros((k, m))
    R[np.arange(k), perm[:k]] = 1.0
    R[:, perm[k:]] = T
    err = np.linalg.norm(A - A[:, perm[:k]] @ R) / np.linalg.norm(A)
    assert abs(k - ref.k) <= max(3, ref.k // 20), (k, ref.k)
    assert err <= 50 * eps, err
    assert len(set(perm.tolist())) == m


def test_blocked_id_tall_panel_two_stage():
    """Panels taller than one cluster holds (> 12288 rows; the level-1 boxes of
    a 2048^2 grid have 16416) go through the two-stage panel (TSQR of two row
    chunks + Householder reconstruction, csrc/tallpanel.cu).  Ragged batch:
    the second matrix is shorter, so its second chunk is shorter too; the
    third fits one cluster after the first blocks' rows are finished.  Same
    contract as the one-stage path: rank within a few of LAPACK's ID
    (oracle.column_id), reconstruction at the tolerance, perm a permutation."""
    import oracle.hssd as O
    from paper_1303_5466_b200.dense_core import interp_decomp_batched
    rng = np.random.default_rng(11)
    eps = 1e-10
    mats = []
    for p, m in [(16416, 144), (13001, 120), (12310, 96)]:
        src = rng.uniform(-1, 1, (m, 2)) * 0.5
        th = np.linspace(0, 2 * np.pi, p, endpoint=False)
        tgt = np.column_stack([1.3 * np.cos(th), 1.3 * np.sin(th)]) + rng.normal(0, 0.05, (p, 2))
        r = np.hypot(*(tgt[:, None, :] - src[None, :, :]).transpose(2, 0, 1))
        mats.append(np.log(r))
    res = interp_decomp_batched(mats, eps, force_blocked=True)
    for A, (perm, k, T) in zip(mats, res):
        m = A.shape[1]
        ref = O.column_id(A, eps)
        R = np.zeros((k, m))
        R[np.arange(k), perm[:k]] = 1.0
        R[:, perm[k:]] = T
        err = np.linalg.norm(A - A[:, perm[:k]] @ R) / np.linalg.norm(A)
        assert abs(k - ref.k) <= max(3, ref.k // 20), (k, ref.k)
        assert err <= 50 * eps, err
        assert len(set(perm.tolist())) == m
        assert np.abs(T).max() <= 10.0


def test_blocked_id_wide_block_tournament_selection():
    """More than 8192 live columns (16 CTAs x 512 thread-per-column slots; the
    level-1 boxes of a 2048^2 grid have ~12272): the sketch selection runs as
    a tournament over column ranges (csrc/panels.cu sketch_select_tournament).
    Same contract: rank within a few of LAPACK's ID, reconstruction at the
    tolerance, bounded interpolation coefficients.  The second matrix is
    narrower (its last range is empty)."""
    import oracle.hssd as O
    from paper_1303_5466_b200.dense_core import interp_decomp_batched
    rng = np.random.default_rng(13)
    eps = 1e-10
    mats = []
    for p, m in [(420, 9001), (380, 8200)]:
        src = rng.uniform(-1, 1, (m, 2)) * 0.5
        th = np.linspace(0, 2 * np.pi, p, endpoint=False)
        tgt = np.column_stack([1.5 * np.cos(th), 1.5 * np.sin(th)]) + rng.normal(0, 0.05, (p, 2))
        r = np.hypot(*(tgt[:, None, :] - src[None, :, :]).transpose(2, 0, 1))
        mats.append(np.log(r))
    res = interp_decomp_batched(mats, eps, force_blocked=True)
    for A, (perm, k, T) in zip(mats, res):
        m = A.shape[1]
        ref = O.column_id(A, eps)
        err = np.linalg.norm(A[:, perm[k:]] - A[:, perm[:k]] @ T) / np.linalg.norm(A)
        assert abs(k - ref.k) <= max(3, ref.k // 20), (k, ref.k)
        assert err <= 50 * eps, err
        assert len(set(perm.tolist())) == m
        assert np.abs(T).max() <= 10.0


def test_fixed_rank_is_least_squares():
    """vief_id_batched with kfix: no pivoting, rank = kfix, T = lstsq(A[:, :k],
    A[:, k:]) (the compressed path's interpolation).  Ragged batch: k off the
    32-column blocks, k = m, k = 0, p = k (square), several blocks."""
    from paper_1303_5466_b200.dense_core import interp_decomp_batched
    rng = np.random.default_rng(9)
    shapes = [(80, 64, 48), (150, 140, 100), (40, 40, 40), (70, 50, 0), (300, 200, 130),
              (100, 90, 100 - 10)]
    mats, ks = [], []
    for p, m, k in shapes:
        A = rng.standard_normal((p, m))
        A[:, :k] *= np.logspace(0, -2, k)  # graded skeleton columns
        mats.append(A)
        ks.append(k)
    out = interp_decomp_batched(mats, 1e-10, kfix=ks)
    for A, k, (perm, kk, T) in zip(mats, ks, out):
        assert kk == k
        np.testing.assert_array_equal(perm, np.arange(A.shape[1]))
        assert T.shape == (k, A.shape[1] - k)
        if k == 0 or k == A.shape[1]:
            continue
        ref = np.linalg.lstsq(A[:, :k], A[:, k:], rcond=None)[0]
        assert np.linalg.norm(T - ref) <= 1e-9 * np.linalg.norm(ref)


@pytest.mark.parametrize("blocked", PATHS)
def test_complex_id_vs_lapack(blocked):
    """Complex IDs (realified, pairwise pivots): a planted-spectrum complex
    matrix is reconstructed to ~eps like the reference's complex ?geqp3 ID,
    with the same rank (dense_core.py:67-100 on complex input)."""
    import scipy.linalg as sla
    from paper_1303_5466_b200.dense_core import interp_decomp
    rng = np.random.default_rng(7)
    m, n = 180, 120
    sv = np.logspace(0, -14, min(m, n))
    u, _ = np.linalg.qr(rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    A = (u * sv) @ v.conj().T
    eps = 1e-8
    f = interp_decomp(A, eps, force_blocked=blocked)
    assert f.T.dtype == np.complex128
    assert np.unique(f.perm).size == n
    err = np.linalg.norm(A - reconstruct(A, f), 2) / np.linalg.norm(A, 2)
    _, r, _ = sla.qr(A, mode="economic", pivoting=True)
    d = np.abs(np.diag(r))
    k_ref = int(np.argmax(d <= eps * d[0])) if (d <= eps * d[0]).any() else d.size
    assert err <= 100 * eps, err
    assert abs(f.rank - k_ref) <= 2, (f.rank, k_ref)
    g = interp_decomp(A, eps, min_rank=f.rank + 5, force_blocked=blocked)   # clamp on the device
    assert g.rank == f.rank + 5
    assert np.linalg.norm(A - reconstruct(A, g), 2) / np.linalg.norm(A, 2) <= 100 * eps


def test_leaf_qrcp_matches_lapack():
    """Leaf-size IDs (p <= 160, m <= 64: the register-resident dlaqp2 kernel)
    against LAPACK's ?geqp3 ID on proxy-style kernel rows: same rank, nearly
    the same pivots, reconstruction at the tolerance; pair mode keeps
    (2t, 2t+1) columns together."""
    import oracle.hssd as O
    from paper_1303_5466_b200.dense_core import interp_decomp_batched
    rng = np.random.default_rng(11)
    mats = []
    for _ in range(64):
        p, m = int(rng.integers(100, 161)), int(rng.integers(40, 65)) & ~1
        src = rng.uniform(-1, 1, (m, 2)) * 0.25
        th = np.linspace(0, 2 * np.pi, p, endpoint=False)
        tgt = np.column_stack([0.8 * np.cos(th), 0.8 * np.sin(th)]) + rng.normal(0, 0.02, (p, 2))
        mats.append(np.log(np.hypot(*(tgt[:, None, :] - src[None, :, :]).transpose(2, 0, 1))))
    eps = 1e-10
    same = tot = 0
    for pairs in (False, True):
        res = interp_decomp_batched(mats, eps, pairs=pairs)
        for A, (perm, k, T) in zip(mats, res):
            m = A.shape[1]
            R = np.zeros((k, m))
            R[np.arange(k), perm[:k]] = 1.0
            R[:, perm[k:]] = T
            err = np.linalg.norm(A - A[:, perm[:k]] @ R) / np.linalg.norm(A)
            ref = O.column_id(A, eps)
            Rr = np.zeros((ref.k, m))
            Rr[np.arange(ref.k), ref.perm[:ref.k]] = 1.0
            Rr[:, ref.perm[ref.k:]] = ref.T
            err_ref = np.linalg.norm(A - A[:, ref.perm[:ref.k]] @ Rr) / np.linalg.norm(A)
            assert err <= max(50 * eps, 5 * err_ref), (err, err_ref)
            assert sorted(perm.tolist()) == list(range(m))
            if pairs:
                assert k % 2 == 0 and (perm[:k:2] ^ 1 == perm[1:k:2]).all()
                continue
            assert abs(k - ref.k) <= 1, (k, ref.k)
            same += int(np.intersect1d(perm[:k], ref.perm[:ref.k]).size)
            tot += ref.k
    assert same >= 0.95 * tot, (same, tot)


@pytest.mark.parametrize("blocked", [False, True])
def test_eps_abs_floor(blocked):
    """interp_decomp's absolute floor (dense_core.py:82-88): the rank is the
    first j with |R_jj| <= max(eps |R_00|, eps_abs); a floor above |R_00| gives
    rank 0 (then min_rank clamps)."""
    import scipy.linalg as sla
    from paper_1303_5466_b200.dense_core import interp_decomp
    rng = np.random.default_rng(21)
    m, n = 90, 70
    sv = 10.0 ** -np.linspace(0, 12, n)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (u * sv) @ v.T
    _, r, _ = sla.qr(A, mode="economic", pivoting=True)
    d = np.abs(np.diag(r))
    for eps_abs in (1e-4, 3e-7):
        cut = max(1e-12 * d[0], eps_abs)
        k_ref = int(np.argmax(d <= cut))
        f = interp_decomp(A, 1e-12, eps_abs=eps_abs, force_blocked=blocked)
        assert abs(f.rank - k_ref) <= 2, (f.rank, k_ref)
        assert np.linalg.norm(A - reconstruct(A, f), 2) <= 100 * eps_abs
    assert interp_decomp(A, 1e-12, eps_abs=10.0 * d[0], force_blocked=blocked).rank == 0
    assert interp_decomp(A, 1e-12, eps_abs=10.0 * d[0], min_rank=3, force_blocked=blocked).rank == 3
