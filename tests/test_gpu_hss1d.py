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
