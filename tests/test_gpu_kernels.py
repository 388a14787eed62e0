"""GPU kernel parity: DMMA GEMM/GEMV vs an fp64 reference, batched
Gauss-Jordan inverse, K1 entries bit-exact vs the oracle, device proxy/near
geometry bit-exact vs the reference's enumeration, and the ID contracts of
the reference's test_dense_core.py:20-77."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1303_5466_b200 import _lib
    _lib.require_cuda()
    return _lib


@pytest.mark.parametrize("tA,tB", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dgemm_batched_ragged(lib, tA, tB):
    rng = np.random.default_rng(0)
    nb, M, N, K = 5, 70, 45, 37
    dev = "cuda"
    A = torch.randn(nb, M if tA else K, K if tA else M, dtype=torch.float64, device=dev)
    B = torch.randn(nb, K if tB else N, N if tB else K, dtype=torch.float64, device=dev)
    # storage is column-major: tensor [item, col, row]
    Mb = torch.tensor(rng.integers(1, M + 1, nb), dtype=torch.int32, device=dev)
    Nb = torch.tensor(rng.integers(1, N + 1, nb), dtype=torch.int32, device=dev)
    Kb = torch.tensor(rng.integers(0, K + 1, nb), dtype=torch.int32, device=dev)
    C = torch.randn(nb, N, M, dtype=torch.float64, device=dev)
    C0 = C.clone()
    lda = A.shape[2]
    ldb = B.shape[2]
    lib.gemm(A, B, C, M=M, N=N, K=K, lda=lda, ldb=ldb, ldc=M, sA=A[0].numel(), sB=B[0].numel(),
             sC=M * N, tA=tA, tB=tB, alpha=-0.5, beta=2.0, batch=nb, Mb=Mb, Nb=Nb, Kb=Kb)
    for b in range(nb):
        m, n, k = int(Mb[b]), int(Nb[b]), int(Kb[b])
        Am = A[b].t()  # stored matrix (rows x cols)
        opA = (Am.t() if tA else Am)[:m, :k]
        Bm = B[b].t()
        opB = (Bm.t() if tB else Bm)[:k, :n]
        ref = -0.5 * opA @ opB + 2.0 * C0[b].t()[:m, :n]
        got = C[b].t()[:m, :n]
        assert torch.allclose(got, ref, rtol=1e-13, atol=1e-13)
        assert torch.equal(C[b].t()[m:, :], C0[b].t()[m:, :])


@pytest.mark.parametrize("tA", [0, 1])
def test_dgemv_batched(lib, tA):
    nb, M, K = 7, 300, 1100
    dev = "cuda"
    A = torch.randn(nb, M if tA else K, K if tA else M, dtype=torch.float64, device=dev)
    x = torch.randn(nb, K, dtype=torch.float64, device=dev)
    y = torch.randn(nb, M, dtype=torch.float64, device=dev)
    y0 = y.clone()
    lib.gemv(A, x, y, M=M, K=K, lda=A.shape[2], sA=A[0].numel(), sx=K, sy=M, tA=tA,
             alpha=1.5, beta=-1.0, batch=nb)
    for b in range(nb):
        Am = A[b].t()
        op = Am.t() if tA else Am
        ref = 1.5 * op @ x[b] - y0[b]
        assert torch.allclose(y[b], ref, rtol=1e-12, atol=1e-12)
    # bitwise determinism (solver_dense apply requirement)
    y2 = y0.clone()
    lib.gemv(A, x, y2, M=M, K=K, lda=A.shape[2], sA=A[0].numel(), sx=K, sy=M, tA=tA,
             alpha=1.5, beta=-1.0, batch=nb)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("n", [1, 5, 64, 65, 100, 128, 129, 257])
def test_inverse_batched(lib, n):
    nb = 4
    A = torch.randn(nb, n, n, dtype=torch.float64, device="cuda") + 3 * torch.eye(n, device="cuda", dtype=torch.float64)
    A[1] = torch.randn(n, n, dtype=torch.float64)  # needs pivoting
    X = A.clone()
    pmin, pmax = lib.inv_batched(X, n * n, n, n, nb)
    for b in range(nb):
        M = A[b].t()
        Xi = X[b].t()
        assert torch.allclose(M @ Xi, torch.eye(n, dtype=torch.float64, device="cuda"), atol=1e-9)
        lu = torch.linalg.lu_factor(M.cpu())[0]
        d = lu.diagonal().abs()
        assert np.isclose(float(pmin[b]), float(d.min()), rtol=1e-8)
        assert np.isclose(float(pmax[b]), float(d.max()), rtol=1e-8)


def test_inverse_singular_reports_zero_pivot(lib):
    A = torch.zeros(1, 3, 3, dtype=torch.float64, device="cuda")
    A[0, 0, 0] = 1.0
    pmin, pmax = lib.inv_batched(A, 9, 3, 3, 1)
    assert float(pmin[0]) == 0.0
