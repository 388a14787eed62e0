"""Batched library calls with more items than one CUDA grid dimension holds
(65 535): every C-ABI entry point splits such a batch into chunks; results
must equal the item-by-item reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
NB = 70001


def test_gemm_gemv_copy_gather_in_chunks():
    from paper_1303_5466_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn((NB, 5, 4), dtype=torch.float64, device="cuda", generator=g)   # 4 x 5 col-major
    B = torch.randn((NB, 3, 5), dtype=torch.float64, device="cuda", generator=g)   # 5 x 3
    C = torch.zeros((NB, 3, 4), dtype=torch.float64, device="cuda")
    _lib.gemm(A, B, C, M=4, N=3, K=5, lda=4, ldb=5, ldc=4, sA=20, sB=15, sC=12, batch=NB)
    ref = torch.bmm(B, A)          # (B^T-layout) C^T = B^T A^T
    assert torch.allclose(C, ref, rtol=1e-13, atol=1e-13)
    x = torch.randn((NB, 5), dtype=torch.float64, device="cuda", generator=g)
    y = torch.zeros((NB, 4), dtype=torch.float64, device="cuda")
    _lib.gemv(A, x, y, M=4, K=5, lda=4, sA=20, sx=5, sy=4, batch=NB)
    assert torch.allclose(y, torch.einsum("bkm,bk->bm", A, x), rtol=1e-13, atol=1e-13)
    D = torch.zeros_like(A)
    _lib.copy2d(A, 20, 4, D, 20, 4, None, 4, None, 5, NB)
    assert torch.equal(D, A)
    # rows gathered per item: dst[c, b*3 + i] = src[c, b*4 + idx[b, i]]
    src = torch.randn((2, NB * 4), dtype=torch.float64, device="cuda", generator=g)
    idx = torch.stack([torch.randperm(4, device="cuda", generator=g)[:3] for _ in range(8)]).int()
    idx = idx.repeat((NB + 7) // 8, 1)[:NB].contiguous()
    dst = torch.zeros((2, NB * 3), dtype=torch.float64, device="cuda")
    n3 = torch.full((NB,), 3, dtype=torch.int32, device="cuda")
    _lib.gather_rows(src, 4, NB * 4, idx, 3, dst, 3, NB * 3, n3, 3, None, 2, NB)
    ref = src.reshape(2, NB, 4).gather(2, idx.long()[None].expand(2, NB, 3)).reshape(2, NB * 3)
    assert torch.equal(dst, ref)
    back = torch.zeros_like(src)
    _lib.scatter_rows(dst, 3, NB * 3, idx, 3, back, 4, NB * 4, n3, 3, None, 2, NB)
    chk = torch.zeros((2, NB, 4), dtype=torch.float64, device="cuda")
    chk.scatter_(2, idx.long()[None].expand(2, NB, 3), ref.reshape(2, NB, 3))
    assert torch.equal(back, chk.reshape(2, NB * 4))


def test_inverse_and_id_in_chunks():
    from paper_1303_5466_b200 import _lib
    from paper_1303_5466_b200 import solver_dense as sd
    g = torch.Generator(device="cuda").manual_seed(4)
    M = torch.randn((NB, 3, 3), dtype=torch.float64, device="cuda", generator=g)
    M = M + 4.0 * torch.eye(3, dtype=torch.float64, device="cuda")
    X = M.clone()
    pmin, pmax = _lib.inv_batched(X, 9, 3, 3, NB)
    eye = torch.eye(3, dtype=torch.float64, device="cuda").expand(NB, 3, 3)
    assert torch.allclose(torch.bmm(X, M), eye, atol=1e-11)
    assert bool((pmin > 0).all()) and bool((pmax >= pmin).all())
    # IDs: 8 x 6 items of rank 3 (pairs with coupled ranks)
    p, m, k = 8, 6, 3
    U = torch.randn((NB, p, k), dtype=torch.float64, device="cuda", generator=g)
    V = torch.randn((NB, k, m), dtype=torch.float64, device="cuda", generator=g)
    A = torch.bmm(U, V)                                   # (NB, p, m)
    Ad = A.transpose(1, 2).contiguous()                   # item: m columns of length p
    pv = torch.full((NB,), p, dtype=torch.int32, device="cuda")
    mv = torch.full((NB,), m, dtype=torch.int32, device="cuda")
    cnt = NB - NB % 2
    rank = torch.zeros(cnt, dtype=torch.int32, device="cuda")
    perm = torch.zeros((cnt, m), dtype=torch.int32, device="cuda")
    T = torch.zeros((cnt, m, m), dtype=torch.float64, device="cuda")
    sd._id_batched("cuda", Ad[:cnt].clone(), m * p, p, pv, mv, p, m, cnt, 2, 1e-10, rank, perm, T, 1, 0)
    assert bool((rank == k).all())
    pl = perm.long()
    Ap = A[:cnt].gather(2, pl[:, None, :].expand(cnt, p, m))        # columns in pivot order
    Tk = T[:, :m - k, :k].transpose(1, 2)                           # (cnt, k, m - k)
    err = (Ap[:, :, k:] - torch.bmm(Ap[:, :, :k], Tk)).abs().amax()
    assert float(err) <= 1e-9 * float(A.abs().amax())
