"""K1 on the B200: matrix entries bit-identical to the reference's numpy
assembly (golden vectors from the reference), the reference's kernel-level
pins (test_kernels.py), and device proxy/near geometry bit-identical to the
reference's enumeration."""
import ctypes
import hashlib
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def _specs():
    from paper_1303_5466_b200 import KernelSpec, make_field
    return {
        "nti": KernelSpec("laplace2d", b_field=make_field("gaussian_bump"),
                          c_field=make_field("gaussian_bump")),
        "rows": KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                           c_field=make_field("one")),
        "helm": KernelSpec("helmholtz2d", k=2 * np.pi * 2),
        "yuk": KernelSpec("yukawa2d", k=3.0, b_field=make_field("gaussian_bump")),
    }


@pytest.mark.parametrize("spec", ["nti", "rows", "helm", "yuk"])
@pytest.mark.parametrize("quad", ["plain", "h4", "cell"])
def test_entries_bitexact_vs_reference(spec, quad):
    from paper_1303_5466_b200 import CELL, H4, PLAIN, Grid, assemble_dense, build_tree, get_assembler, proxy_points
    from paper_1303_5466_b200 import solver_dense as sd
    s = _specs()[spec]
    if quad == "cell" and s.family != "laplace2d":
        pytest.skip("cell diagonal is Laplace-only")
    q = {"plain": PLAIN, "h4": H4, "cell": CELL}[quad]
    g = np.load(os.path.join(G, "entries.npz"))
    for n in (4, 12):
        idx = np.arange(n * n)
        A = assemble_dense(s, Grid(n), q, idx, idx)
        np.testing.assert_array_equal(A, g[f"A_{spec}_{quad}_{n}"])
    # proxy row/column blocks through the ID-matrix generator
    if s.is_complex:
        return
    asm = get_assembler(s, Grid(12), q)
    tree = build_tree(Grid(12), 36)
    box = tree.nodes[3]
    rows = tree.owned_indices(box)
    zp = proxy_points(box, 2)
    dev = "cuda"
    pts = torch.as_tensor(rows.astype(np.int32), device=dev)
    sx = torch.as_tensor(zp.astype(np.int32), device=dev).contiguous()
    sg = torch.full((len(zp),), -1, dtype=torch.int32, device=dev)
    p, m = len(zp), len(rows)
    out = torch.empty((m, p), dtype=torch.float64, device=dev)
    from paper_1303_5466_b200 import _lib
    for kind, key in ((0, "pc"), (1, "pr")):
        _lib.call("vief_gen_idmat", ctypes.byref(asm.problem), kind, _lib.ptr(pts), 0, None, m,
                  _lib.ptr(sx), _lib.ptr(sg), 0, None, p, _lib.ptr(out), 0, p, 1,
                  _lib.stream_handle())
        got = out.t().cpu().numpy()  # p x m
        ref = g[f"{key}_{spec}_{quad}"]
        np.testing.assert_array_equal(got, ref.T if kind == 0 else ref)


def test_kernel_pins_from_reference_tests():
    from paper_1303_5466_b200 import Grid, KernelSpec, PLAIN, assemble_dense, assemble_entry
    grid = Grid(4)
    assert assemble_entry(KernelSpec("laplace2d"), grid, PLAIN, 3, 3) == 1.0
    spec = _specs()["nti"]
    rng = np.random.default_rng(0)
    g8 = Grid(8)
    for _ in range(20):
        i, j = (int(v) for v in rng.integers(0, g8.n, size=2))
        assert assemble_entry(spec, g8, PLAIN, i, j) == assemble_entry(spec, g8, PLAIN, j, i)
    lap = KernelSpec("laplace2d")
    assert assemble_entry(lap, g8, PLAIN, 9, 20) == assemble_entry(lap, g8, PLAIN, 12, 23)
    g14 = Grid(14)
    full = assemble_dense(spec, g14, PLAIN, np.arange(196), np.arange(196))
    I, J = np.arange(49), np.arange(49, 196)
    np.testing.assert_array_equal(assemble_dense(spec, g14, PLAIN, I, J), full[np.ix_(I, J)])
    assert assemble_dense(spec, g14, PLAIN, np.array([0]), np.zeros(0, np.int64)).shape == (1, 0)


def test_dense_entry_cap():
    import paper_1303_5466_b200.kernels as K
    from paper_1303_5466_b200 import Grid, KernelSpec, PLAIN, ResourceError
    old = K.DENSE_ENTRY_CAP
    K.DENSE_ENTRY_CAP = 10_000
    try:
        with pytest.raises(ResourceError):
            K.assemble_dense(KernelSpec("laplace2d"), Grid(64), PLAIN, np.arange(4096), np.arange(4096))
    finally:
        K.DENSE_ENTRY_CAP = old


def _device_sources(rects, pad, n):
    from paper_1303_5466_b200 import _lib
    from paper_1303_5466_b200.tree import near_count, proxy_count
    p = np.array([proxy_count(int(r[1] - r[0]), int(r[3] - r[2]), pad) for r in rects])
    p = p + near_count(rects, n, pad)
    pmax = int(p.max())
    nb = len(rects)
    R = torch.as_tensor(rects.astype(np.int32), device="cuda")
    xy = torch.empty((nb, pmax, 2), dtype=torch.int32, device="cuda")
    gg = torch.empty((nb, pmax), dtype=torch.int32, device="cuda")
    pd = torch.empty(nb, dtype=torch.int32, device="cuda")
    _lib.call("vief_box_sources", _lib.ptr(R), nb, pad, n, _lib.ptr(xy), _lib.ptr(gg), pmax,
              _lib.ptr(pd), _lib.stream_handle())
    return p, xy.cpu().numpy(), gg.cpu().numpy(), pd.cpu().numpy()


@pytest.mark.parametrize("n,nmax", [(28, 49), (18, 81), (30, 64)])
@pytest.mark.parametrize("pad", [1, 2, 3])
def test_device_proxy_near_bitexact(n, nmax, pad):
    from paper_1303_5466_b200 import Grid, build_tree
    g = np.load(os.path.join(G, "geometry.npz"))
    t = build_tree(Grid(n), nmax)
    rects = np.array([(b.x0, b.x1, b.y0, b.y1) for b in t.nodes])
    p, xy, gg, pd = _device_sources(rects, pad, n)
    np.testing.assert_array_equal(pd, p)
    for b in t.nodes:
        ref_p = g[f"p{n}_{pad}_{b.idx}"]
        ref_n = g[f"n{n}_{pad}_{b.idx}"]
        npx = len(ref_p)
        np.testing.assert_array_equal(xy[b.idx, :npx], ref_p)
        assert (gg[b.idx, :npx] == -1).all()
        np.testing.assert_array_equal(gg[b.idx, npx:p[b.idx]], ref_n)


@pytest.mark.parametrize("n", [128, 256])
def test_device_geometry_digest_vs_reference(n):
    from paper_1303_5466_b200 import Grid, build_tree
    g = np.load(os.path.join(G, "geometry.npz"))
    t = build_tree(Grid(n), 64)
    rects = np.array([(b.x0, b.x1, b.y0, b.y1) for b in t.nodes])
    p, xy, gg, pd = _device_sources(rects, 2, n)
    hp, hn = hashlib.sha256(), hashlib.sha256()
    from paper_1303_5466_b200.tree import proxy_count
    for b in t.nodes:
        npx = proxy_count(b.width, b.height, 2)
        hp.update(np.ascontiguousarray(xy[b.idx, :npx].astype(np.int64)).tobytes()); hp.update(b"|")
        hn.update(np.ascontiguousarray(gg[b.idx, npx:p[b.idx]].astype(np.int64)).tobytes()); hn.update(b"|")
    assert hp.hexdigest() == bytes(g[f"dig_proxy_{n}"]).decode()
    assert hn.hexdigest() == bytes(g[f"dig_near_{n}"]).decode()
