"""Host-side (CPU) logic of the product package: tree, proxy/near geometry,
options, fields, errors, and the C-ABI library's exported surface.  No GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1303_5466_b200 import (CELL, H4, PLAIN, ConfigError, Grid, KernelSpec,
                                  QuadratureCorrection, SingularFactorError, SolverOptions,
                                  build_tree, kernel_eval, make_field)
from paper_1303_5466_b200.tree import near_count, near_field_indices, proxy_count, proxy_points

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")

TREES = [(7, 49), (14, 49), (28, 49), (18, 81), (9, 25), (30, 64), (128, 64), (64, 64)]


@pytest.mark.parametrize("n,nmax", TREES)
def test_build_tree_matches_reference(n, nmax):
    g = np.load(os.path.join(G, "trees.npz"))
    t = build_tree(Grid(n), nmax)
    rect = np.array([(b.x0, b.x1, b.y0, b.y1) for b in t.nodes])
    np.testing.assert_array_equal(rect, g[f"t{n}_{nmax}_rect"])
    np.testing.assert_array_equal([b.level for b in t.nodes], g[f"t{n}_{nmax}_level"])
    np.testing.assert_array_equal([b.parent for b in t.nodes], g[f"t{n}_{nmax}_parent"])
    kids = np.array([b.children if b.children else (-1, -1) for b in t.nodes])
    np.testing.assert_array_equal(kids, g[f"t{n}_{nmax}_kids"])
    # per-level arrays agree with the node list
    for lv in range(t.depth + 1):
        np.testing.assert_array_equal(t.rects[lv], rect[t.levels[lv]])


def test_tree_reference_pins():
    t = build_tree(Grid(28), 49)          # test_tree.py:10-16
    assert t.depth == 4 and len(t.leaves()) == 16
    assert all(b.npoints == 49 for b in t.leaves())
    t1 = build_tree(Grid(7), 49)
    assert t1.depth == 0 and t1.root.is_leaf
    allidx = np.concatenate([t.owned_indices(b) for b in t.leaves()])
    np.testing.assert_array_equal(np.sort(allidx), np.arange(28 * 28))
    own = t.owned_level(t.depth)
    np.testing.assert_array_equal(own, np.stack([t.owned_indices(b) for b in t.leaves()]))


def test_tree_errors():
    with pytest.raises(ConfigError):
        build_tree(Grid(8), 3)
    with pytest.raises(ConfigError):
        build_tree(Grid(3), 49)
    with pytest.raises(ConfigError):
        build_tree(Grid(9), 16)   # 4x4 and 5x5 leaves straddle the leaf size


@pytest.mark.parametrize("n,nmax", [(28, 49), (18, 81), (30, 64)])
def test_proxy_and_near_match_reference(n, nmax):
    g = np.load(os.path.join(G, "geometry.npz"))
    t = build_tree(Grid(n), nmax)
    for pad in (1, 2, 3):
        for b in t.nodes:
            pp = proxy_points(b, pad)
            np.testing.assert_array_equal(pp, g[f"p{n}_{pad}_{b.idx}"])
            assert proxy_count(b.width, b.height, pad) == len(pp)
            nf = near_field_indices(b, t.grid, pad)
            np.testing.assert_array_equal(nf, g[f"n{n}_{pad}_{b.idx}"])
            assert near_count(np.array([[b.x0, b.x1, b.y0, b.y1]]), n, pad)[0] == len(nf)


def test_proxy_ring_enumeration_oracle():
    box = build_tree(Grid(7), 49).root   # test_tree.py:89-100
    ring1 = proxy_points(box, 1)
    cells = {(x, y) for x in range(-1, 8) for y in range(-1, 8) if not (0 <= x < 7 and 0 <= y < 7)}
    assert len(ring1) == len(cells) == 32 and {tuple(c) for c in ring1} == cells
    pts = proxy_points(box, 2, budget=40)
    assert pts.shape[0] == 40 and len({tuple(c) for c in pts}) == 40


def test_options_and_layers():
    o = SolverOptions()
    lap = KernelSpec("laplace2d")
    assert o.resolved_proxy_layers(lap) == 2
    assert SolverOptions(eps=1e-4).resolved_proxy_layers(lap) == 1
    assert SolverOptions(proxy_layers=3).resolved_proxy_layers(lap) == 3
    assert o.resolved_layers(KernelSpec("helmholtz2d", k=2 * np.pi * 8)) == 2
    assert o.resolved_layers(KernelSpec("helmholtz2d", k=2 * np.pi * 20)) == 3
    with pytest.raises(ConfigError):
        o.resolved_layers(KernelSpec("helmholtz2d", k=2 * np.pi * 40))
    assert o.with_(eps=1e-6).eps == 1e-6


def test_fields_and_specs():
    with pytest.raises(ConfigError):
        make_field("nope")
    with pytest.raises(ConfigError):
        KernelSpec("laplace2d", k=1.0)
    with pytest.raises(ConfigError):
        KernelSpec("helmholtz2d")
    with pytest.raises(ConfigError):
        KernelSpec("bogus")
    spec = KernelSpec("laplace2d", b_field=make_field("gaussian_bump"),
                      c_field=make_field("gaussian_bump"))
    assert spec.symmetric and not spec.translation_invariant
    assert KernelSpec("laplace2d").translation_invariant
    assert kernel_eval(KernelSpec("laplace2d"), 1.0) == 0.0
    assert np.isclose(kernel_eval(KernelSpec("laplace2d"), np.e), 1 / (2 * np.pi), rtol=1e-15)
    with pytest.raises(ValueError):
        kernel_eval(KernelSpec("laplace2d"), 0.0)
    with pytest.raises(ConfigError):
        QuadratureCorrection("bad")
    h = Grid(64).h
    assert PLAIN.diagonal_term(KernelSpec("laplace2d"), h) == 0.0
    assert np.isclose(CELL.diagonal_term(KernelSpec("laplace2d"), h),
                      (np.log(h) - 1.5 + np.pi / 4 - 0.5 * np.log(2)) / (2 * np.pi))
    assert H4.diagonal_term(KernelSpec("laplace2d"), h) != 0.0


def test_singular_error_carries_context():
    e = SingularFactorError("box 3 level 2", 1e-301)
    assert e.where == "box 3 level 2" and e.pivot == 1e-301
    assert "box 3 level 2" in str(e)


def test_library_exports_every_header_symbol():
    from paper_1303_5466_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    hdr = open(os.path.join(ROOT, "include", "vief_b200.h")).read()
    names = sorted(set(re.findall(r"\b(vief_[a-z0-9_]+)\s*\(", hdr)))
    assert len(names) >= 15
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(_lib.exported_symbols())
    assert lib.vief_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    from paper_1303_5466_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.LibraryError):
        _lib.require_cuda()
