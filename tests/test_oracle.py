"""The CPU oracle (oracle/hssd.py) pinned against golden vectors produced by
the REFERENCE implementation (tests/golden/make_golden.py): tree and proxy /
near-field integers bit-exact, matrix entries bit-exact, and the full
compress + invert + apply path reproducing the reference's solutions."""
import math
import os

import numpy as np
import pytest

import oracle.hssd as O

G = os.path.join(os.path.dirname(__file__), "golden")


def _npz(name):
    return np.load(os.path.join(G, name))


TREES = [(7, 49), (14, 49), (28, 49), (18, 81), (9, 25), (30, 64), (128, 64), (64, 64)]


@pytest.mark.parametrize("n,nmax", TREES)
def test_oracle_tree_bitexact(n, nmax):
    g = _npz("trees.npz")
    t = O.make_tree(n, nmax)
    np.testing.assert_array_equal(t.rect, g[f"t{n}_{nmax}_rect"])
    np.testing.assert_array_equal(t.level, g[f"t{n}_{nmax}_level"])
    np.testing.assert_array_equal(t.parent, g[f"t{n}_{nmax}_parent"])
    np.testing.assert_array_equal(t.kids, g[f"t{n}_{nmax}_kids"])


@pytest.mark.parametrize("n,nmax", [(28, 49), (18, 81), (30, 64)])
@pytest.mark.parametrize("pad", [1, 2, 3])
def test_oracle_proxy_and_near_bitexact(n, nmax, pad):
    g = _npz("geometry.npz")
    t = O.make_tree(n, nmax)
    for b in range(len(t.rect)):
        np.testing.assert_array_equal(O.proxy_ring(t.rect[b], pad), g[f"p{n}_{pad}_{b}"])
        np.testing.assert_array_equal(O.near_field(t.rect[b], n, pad), g[f"n{n}_{pad}_{b}"])


SPECS = {
    "nti": dict(family="laplace2d", b=("gaussian_bump", ()), c=("gaussian_bump", ())),
    "rows": dict(family="laplace2d", b=("centre_bump", (("scale", math.pi / 2),)), c=("one", ())),
    "helm": dict(family="helmholtz2d", k=2 * np.pi * 2),
    "yuk": dict(family="yukawa2d", k=3.0, b=("gaussian_bump", ())),
}


def _problem(name, n, quad):
    kw = dict(SPECS[name])
    return O.Problem(n, kw.pop("family"), kw.pop("k", 0.0), ("one", ()), kw.pop("b", ("one", ())),
                     kw.pop("c", ("one", ())), {"plain": "none", "h4": "h4", "cell": "cell"}[quad])


@pytest.mark.parametrize("spec", list(SPECS))
@pytest.mark.parametrize("quad", ["plain", "h4", "cell"])
def test_oracle_entries_bitexact(spec, quad):
    if quad == "cell" and SPECS[spec]["family"] != "laplace2d":
        pytest.skip("cell diagonal is Laplace-only")
    g = _npz("entries.npz")
    for n in (4, 12):
        P = _problem(spec, n, quad)
        np.testing.assert_array_equal(O.dense_matrix(P), g[f"A_{spec}_{quad}_{n}"])
    P = _problem(spec, 12, quad)
    t = O.make_tree(12, 36)
    rows = t.owned(3)
    zp = O.proxy_ring(t.rect[3], 2)
    np.testing.assert_array_equal(O.proxy_src(P, rows, zp), g[f"pc_{spec}_{quad}"])
    np.testing.assert_array_equal(O.proxy_tgt(P, zp, rows), g[f"pr_{spec}_{quad}"])


CASES = {
    "nti28": (dict(family="laplace2d", b=("gaussian_bump", ()), c=("gaussian_bump", ())), 28, 49, 1e-10, "none"),
    "rows14": (dict(family="laplace2d", b=("gaussian_bump", ()), c=("one", ())), 14, 49, 1e-10, "none"),
    "rows30": (dict(family="laplace2d", b=("gaussian_bump", ()), c=("one", ())), 30, 64, 1e-10, "none"),
    "helm18": (dict(family="helmholtz2d", k=2 * np.pi * 2), 18, 81, 1e-10, "none"),
    "single7": (dict(family="laplace2d", b=("gaussian_bump", ()), c=("gaussian_bump", ())), 7, 49, 1e-10, "none"),
    "eps5_28": (dict(family="laplace2d", b=("gaussian_bump", ()), c=("one", ())), 28, 49, 1e-5, "h4"),
}


@pytest.mark.parametrize("case", list(CASES))
def test_oracle_solves_match_reference(case):
    kw, n, leaf, eps, quad = CASES[case]
    kw = dict(kw)
    g = _npz(f"solve_{case}.npz")
    P = O.Problem(n, kw.pop("family"), kw.pop("k", 0.0), ("one", ()), kw.pop("b", ("one", ())),
                  kw.pop("c", ("one", ())), quad)
    x, H, inv = O.solve(P, leaf, eps, g["f"])
    tree = H.tree
    rank = np.array([H.rskel[b].size if b in H.rskel else -1 for b in range(len(tree.rect))])
    np.testing.assert_array_equal(rank, g["rank"])
    np.testing.assert_array_equal(np.concatenate([H.rskel.get(b, np.zeros(0, int)) for b in range(len(tree.rect))]),
                                  g["row_skel"])
    assert np.linalg.norm(x - g["x"]) <= 1e-12 * np.linalg.norm(g["x"])
    assert inv.nbytes() == int(g["nbytes_inv"])
    hx = O.matvec(H, x)
    assert np.linalg.norm(hx - g["hx"]) <= 1e-12 * np.linalg.norm(g["hx"])


def test_oracle_singular_raises():
    A = np.zeros((3, 3))
    A[0, 0] = 1.0
    with pytest.raises(O.Singular):
        O.lu_checked(A, "x")


def test_oracle_digest_geometry_128():
    import hashlib
    g = _npz("geometry.npz")
    for n in (128, 256):
        t = O.make_tree(n, 64)
        for kind, fn in (("proxy", lambda r: O.proxy_ring(r, 2)), ("near", lambda r: O.near_field(r, n, 2))):
            h = hashlib.sha256()
            for b in range(len(t.rect)):
                h.update(np.ascontiguousarray(np.asarray(fn(t.rect[b]), np.int64)).tobytes())
                h.update(b"|")
            assert h.hexdigest() == bytes(g[f"dig_{kind}_{n}"]).decode()
