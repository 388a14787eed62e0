"""Factor persistence (persist.py, the analogue of the
reference's _Spill memmaps solver_dense.py:37-55 and hss1d to_blob/from_blob
hss1d/ops.py:218-267).  CPU tests cover the file format with host tensors;
GPU tests check that a loaded factorization solves bitwise like the saved one."""
import numpy as np
import pytest
import torch

from paper_1303_5466_b200 import persist


def _roundtrip(tmp_path, levels, problem=None):
    path = str(tmp_path / "f.vief")
    persist.write_state(path, problem or {"x": 1}, "test", levels)
    return persist.read_state(path, "cpu")


def test_format_roundtrip_cpu(tmp_path):
    base = torch.randn(5, 7, 3, dtype=torch.float64)
    view = base[2]                                  # aliases base
    strided = base[:, 1:, 0].t()                    # non-contiguous view
    ints = torch.arange(11, dtype=torch.int32)
    arr = np.arange(12, dtype=np.int64).reshape(3, 4)
    levels = [None,
              {"B": base, "root": (view, 3, 4.5, strided), "k": arr, "leaf": True,
               "ids": ints, "kmax": np.int64(9), "none": None},
              {"lst": [1, 2, "a"], "f": np.float64(0.25)}]
    kind, pb, out = _roundtrip(tmp_path, levels, {"n_side": 8, "eps": 1e-10})
    assert kind == "test" and pb == {"n_side": 8, "eps": 1e-10}
    assert out[0] is None
    L = out[1]
    assert torch.equal(L["B"], base)
    v, a, b, s = L["root"]
    assert torch.equal(v, view) and (a, b) == (3, 4.5) and torch.equal(s, strided)
    assert s.stride() == strided.stride()
    # aliasing is preserved: the view shares the loaded base's storage
    assert v.untyped_storage().data_ptr() == L["B"].untyped_storage().data_ptr()
    v.fill_(7.0)
    assert torch.all(L["B"][2] == 7.0)
    assert np.array_equal(L["k"], arr) and L["k"].dtype == np.int64
    assert torch.equal(L["ids"], ints) and L["leaf"] is True and L["none"] is None
    assert L["kmax"] == 9
    assert out[2] == {"lst": [1, 2, "a"], "f": 0.25}


def test_problem_header_is_plain_json(tmp_path):
    """The problem description is JSON (no pickle): spec, fields, quadrature,
    options and level slices round-trip through their own constructors."""
    import json
    from paper_1303_5466_b200 import CELL, KernelSpec, SolverOptions, make_field
    spec = KernelSpec("helmholtz2d", k=20.0, b_field=make_field("centre_bump", scale=-400.0,
                                                                 base=0.0, amp=1.0, width=0.09))
    pb = {"spec": spec, "quad": CELL, "opts": SolverOptions(eps=1e-8, leaf_size=64, k_cut=None),
          "eps": 1e-8, "n_side": 16, "n_max": 64, "level_slices": {2: (0, 2), 3: (0, 4)},
          "ti_mode": False}
    kind, back, _ = _roundtrip(tmp_path, [None], pb)
    assert back == pb
    path = str(tmp_path / "f.vief")
    hdr = persist.read_header(path)
    assert json.loads(json.dumps(hdr)) == hdr
    assert "pickle" not in open(persist.__file__).read().replace("no pickle", "")


def test_format_alignment_and_magic(tmp_path):
    path = str(tmp_path / "f.vief")
    persist.write_state(path, {}, "test", [{"a": torch.ones(3, dtype=torch.float64),
                                            "b": np.zeros(5, dtype=np.int32)}])
    h = persist.read_header(path)
    assert [s["offset"] % 4096 for s in h["storages"]] == [0, 0]
    assert [s["nbytes"] for s in h["storages"]] == [24, 20]
    with open(path, "r+b") as f:
        f.write(b"XXXXXXXX")
    with pytest.raises(ValueError):
        persist.read_header(path)


def test_format_rejects_unknown_types(tmp_path):
    with pytest.raises(TypeError):
        persist.write_state(str(tmp_path / "f"), {}, "test", [{"a": object()}])


# ---------------------------------------------------------------------------

def _problem(n_side, complex_=False):
    import paper_1303_5466_b200 as P
    if complex_:
        spec = P.KernelSpec("helmholtz2d", k=6.0, b_field=P.make_field("gaussian_bump"))
    else:
        spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"))
    grid = P.Grid(n_side)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    return spec, grid, opts


@pytest.mark.gpu
@pytest.mark.parametrize("complex_", [False, True])
def test_inverse_save_load_bitwise(tmp_path, complex_):
    from paper_1303_5466_b200 import solver_compressed as sc
    from paper_1303_5466_b200.solver_compressed import CompressedInverse
    spec, grid, opts = _problem(64 if not complex_ else 32, complex_)
    inv = sc.compress_inverse(spec, grid, eps=1e-10, opts=opts)
    rng = np.random.default_rng(3)
    f = rng.standard_normal((grid.n, 3))
    if complex_:
        f = f + 1j * rng.standard_normal((grid.n, 3))
    x0 = inv.apply(f)
    path = str(tmp_path / "inv.vief")
    inv.save(path)
    inv2 = CompressedInverse.load(path)
    assert isinstance(inv2, CompressedInverse)
    x1 = inv2.apply(f)
    assert x1.dtype == x0.dtype and np.array_equal(x0, x1)
    assert inv2.nbytes() == inv.nbytes()
    H0, H1 = inv.dense_matvec_source, inv2.dense_matvec_source
    for i in list(H0.row_skel)[:20]:
        assert np.array_equal(H0.row_skel[i], H1.row_skel[i])
    assert np.array_equal(H0.matvec(f), H1.matvec(f))
    assert np.array_equal(inv.apply(f[:, 0]), inv2.apply(f[:, 0]))


@pytest.mark.gpu
def test_dense_inverse_and_matrix_save_load(tmp_path):
    from paper_1303_5466_b200 import solver_dense as sd
    import paper_1303_5466_b200 as P
    spec, grid, opts = _problem(64)
    tree = P.build_tree(grid, 64)
    H = sd.compress_outer(spec, grid, tree, 1e-10, opts)
    pH = str(tmp_path / "H.vief")
    H.save(pH)
    inv = sd.invert_dense_block(H)
    pI = str(tmp_path / "inv.vief")
    inv.save(pI)
    H2 = sd.Hss2dMatrix.load(pH)
    inv2 = sd.DenseBlockInverse.load(pI)
    x = np.random.default_rng(0).standard_normal(grid.n)
    assert np.array_equal(H.matvec(x), H2.matvec(x))
    assert np.array_equal(inv.apply(x), inv2.apply(x))
    assert H2.nbytes() == H.nbytes()
    for i in list(inv.E)[:10]:
        assert np.array_equal(inv.E[i], inv2.E[i])
    assert np.array_equal(inv.Finv[0], inv2.Finv[0])


@pytest.mark.gpu
def test_lean_factors_save_load_bitwise(tmp_path):
    """The low-memory schedule's lean factor set (F^-1, E, T: what a 2048^2
    factorization holds) written and read back: bitwise the same solves."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200 import solver_compressed as sc
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(128)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=None, low_memory=True)
    inv = sc.compress_inverse(spec, grid, eps=1e-10, opts=opts)
    H = inv.dense_matvec_source
    assert all(getattr(L, "hss_kind", None) == "lean" for L in H.levels if L is not None and L.lv > 0)
    f = np.random.default_rng(5).standard_normal((grid.n, 3))
    x0 = inv.apply(f)
    path = str(tmp_path / "lean.vief")
    inv.save(path)
    inv2 = sc.CompressedInverse.load(path)
    assert np.array_equal(inv2.apply(f), x0)
    assert np.array_equal(inv2.apply(f[:, 0]), inv.apply(f[:, 0]))
    assert inv2.nbytes() == inv.nbytes()


@pytest.mark.gpu
def test_hss1d_factors_save_load_bitwise(tmp_path):
    """Finite k_cut with the large blocks in 1-D HSS form: the forms (tree
    intervals, generators per level, ranks) and the a-priori band width
    survive the file; solves and factor views are bitwise the same."""
    import paper_1303_5466_b200 as P
    from paper_1303_5466_b200 import compressed_store, solver_compressed as sc
    spec = P.KernelSpec("laplace2d", b_field=P.make_field("gaussian_bump"), c_field=P.make_field("one"))
    grid = P.Grid(64)
    opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=32)
    inv = sc.compress_inverse(spec, grid, eps=1e-10, opts=opts)
    assert compressed_store.compact(inv.factors, force_hss=True) >= 2
    f = np.random.default_rng(6).standard_normal((grid.n, 2))
    x0 = inv.apply(f)
    path = str(tmp_path / "hss.vief")
    inv.save(path)
    inv2 = sc.CompressedInverse.load(path)
    assert np.array_equal(inv2.apply(f), x0)
    assert inv2.nbytes() == inv.nbytes()
    b0, b1 = inv.factor_of(inv.tree.nodes[1]), inv2.factor_of(inv2.tree.nodes[1])
    assert b0.k == b1.k and np.array_equal(b0.E, b1.E) and np.array_equal(b0.Finv, b1.Finv)
