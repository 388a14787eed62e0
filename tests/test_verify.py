"""The exact FFT forward operator (verify.FFTOperator) against the oracle's
dense A on the same problems: every kernel family, every diagonal rule,
non-constant a/b/c fields, 1-D and 2-D inputs.  CPU (torch.fft), no GPU."""
import numpy as np
import pytest

import oracle.hssd as O
from paper_1303_5466_b200 import CELL, H4, PLAIN, Grid, KernelSpec, make_field
from paper_1303_5466_b200.verify import FFTOperator, true_residual

QUADS = {"none": PLAIN, "h4": H4, "cell": CELL}

CASES = [
    # (n, family, k, a, b, c, quad)
    (12, "laplace2d", 0.0, ("one", ()), ("gaussian_bump", ()), ("one", ()), "none"),
    (16, "laplace2d", 0.0, ("one", ()), ("centre_bump", (("scale", np.pi / 2),)), ("one", ()), "cell"),
    (15, "laplace2d", 0.0, ("tanh_box", (("d", 0.5), ("eps_edge", 0.1))), ("one", ()),
     ("gaussian_bump", ()), "h4"),
    (14, "yukawa2d", 3.0, ("one", ()), ("one", ()), ("one", ()), "h4"),
    (13, "helmholtz2d", 10.0, ("one", ()), ("gaussian_bump", ()), ("one", ()), "none"),
    (16, "helmholtz2d", 20.0, ("one", ()), ("one", ()), ("one", ()), "h4"),
    (11, "laplace3d_sl", 0.0, ("one", ()), ("one", ()), ("one", ()), "none"),
]


def _spec(family, k, a, b, c):
    return KernelSpec(family, k=k, a_field=make_field(a[0], **dict(a[1])),
                      b_field=make_field(b[0], **dict(b[1])), c_field=make_field(c[0], **dict(c[1])))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[1]}-{c[0]}-{c[6]}")
def test_fft_operator_matches_dense(case):
    n, family, k, a, b, c, quad = case
    P = O.Problem(n, family, k, a, b, c, quad)
    A = O.dense_matrix(P)
    op = FFTOperator(_spec(family, k, a, b, c), Grid(n), QUADS[quad], device="cpu")
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n * n)
    y = op.matvec(x)
    ref = A @ x
    assert y.shape == ref.shape and y.dtype == ref.dtype
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    X = rng.standard_normal((n * n, 3))
    Y = op.matvec(X)
    assert np.linalg.norm(Y - A @ X) <= 1e-13 * np.linalg.norm(A @ X)


def test_true_residual_of_dense_solve():
    n = 14
    P = O.Problem(n, "laplace2d", 0.0, ("one", ()), ("gaussian_bump", ()), ("one", ()), "none")
    A = O.dense_matrix(P)
    f = np.random.default_rng(0).standard_normal(n * n)
    x = np.linalg.solve(A, f)
    spec = _spec("laplace2d", 0.0, ("one", ()), ("gaussian_bump", ()), ("one", ()))
    assert true_residual(spec, Grid(n), PLAIN, f, x, FFTOperator(spec, Grid(n), PLAIN, "cpu")) < 1e-13
    r = true_residual(spec, Grid(n), PLAIN, f, x + 1e-3, FFTOperator(spec, Grid(n), PLAIN, "cpu"))
    assert r > 1e-6
