"""Scattering driver (scattering.py) against the reference's own outputs
(tests/golden/scattering.npz, made by make_golden_scattering.py).  The
set-up and the outgoing field are host code (CPU tests); the direct solve
runs the B200 factor/solve path (gpu)."""
import os

import numpy as np
import pytest

from paper_1303_5466_b200 import ConfigError
from paper_1303_5466_b200.scattering import ScatteringProblem, outgoing_field, setup_ls

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "scattering.npz"))


def test_setup_ls_matches_reference():
    spec, rhs = setup_ls(ScatteringProblem(kappa=2.0, n_side=28))
    assert spec.family == "helmholtz2d" and spec.symmetric
    np.testing.assert_array_equal(rhs, G["rhs"])


def test_outgoing_field_matches_reference():
    prob = ScatteringProblem(kappa=2.0, n_side=28)
    u = outgoing_field(prob, G["tau"], G["targets"])
    np.testing.assert_allclose(u, G["u_out"], rtol=1e-13, atol=0)
    assert outgoing_field(prob, G["tau"], G["targets"][0]).shape == (1,)


def test_problem_errors():
    with pytest.raises(ConfigError):
        ScatteringProblem(kappa=2.0, n_side=28, source=(0.5, 0.0))
    with pytest.raises(ConfigError):
        ScatteringProblem(kappa=0.0, n_side=28)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["dense", "compressed"])
def test_solve_direct_matches_reference(mode):
    from paper_1303_5466_b200.scattering import solve_direct
    eps = 1e-10
    prob = ScatteringProblem(kappa=2.0, n_side=28)
    tau, info = solve_direct(prob, eps=eps, refine=True, mode=mode, n_probe_rhs=2)
    ref = G["tau"]
    # the refinement converges to the inverse of each build's own compressed
    # operator; the two operators differ by ~eps, so the solutions differ by
    # ~cond(A) eps (cond ~ 20 for this k^2 = 158 contrast): 100 eps here, while
    # the residual against the exact A (FFT) is held to 10 eps
    assert np.linalg.norm(tau - ref) / np.linalg.norm(ref) <= 100 * eps
    assert info["residual"] <= 10 * eps and info["true_residual"] <= 10 * eps
    # compressed mode = a-priori skeletons (finite k_cut): the unrefined inverse
    # is a preconditioner-grade solve here (the reference's own compressed mode
    # gives E = 8e-3 on this problem, residual 2e-4 after refinement; ours ~1e-7)
    assert info["approx_residual"] <= (10 * eps if mode == "dense" else 1e-6)
    u = info["u_out"](G["targets"])
    assert np.linalg.norm(u - G["u_out"]) <= 100 * eps * np.linalg.norm(G["u_out"])
