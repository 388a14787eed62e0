"""Golden fixture for the scattering driver, made by running the REFERENCE
(build container only; needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_scattering.py

Writes tests/golden/scattering.npz: the Lippmann-Schwinger right-hand side,
the refined direct solution (mode="dense"), its residual and the outgoing
field at three targets, for ScatteringProblem(kappa=2, n_side=28, H4).
"""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from vief.scattering import ScatteringProblem, setup_ls, solve_direct  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TARGETS = np.array([[2.0, 0.0], [-1.5, 1.7], [0.3, -2.5]])

if __name__ == "__main__":
    prob = ScatteringProblem(kappa=2.0, n_side=28)
    spec, rhs = setup_ls(prob)
    tau, info = solve_direct(prob, eps=1e-10, refine=True, mode="dense", n_probe_rhs=0)
    np.savez_compressed(os.path.join(OUT, "scattering.npz"), rhs=rhs, tau=tau,
                        residual=info["residual"], targets=TARGETS, u_out=info["u_out"](TARGETS))
    print("residual", info["residual"], "|tau|", np.linalg.norm(tau))
