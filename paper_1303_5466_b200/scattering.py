"""Volume-scattering driver on the B200 factor/solve path:
the Lippmann-Schwinger system set-up, the direct solve with one residual
correction, the outgoing field and the approximate-residual probe of the
reference's scattering.py, with the same names, arguments and return
conventions.  (The preconditioned iterative solve and the convergence study
are not part of this build.)

Differences, all confined to what this build covers:
  * mode="compressed" (the reference default, k_cut = 64) runs the
    compressed path's a-priori skeletons with the scatterer support mask
    (solver_compressed.compress_inverse, dense blocks) and refines against
    the ID-compressed operator H, as the reference does; k_cut=None runs the
    dense-block inverse of H itself.
  * info additionally carries "true_residual": ||rhs - A tau|| / ||rhs|| with
    A applied exactly by FFT (verify.py), not just the compressed matvec.
Reference: scattering.py:22-128 (problem, setup_ls, outgoing_field,
solve_direct), :154-163 (approx_residual).
"""

from dataclasses import dataclass, replace

import numpy as np

from .config import SolverOptions
from .errors import ConfigError
from .kernels import H4, Grid, KernelSpec, kernel_eval, make_field
from .solver_compressed import compress_inverse
from .solver_dense import compress_outer, invert_dense_block
from .tree import build_tree

__all__ = ["ScatteringProblem", "setup_ls", "outgoing_field", "solve_direct", "approx_residual"]


@dataclass(frozen=True)
class ScatteringProblem:
    """scattering.py:22-63: wave-speed deviation b >= 0 (product-tanh profile
    scaled by k^2), point source outside [-1,1]^2."""
    kappa: float
    n_side: int
    d: float = 15.0
    eps_edge: float = 0.3
    source: tuple = (2.0, 2.0)
    quad: object = H4

    def __post_init__(self):
        if max(abs(self.source[0]), abs(self.source[1])) <= 1.0:
            raise ConfigError("source must lie outside the domain")
        if self.kappa <= 0:
            raise ConfigError("kappa must be positive")

    @property
    def k(self):
        return 2.0 * np.pi * self.kappa

    @property
    def grid(self):
        return Grid(self.n_side)

    def b_values(self, xy):
        return make_field("tanh_box", d=self.d, eps_edge=self.eps_edge, scale=self.k ** 2)(xy)

    def sqrt_b_field(self):
        return make_field("tanh_box_sqrt", d=self.d, eps_edge=self.eps_edge, scale=self.k ** 2)

    def free_kernel(self):
        return KernelSpec("helmholtz2d", k=self.k)

    def incoming(self, xy):
        r = np.hypot(xy[..., 0] - self.source[0], xy[..., 1] - self.source[1])
        return kernel_eval(self.free_kernel(), r)


def setup_ls(problem):
    """(KernelSpec, rhs) of the symmetrised second-kind system: sqrt(b) row
    and column weights, rhs = -sqrt(b) u_in (scattering.py:66-76)."""
    grid = problem.grid
    xy = grid.points()
    b = problem.b_values(xy)
    if np.any(b < 0):
        raise ConfigError("deviation field must be nonnegative")
    w = problem.sqrt_b_field()
    spec = KernelSpec("helmholtz2d", k=problem.k, b_field=w, c_field=w)
    return spec, -np.sqrt(b) * problem.incoming(xy)


def outgoing_field(problem, tau, targets, chunk=1 << 22):
    """u_out(t) = h^2 sum_j K(|t - x_j|) sqrt(b_j) tau_j (scattering.py:79-89),
    evaluated for all targets at once in blocks of `chunk` kernel values."""
    grid = problem.grid
    xy = grid.points()
    dens = (grid.h ** 2) * np.sqrt(problem.b_values(xy)) * np.asarray(tau)
    tg = np.atleast_2d(np.asarray(targets, dtype=float))
    spec = problem.free_kernel()
    per = max(1, chunk // max(1, grid.n))
    parts = []
    for t0 in range(0, tg.shape[0], per):
        t = tg[t0:t0 + per]
        r = np.hypot(t[:, None, 0] - xy[None, :, 0], t[:, None, 1] - xy[None, :, 1])
        parts.append(kernel_eval(spec, r) @ dens)
    return np.concatenate(parts).astype(np.complex128) if parts else np.zeros(0, np.complex128)


def _support_mask(spec, grid):
    """Points with nonzero contrast; None when the support is everything
    (scattering.py:87-89)."""
    vals = np.abs(spec.b_field(grid.points()))
    return vals > 0.0 if np.any(vals == 0.0) else None


def approx_residual(H, inv, grid, n_rhs=3, rng=None):
    """max over random v of ||v - H inv(v)|| / ||v|| (scattering.py:154-163)."""
    rng = rng or np.random.default_rng(0)
    worst = 0.0
    for _ in range(n_rhs):
        v = rng.standard_normal(grid.n)
        x = inv.apply(v)
        worst = max(worst, float(np.linalg.norm(v - H.matvec(x)) / np.linalg.norm(v)))
    return worst


def solve_direct(problem, eps=1e-10, refine=True, mode="compressed", opts=None,
                 n_probe_rhs=3, rng=None):
    """Direct solve of the scattering system (scattering.py:98-128).

    Returns (tau, info): info holds the compressed operator ("matrix"), the
    inverse, the compressed-operator residual, the exact (FFT) residual, a
    callable u_out(targets) and, with n_probe_rhs, the approximate residual E.
    With `refine`, one residual correction tau += inv(rhs - H tau)."""
    from .verify import FFTOperator
    spec, rhs = setup_ls(problem)
    grid = problem.grid
    opts = opts or SolverOptions(eps=eps)
    info = {}
    if np.linalg.norm(rhs) == 0.0:
        tau = np.zeros(grid.n, dtype=np.complex128)
        info.update(residual=0.0, true_residual=0.0,
                    u_out=lambda t: np.zeros(len(np.atleast_2d(t)), dtype=np.complex128))
        return tau, info
    tree = build_tree(grid, opts.leaf_size)
    finite = not (opts.k_cut is None or opts.k_cut == np.inf)
    if mode == "dense":
        H = compress_outer(spec, grid, tree, eps, opts, quad=problem.quad)
        inv = invert_dense_block(H)
    elif finite:
        H = compress_outer(spec, grid, tree, eps, opts, quad=problem.quad)
        inv = compress_inverse(spec, grid, tree=build_tree(grid, opts.leaf_size), eps=eps,
                               opts=opts, quad=problem.quad,
                               support_mask=_support_mask(spec, grid))
    else:
        inv = compress_inverse(spec, grid, tree=tree, eps=eps, opts=opts, quad=problem.quad)
        H = inv.dense_matvec_source
    tau = inv.apply(rhs)
    if refine:
        tau = tau + inv.apply(rhs - H.matvec(tau))
    resid = np.linalg.norm(rhs - H.matvec(tau)) / np.linalg.norm(rhs)
    op = FFTOperator(spec, grid, problem.quad)
    true = np.linalg.norm(rhs - op.matvec(tau)) / np.linalg.norm(rhs)
    info.update(matrix=H, inverse=inv, residual=float(resid), true_residual=float(true),
                u_out=lambda targets: outgoing_field(problem, tau, targets))
    if n_probe_rhs:
        info["approx_residual"] = approx_residual(H, inv, grid, n_rhs=n_probe_rhs, rng=rng)
    return tau, info
