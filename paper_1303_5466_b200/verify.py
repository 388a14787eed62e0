"""Exact forward operator by FFT: the independent
residual check the reference lacks at scale.

On the uniform cell-centred lattice the off-diagonal entries depend only on
the lattice offset, so (kernels.py:258-275, restated)

    (A x)_i = a_i x_i + h^2 b_i corr c_i x_i + h^2 b_i sum_{j != i} K(|x_i - x_j|) c_j x_j

and the sum is a 2-D Toeplitz (BTTB) convolution.  It is evaluated by a
zero-padded (2n)^2 FFT in O(N log N) -- at N = 1024^2 one matvec is a few
milliseconds on the GPU, against a dense A of 8 TB.  The kernel values are
the reference's own expression on q = dx^2 + dy^2 (kernel_eval, the same
table the entry kernels read), so the operator is A up to FFT rounding
(~1e-15 relative).

This is a verification tool (bench residuals, tests); the factor/solve path
does not use it.  Runs on any torch device.
"""

import numpy as np
import torch

from .kernels import PLAIN, kernel_eval

__all__ = ["FFTOperator", "true_residual"]


class FFTOperator:
    """A as a matvec for (spec, grid, quad); x in global grid order
    (linear index iy*n + ix), shape (N,) or (N, r), numpy or torch."""

    def __init__(self, spec, grid, quad=PLAIN, device=None):
        self.spec, self.grid, self.quad = spec, grid, quad
        self.device = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
        n = grid.n_side
        self.n = n
        h = grid.h
        cdt = torch.complex128
        d = np.arange(2 * n)
        d = np.where(d < n, d, d - 2 * n)            # circular offsets -(n-1)..(n-1), row n unused
        q = d[:, None] ** 2 + d[None, :] ** 2
        kern = np.zeros((2 * n, 2 * n), dtype=np.complex128)
        nz = q > 0
        kern[nz] = kernel_eval(spec, h * np.sqrt(q[nz].astype(np.float64)))
        kern[n, :] = 0.0                              # offsets of magnitude n never occur
        kern[:, n] = 0.0
        self.khat = torch.fft.fft2(torch.from_numpy(kern).to(self.device, cdt))
        xy = grid.points()
        a = np.asarray(spec.a_field(xy), dtype=np.float64)
        b = np.asarray(spec.b_field(xy), dtype=np.float64)
        c = np.asarray(spec.c_field(xy), dtype=np.float64)
        corr = complex(quad.diagonal_term(spec, h))
        hh = h * h
        self.bh = torch.from_numpy(b * hh).to(self.device)
        self.c = torch.from_numpy(c).to(self.device)
        self.diag = torch.from_numpy(a + hh * b * c * corr).to(self.device, cdt)
        self.complex = spec.is_complex or corr.imag != 0.0

    def matvec(self, x):
        """A x (same container type and shape as x; complex only for complex specs)."""
        is_np = isinstance(x, np.ndarray)
        xt = torch.as_tensor(x, device=self.device)
        single = xt.dim() == 1
        X = xt.reshape(-1, 1) if single else xt
        n = self.n
        r = X.shape[1]
        Xc = X.to(torch.complex128)
        v = (self.c[:, None] * Xc).t().reshape(r, n, n)       # [rhs, iy, ix]
        pad = torch.zeros((r, 2 * n, 2 * n), dtype=torch.complex128, device=self.device)
        pad[:, :n, :n] = v
        conv = torch.fft.ifft2(torch.fft.fft2(pad) * self.khat)[:, :n, :n]
        Y = self.bh[:, None] * conv.reshape(r, n * n).t() + self.diag[:, None] * Xc
        if not (self.complex or torch.is_complex(X)):
            Y = Y.real
        Y = Y.reshape(-1) if single else Y
        return Y.cpu().numpy() if is_np else Y


def true_residual(spec, grid, quad, f, x, op=None):
    """||f - A x|| / ||f|| with the exact FFT operator (per column for 2-D f)."""
    op = op or FFTOperator(spec, grid, quad)
    ft = torch.as_tensor(f, device=op.device)
    ax = op.matvec(torch.as_tensor(x, device=op.device))
    res = (ft.to(ax.dtype) - ax)
    if res.dim() == 1:
        return float(torch.linalg.vector_norm(res) / torch.linalg.vector_norm(ft))
    return (torch.linalg.vector_norm(res, dim=0) / torch.linalg.vector_norm(ft, dim=0)).cpu().numpy()
