"""`compress_inverse` façade (solver_compressed.py:514-535 of the reference).

With opts.k_cut = None (or inf) the reference delegates outright to the
dense-block path; this package implements exactly that delegation on the
B200.  The finite-k_cut O(N) compressed-block solver (1-D HSS algebra,
solver_compressed.py:223-591 and hss1d/) is out of this build's scope
 and raises NotImplementedError.
"""

import numpy as np

from .config import SolverOptions
from .errors import ConfigError
from .kernels import PLAIN
from .solver_dense import compress_outer, factorize, invert_dense_block
from .tree import build_tree


class CompressedInverse:
    def __init__(self, spec, grid, tree, eps, opts, quad, ti_mode):
        self.spec, self.grid, self.tree = spec, grid, tree
        self.eps, self.opts, self.quad, self.ti_mode = eps, opts, quad, ti_mode
        self.dense_delegate = None
        self.dense_matvec_source = None

    def nbytes(self):
        return self.dense_delegate.nbytes()

    def apply(self, f):
        return self.dense_delegate.apply(f)

    def save(self, path):
        """Write the factors to `path` (persist.py): factor once, solve in
        later runs."""
        from . import persist
        persist.save(self, path)

    @staticmethod
    def load(path, device=None):
        from . import persist
        return persist.load(path, device)


def compress_inverse(spec, grid, tree=None, eps=1e-10, opts=None, quad=PLAIN, ti_mode=False,
                     support_mask=None):
    opts = opts or SolverOptions(eps=eps)
    if ti_mode and not spec.translation_invariant:
        raise ConfigError("ti_mode requires a translation-invariant kernel")
    if not (opts.k_cut is None or opts.k_cut == np.inf):
        raise NotImplementedError(
            "finite k_cut (O(N) compressed-block factors) is not part of the B200 build; "
            "use k_cut=None (dense-block path)")
    if tree is None:
        tree = build_tree(grid, opts.leaf_size)
    inv = CompressedInverse(spec, grid, tree, eps, opts, quad, ti_mode)
    # compress_outer + invert_dense_block, levels pipelined over two streams
    H, inv.dense_delegate = factorize(spec, grid, tree, eps, opts, quad)
    inv.dense_matvec_source = H
    return inv


def apply_inverse_compressed(inv, f):
    return inv.apply(f)
