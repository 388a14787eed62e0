"""`compress_inverse` façade (solver_compressed.py:514-591 of the reference).

k_cut = None (or inf): the reference delegates outright to the dense-block
path; this package runs exactly that delegation on the B200 (ID skeletons,
pipelined factorization).

Finite k_cut: the compressed path's a-priori skeletons.  Every box keeps the
boundary band of width `layers` of its candidates (tree.annotate_skeletons,
tree.py:237-269), the interpolation is the least-squares fit against the
proxy rings (solver_compressed.py:223-266, batched fixed-rank QR on the
device) and the factors are F^-1 and E = ([I T_up] F^-1 [I; T_dn^T])^-1 per
box (_dense_factors / _dense_E_from_lu, solver_compressed.py:437-483), the
root F = cross + diag(E1, E2) (solver_compressed.py:560-577).  The reference
stores the blocks of boxes with more than k_cut skeleton points in 1-D HSS
form (eps-accurate, O(N) memory); here every block stays dense in HBM, so
results agree with the reference to its eps while the storage is the
dense-block one.  ti_mode is validated like the reference's but factors every
box (no per-level record sharing).  Complex kernels run realified like the
dense-block path (the realified least-squares fit is the realified complex one).
"""

import numpy as np

from .config import SolverOptions
from .errors import ConfigError
from .kernels import PLAIN
from .solver_dense import compress_outer, factorize, invert_dense_block
from .tree import annotate_skeletons, build_tree


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
    if tree is None:
        tree = build_tree(grid, opts.leaf_size)
    inv = CompressedInverse(spec, grid, tree, eps, opts, quad, ti_mode)
    if opts.k_cut is None or opts.k_cut == np.inf:
        # compress_outer + invert_dense_block, levels pipelined over two streams
        H, inv.dense_delegate = factorize(spec, grid, tree, eps, opts, quad)
        inv.dense_matvec_source = H
        return inv
    layers = opts.resolved_layers(spec)
    if tree.nodes[0].sk_idx is None:
        kw = {}
        if opts.keep_interface_interior(spec):
            kw = dict(k_wave=spec.k, points_per_wavelength=opts.points_per_wavelength)
        annotate_skeletons(tree, layers, support_mask=support_mask, **kw)
    H, inv.factors = factorize(spec, grid, tree, eps, opts, quad, apriori=layers)
    inv.dense_delegate = inv.factors
    inv.dense_matvec_source = H
    return inv


def apply_inverse_compressed(inv, f):
    return inv.apply(f)
