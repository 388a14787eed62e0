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
form (eps-accurate, O(N) memory); here the blocks are formed dense on the
device and, with SolverOptions(block_storage="hss1d"), compressed level by
level into batched 1-D HSS forms for storage and the solve sweeps
(compressed_store.py, hss1d.py); the default keeps them dense in HBM (fastest
solve).  ti_mode (translation-invariant kernels) keeps one factor
record per level after the factorization (share_level_records: the sweeps read
it with batch stride 0), as the reference's TI mode does; every box is still
factored.  Complex kernels run realified like the
dense-block path (the realified least-squares fit is the realified complex one).
"""

import numpy as np

from .config import SolverOptions
from .errors import ConfigError
from .kernels import PLAIN
from .solver_dense import compress_outer, factorize, invert_dense_block, share_level_records
from .tree import annotate_skeletons, build_tree


class BoxFactors:
    """Host view of one non-root box's factors on the finite-k_cut path, in the
    reference's [sk, rs] ordering (BoxFactors, solver_compressed.py:73-140).
    Every box here is of the dense kinds ("leaf" / "dense"): T_up, T_dn, E
    and F^-1 are plain arrays copied from HBM on access.  Real kernels."""

    def __init__(self, inv, box):
        if inv.spec.is_complex:
            raise NotImplementedError("factor views are built for real kernels")
        H, D = inv.dense_matvec_source, inv.dense_delegate
        i = box.idx
        self.kind = "leaf" if box.is_leaf else "dense"
        self.k, self.r = int(box.sk_idx.size), int(box.rs_idx.size)
        self.k1 = None if box.is_leaf else int(inv.tree.nodes[box.children[0]].sk_idx.size)
        wp = box.work_perm
        self.perm = None if box.is_leaf else wp
        self.iperm = None
        if not box.is_leaf:
            self.iperm = np.empty_like(wp)
            self.iperm[wp] = np.arange(wp.size)
        self.T_up = H.Rfac[i].T
        self.T_dn = H.Lfac[i].T
        self.E = D.E[i]
        self.Finv = D.Finv[i][np.ix_(wp, wp)]

    def nbytes(self):
        return self.T_up.nbytes + self.T_dn.nbytes + self.E.nbytes + self.Finv.nbytes

    def apply_finv(self, u):
        """sigma = F^-1 u on the box ordering [sk, rs]."""
        return self.Finv @ u

    def apply_R(self, phi):
        return phi[:self.k] + self.T_up @ phi[self.k:]

    def apply_L(self, w):
        return np.vstack([w, self.T_dn.T @ w])

    def apply_E(self, x):
        return self.E @ x


class CompressedInverse:
    def __init__(self, spec, grid, tree, eps, opts, quad, ti_mode):
        self.spec, self.grid, self.tree = spec, grid, tree
        self.eps, self.opts, self.quad, self.ti_mode = eps, opts, quad, ti_mode
        self.dense_delegate = None
        self.dense_matvec_source = None

    def nbytes(self):
        return self.dense_delegate.nbytes()

    def factor_of(self, box):
        """Factors of a non-root box (finite k_cut; solver_compressed.py:166-167)."""
        if self.dense_delegate is None or not hasattr(self.tree.nodes[0], "sk_idx") \
                or self.tree.nodes[0].sk_idx is None or box.idx == 0:
            raise KeyError(box.idx)
        return BoxFactors(self, box)

    def record_count(self):
        """Factor records: one per non-root box plus the top, or one per level
        in TI mode (solver_compressed.py:169-171)."""
        if self.ti_mode and self.dense_delegate is not None and self.tree.nodes[0].sk_idx is not None:
            return self.tree.depth + 1
        return len(self.tree.nodes)

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


def ensure_apriori_skeletons(spec, tree, opts, support_mask=None):
    """Annotate `tree` with the compressed path's a-priori skeletons exactly as
    the reference's compress_inverse does (solver_compressed.py:536-542): the
    boundary band of `resolved_layers`, plus the oscillatory interior
    retention for Helmholtz above the kappa threshold, restricted to an
    optional support mask.  Every caller that factors on the finite-k_cut path
    (compress_inverse, distributed.ShardedInverse) goes through here, so all of
    them choose the same skeletons.  Returns the layer width."""
    layers = opts.resolved_layers(spec)
    if tree.nodes[0].sk_idx is None:
        kw = {}
        if opts.keep_interface_interior(spec):
            kw = dict(k_wave=spec.k, points_per_wavelength=opts.points_per_wavelength)
        annotate_skeletons(tree, layers, support_mask=support_mask, **kw)
    return layers


def _levels_uniform(tree):
    """Every level's boxes have one width and height (all translates)."""
    for r in tree.rects:
        r = np.asarray(r)
        wh = np.stack([r[:, 1] - r[:, 0], r[:, 3] - r[:, 2]], 1)
        if not (wh == wh[0]).all():
            return False
    return True


def compress_inverse(spec, grid, tree=None, eps=1e-10, opts=None, quad=PLAIN, ti_mode=False,
                     support_mask=None):
    opts = opts or SolverOptions(eps=eps)
    if ti_mode and not spec.translation_invariant:
        raise ConfigError("ti_mode requires a translation-invariant kernel")
    if tree is None:
        tree = build_tree(grid, opts.leaf_size)
    inv = CompressedInverse(spec, grid, tree, eps, opts, quad, ti_mode)
    if opts.block_storage not in ("dense", "hss1d"):
        raise ConfigError(f"unknown block_storage {opts.block_storage!r}")
    if opts.low_memory:
        return _compress_inverse_low_memory(inv, spec, grid, tree, eps, opts, quad, ti_mode,
                                            support_mask)
    if opts.k_cut is None or opts.k_cut == np.inf:
        # compress_outer + invert_dense_block, levels pipelined over two streams
        H, inv.dense_delegate = factorize(spec, grid, tree, eps, opts, quad)
        inv.dense_matvec_source = H
        return inv
    layers = ensure_apriori_skeletons(spec, tree, opts, support_mask)
    # TI mode factors the first box of every level only (solver_compressed.py:
    # 548-552) when every box is a translate of it: uniform levels, no support
    # mask; otherwise every box is factored and uniform levels share a record
    share = ti_mode and support_mask is None and _levels_uniform(tree)
    H, inv.factors = factorize(spec, grid, tree, eps, opts, quad, apriori=layers, ti=share)
    if ti_mode and not share:
        share_level_records(inv.factors)
    if opts.block_storage == "hss1d":
        # boxes above k_cut keep F^-1 and E in 1-D HSS form (solver_compressed.py:
        # 490-511 _compressed_factors); TI records and refined levels stay dense
        from . import compressed_store
        inv.hss_levels = compressed_store.compact(inv.factors)
    inv.dense_delegate = inv.factors
    inv.dense_matvec_source = H
    return inv


def _compress_inverse_low_memory(inv, spec, grid, tree, eps, opts, quad, ti_mode, support_mask):
    """SolverOptions(low_memory=True): level-by-level compression and inversion
    with one level's sources resident at a time (invert_dense_block(compress=
    True, free_source=True)), lean or 1-D HSS factor storage.  2048^2 at eps =
    1e-10 fits one B200 this way (profiles/r02_c5_2048_single_gpu*.json)."""
    from . import solver_dense as sd
    if ti_mode:
        raise ConfigError("low_memory does not combine with ti_mode (TI records are small already)")
    H = sd.Hss2dMatrix(spec, grid, tree, eps, opts, quad)
    dense_path = opts.k_cut is None or opts.k_cut == np.inf
    if not dense_path:
        H.apriori = ensure_apriori_skeletons(spec, tree, opts, support_mask)
    storage = "hss1d" if (opts.block_storage == "hss1d" and not dense_path) else "lean"
    factors = invert_dense_block(H, free_source=True, storage=storage, compress=True)
    if not dense_path:
        inv.factors = factors
        inv.hss_levels = sum(getattr(L, "hss_kind", None) == "hss" for L in H.levels if L is not None)
    inv.dense_delegate = factors
    inv.dense_matvec_source = H
    return inv


def apply_inverse_compressed(inv, f):
    return inv.apply(f)
