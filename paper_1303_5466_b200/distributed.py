"""Subtree-sharded factor / solve across GPUs.

Boxes of one level depend only on their children, so with P = 2^s ranks the
tree splits at level s: rank g factors the subtree rooted at the g-th box of
level s (levels s..depth) with no communication; rank 0 then factors the top
levels 0..s-1 from the subtree roots' interface data — skeleton index lists
and the k x k reduced operators E — gathered over NCCL.  The solve runs the up
sweep locally, gathers the subtree roots' `ups` to rank 0, runs the top of the
tree there, broadcasts the phi_dn slices back and finishes the down sweep
locally.  Every rank holds only its subtree's factors (the 2048^2 case needs
~200 GB in total).

The algorithm is written as explicit phases so that the same code runs
  * over torch.distributed (one process per GPU, NCCL; gloo for CPU tests), or
  * emulated in one process on one GPU (`emulate=True`), which is how it is
    exercised on a single B200 (no rank ever waits on a kernel of another).
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import solver_dense as sd

_F64, _I32 = torch.float64, torch.int32


# ---------------------------------------------------------------------------
# host planning (pure integers; unit-tested with gloo on CPU)

@dataclass
class SplitPlan:
    world: int
    split: int                 # level s = log2(world)
    slices: list              # per rank: {level: (lo, hi)} of that level's box list
    top: dict = field(default_factory=dict)  # rank 0: {level: (lo, hi)} for levels < s


def subtree_plan(tree, world):
    """Rank g owns boxes [g 2^(l-s), (g+1) 2^(l-s)) of every level l >= s."""
    if world < 1 or world & (world - 1):
        raise ValueError("world size must be a power of two")
    s = world.bit_length() - 1
    if s > tree.depth:
        raise ValueError(f"tree depth {tree.depth} too shallow for {world} ranks")
    slices = []
    for g in range(world):
        d = {}
        for lv in range(s, tree.depth + 1):
            width = len(tree.ids[lv]) >> s
            d[lv] = (g * width, (g + 1) * width)
        slices.append(d)
    top = {lv: (0, len(tree.ids[lv])) for lv in range(s)}
    return SplitPlan(world, s, slices, top)


def owned_points(tree, plan, rank):
    """Grid points owned by a rank (its subtree's leaves)."""
    lo, hi = plan.slices[rank][tree.depth]
    own = tree.owned_level(tree.depth)[lo:hi]
    return np.sort(own[own >= 0].ravel())


# ---------------------------------------------------------------------------
# communication

class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def gather0(self, t):
        """Tensors of any shape (same dtype/ndim) -> list on rank 0, None elsewhere."""
        dist = self.dist
        shape = torch.tensor(list(t.shape), dtype=torch.int64, device=t.device)
        shapes = [torch.zeros_like(shape) for _ in range(self.world)]
        dist.all_gather(shapes, shape)
        mx = torch.stack(shapes).max(dim=0).values.tolist()
        pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
        pad[tuple(slice(0, s) for s in t.shape)] = t
        bufs = [torch.zeros_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad)
        if self.rank != 0:
            return None
        return [b[tuple(slice(0, int(s)) for s in sh.tolist())] for b, sh in zip(bufs, shapes)]

    def bcast0(self, t, shape=None, dtype=None, device=None):
        dist = self.dist
        if self.rank != 0:
            t = torch.empty(shape, dtype=dtype, device=device)
        else:
            t = t.contiguous()  # collectives move raw storage
        dist.broadcast(t, src=0)
        return t

    def bcast_shape0(self, shape, device):
        v = torch.tensor(list(shape) if shape is not None else [0, 0], dtype=torch.int64,
                         device=device)
        self.dist.broadcast(v, src=0)
        return tuple(v.tolist())

    def allreduce_sum(self, t):
        t = t.contiguous()
        self.dist.all_reduce(t)
        return t


# ---------------------------------------------------------------------------
# device phases

def _interface_payload(Hl, invl, split):
    """The subtree root's data the top levels need: k, row/col skeletons, E."""
    L = Hl.levels[split]
    k = int(L.k[0])
    rs = L.rskel[0, :k].to(torch.int64)
    cs = L.cskel[0, :k].to(torch.int64)
    E = L.E[0, :k, :k].contiguous()        # storage [col, row]
    return k, rs, cs, E


def _virtual_level(Ht, split, ks, rskels, cskels, Es, dev):
    """Populate level `split` of the top object with the gathered interface."""
    V = Ht.levels[split]
    V.virtual = True
    V.k = np.asarray(ks, dtype=np.int32)
    V.kmax = max(int(V.k.max()), 1)
    V.k_d = sd._dev_i32(V.k, dev)
    P = len(ks)
    V.rskel = torch.zeros((P, V.kmax), dtype=_I32, device=dev)
    V.cskel = torch.zeros((P, V.kmax), dtype=_I32, device=dev)
    V.E = torch.zeros((P, V.kmax, V.kmax), dtype=_F64, device=dev)
    for g in range(P):
        k = int(ks[g])
        V.rskel[g, :k] = rskels[g].to(dev, _I32)
        V.cskel[g, :k] = cskels[g].to(dev, _I32)
        V.E[g, :k, :k] = Es[g].to(dev)
    return V


class ShardedInverse:
    """Subtree-sharded HSS-D factorization.  Construct with a communicator
    (TorchComm) for one-process-per-GPU runs, or with `emulate=True` to run
    all shards in this process (single-GPU validation of the sharded path)."""

    def __init__(self, spec, grid, tree, eps, opts, quad, world, comm=None, emulate=False,
                 support_mask=None):
        self.spec, self.grid, self.tree, self.eps, self.opts, self.quad = spec, grid, tree, eps, opts, quad
        self.plan = subtree_plan(tree, world)
        self.comm = comm
        self.emulate = emulate
        self.ranks = list(range(world)) if emulate else [comm.rank]
        self.local = {}
        # finite k_cut: the compressed path's a-priori skeletons (host annotation
        # is deterministic, so every rank derives the same splits)
        apriori = None
        if not (opts.k_cut is None or opts.k_cut == np.inf):
            from .solver_compressed import ensure_apriori_skeletons
            apriori = ensure_apriori_skeletons(spec, tree, opts, support_mask)
        s = self.plan.split
        payloads = {}
        for g in self.ranks:
            Hl = sd.Hss2dMatrix(spec, grid, tree, eps, opts, quad, level_slices=self.plan.slices[g])
            Hl.apriori = apriori
            sd.compress_levels(Hl)
            invl = sd.invert_dense_block(Hl)
            self.local[g] = (Hl, invl)
            if world > 1:
                payloads[g] = _interface_payload(Hl, invl, s)
        self.dev = next(iter(self.local.values()))[0].device
        self.realified = next(iter(self.local.values()))[0].realified
        self.top = None
        if world == 1:
            return
        if emulate:
            ks = [payloads[g][0] for g in range(world)]
            rsk = [payloads[g][1] for g in range(world)]
            csk = [payloads[g][2] for g in range(world)]
            Es = [payloads[g][3] for g in range(world)]
        else:
            k, rs, cs, E = payloads[comm.rank]
            ks_t = comm.gather0(torch.tensor([k], dtype=torch.int64, device=self.dev))
            rsk = comm.gather0(rs)
            csk = comm.gather0(cs)
            Es = comm.gather0(E)
            ks = [int(x.item()) for x in ks_t] if ks_t is not None else None
        if self.emulate or comm.rank == 0:
            top_slices = dict(self.plan.top)
            top_slices[s] = (0, world)
            Ht = sd.Hss2dMatrix(spec, grid, tree, eps, opts, quad, level_slices=top_slices)
            _virtual_level(Ht, s, ks, rsk, csk, Es, self.dev)
            Ht.apriori = apriori
            sd.compress_levels(Ht)
            self.top = (Ht, sd.invert_dense_block(Ht))

    # -- solve ----------------------------------------------------------------
    def apply_device(self, fd):
        """fd: (r, N') right-hand sides (every rank passes the full vector);
        returns the full (r, N') solution on every rank."""
        r = fd.shape[0]
        s = self.plan.split
        world = self.plan.world
        st = {}
        for g in self.ranks:
            Hl, _ = self.local[g]
            phi, ups = {}, {}
            sd._sweep_up(Hl, fd, phi, ups)
            st[g] = (phi, ups)
        out = torch.zeros_like(fd)
        if world == 1:
            Hl, _ = self.local[0]
            phi, ups = st[0]
            sd._sweep_down(Hl, phi, ups, out)
            return out
        # gather the subtree roots' ups (r x k_g) to rank 0
        if self.emulate:
            ups_all = [st[g][1][s] for g in range(world)]
        else:
            ups_all = self.comm.gather0(st[self.comm.rank][1][s])
        pd = None
        if self.top is not None:
            Ht, _ = self.top
            V = Ht.levels[s]
            kk = V.kmax
            U = torch.zeros((r, world * kk), dtype=_F64, device=self.dev)
            for g in range(world):
                k = int(V.k[g])
                U[:, g * kk:g * kk + k] = ups_all[g][:, :k]
            phi_t, ups_t = {}, {s: U}
            sd._sweep_up(Ht, fd, phi_t, ups_t)
            sd._sweep_down(Ht, phi_t, ups_t, torch.zeros_like(fd))
            pd = sd._phi_dn(Ht, V, phi_t, r)          # (r, world * kk)
        if not self.emulate:
            shape = self.comm.bcast_shape0(None if pd is None else pd.shape, self.dev)
            pd = self.comm.bcast0(pd, shape=shape, dtype=_F64, device=self.dev)
        kk = pd.shape[1] // world
        for g in self.ranks:
            Hl, _ = self.local[g]
            phi, ups = st[g]
            k = int(Hl.levels[s].k[0])
            pdg = pd[:, g * kk:g * kk + k].contiguous()
            sd._sweep_down(Hl, phi, ups, out, pd_top=pdg)
        if not self.emulate:
            out = self.comm.allreduce_sum(out)
        return out

    def apply(self, f):
        fd, single = sd._as_device_rhs(f, self.grid.n, self.dev, self.realified)
        return sd._from_device(self.apply_device(fd), f, single, self.realified)

    def nbytes_local(self):
        tot = sum(inv.nbytes() for _, inv in self.local.values())
        if self.top is not None:
            tot += self.top[1].nbytes()
        return tot
