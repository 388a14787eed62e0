"""Subtree-sharded factor / solve across GPUs.

Boxes of one level depend only on their children, so with P = 2^s ranks the
tree splits at level s: rank g factors the subtree rooted at the g-th box of
level s (levels s..depth) with no communication.  The top levels 0..s-1 are
factored as a binary reduction tree: box j of level l < s is owned by rank
j * 2^(s-l) (the owner of its first child), which receives the second child's
interface -- k, row/column skeleton index lists and the k x k reduced operator
E -- from that child's owner (point-to-point, NCCL send/recv), and factors the
box from a "virtual" child level holding both children's interface data.  The
first child's G1 = E1^{-1} (kept before E1 was inverted) never leaves its rank,
so every top box is inverted by block elimination, as on one GPU.  At level l
only 2^l ranks work (rank 0 factors the root); SURVEY §8(e) bounds the factor
speed-up of this plan at 1.92x / 2.89x / 3.54x for P = 2 / 4 / 8 at 1024^2.

The solve follows the same tree: up sweep locally, then for l = s-1 .. 0 the
second child's `ups` (r x k) goes to the parent's owner; down sweep from the
root, the second child's phi_dn slice (r x k) goes back to the child's owner;
the local down sweep finishes on every rank.  Each rank reads only the
right-hand-side rows of its own grid points (`apply` uploads just those) and
writes only its own solution rows; `gather="root"|"all"` assembles the full
solution from the owned rows (a gather of N/P x r per rank, not an all-reduce
of the full array).  Every rank holds only its subtree's factors plus the top
boxes it owns.

The algorithm is written as explicit phases so that the same code runs
  * over torch.distributed (one process per GPU, NCCL; gloo for CPU tests and
    for several ranks sharing one GPU -- host-staged, no rank ever waits on
    another rank's kernel), or
  * emulated in one process on one GPU (`emulate=True`).
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
    top: dict = field(default_factory=dict)  # {level: (lo, hi)} for levels < s (all boxes)


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


def top_owner(plan, lv, j):
    """Rank that factors box j of level lv <= s (level s: the subtree owner)."""
    return j << (plan.split - lv)


def top_boxes(plan, rank):
    """[(level, j)] of the top boxes `rank` factors, finest level first."""
    s = plan.split
    out = []
    for lv in range(s - 1, -1, -1):
        step = 1 << (s - lv)
        if rank % step == 0:
            out.append((lv, rank // step))
    return out


def owned_points(tree, plan, rank):
    """Grid points owned by a rank (its subtree's leaves)."""
    lo, hi = plan.slices[rank][tree.depth]
    own = tree.owned_level(tree.depth)[lo:hi]
    return np.sort(own[own >= 0].ravel())


# ---------------------------------------------------------------------------
# communication

class TorchComm:
    """Point-to-point and collective helpers over torch.distributed (NCCL for
    CUDA tensors, gloo for host tensors or several ranks on one GPU)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.backend = dist.get_backend()

    def _wire(self, t):
        """gloo moves host tensors only."""
        return t.cpu() if self.backend == "gloo" and t.is_cuda else t

    def send(self, t, dst):
        """Ragged send: shape first (int64 vector), then the data."""
        t = t.contiguous()
        dev = "cpu" if self.backend == "gloo" else t.device
        hdr = torch.tensor([t.dim()] + list(t.shape), dtype=torch.int64, device=dev)
        self.dist.send(torch.tensor([hdr.numel()], dtype=torch.int64, device=dev), dst)
        self.dist.send(hdr, dst)
        if t.numel():
            self.dist.send(self._wire(t), dst)

    def recv(self, src, dtype, device):
        dev = "cpu" if self.backend == "gloo" else device
        n = torch.zeros(1, dtype=torch.int64, device=dev)
        self.dist.recv(n, src)
        hdr = torch.zeros(int(n.item()), dtype=torch.int64, device=dev)
        self.dist.recv(hdr, src)
        shape = [int(x) for x in hdr[1:].tolist()]
        t = torch.empty(shape, dtype=dtype, device=dev)
        if t.numel():
            self.dist.recv(t, src)
        return t.to(device)

    def gather0(self, t):
        """Tensors of any shape (same dtype) -> list on rank 0, None elsewhere
        (point-to-point: only rank 0 receives, nobody gets the others' data)."""
        if self.rank != 0:
            self.send(t, 0)
            return None
        out = [t]
        for g in range(1, self.world):
            out.append(self.recv(g, t.dtype, t.device))
        return out

    def bcast0(self, t, shape=None, dtype=None, device=None):
        dist = self.dist
        if self.rank != 0:
            t = torch.empty(shape, dtype=dtype, device=device)
        else:
            t = t.contiguous()  # collectives move raw storage
        w = self._wire(t)
        dist.broadcast(w, src=0)
        return w.to(t.device) if w is not t else t

    def bcast_shape0(self, shape, device):
        dev = "cpu" if self.backend == "gloo" else device
        v = torch.tensor(list(shape) if shape is not None else [0, 0], dtype=torch.int64,
                         device=dev)
        self.dist.broadcast(v, src=0)
        return tuple(v.tolist())

    def allreduce_sum(self, t):
        t = t.contiguous()
        w = self._wire(t)
        self.dist.all_reduce(w)
        return w.to(t.device) if w is not t else t

    def all_gather(self, t):
        """Same-shape tensors -> list on every rank."""
        w = self._wire(t.contiguous())
        bufs = [torch.empty_like(w) for _ in range(self.world)]
        self.dist.all_gather(bufs, w)
        return [b.to(t.device) for b in bufs]


class _LocalComm:
    """Message passing between the emulated ranks of one process (the two
    sides of a split top box run on two threads: wait_recv blocks)."""

    def __init__(self):
        import threading
        self.box = {}
        self.cv = threading.Condition()

    def send(self, t, src, dst, tag):
        with self.cv:
            self.box[(src, dst, tag)] = t
            self.cv.notify_all()

    def recv(self, src, dst, tag):
        with self.cv:
            return self.box.pop((src, dst, tag))

    def wait_recv(self, src, dst, tag, timeout=600):
        with self.cv:
            if not self.cv.wait_for(lambda: (src, dst, tag) in self.box, timeout):
                raise TimeoutError(f"emulated message {tag} from rank {src} never arrived")
            return self.box.pop((src, dst, tag))


# ---------------------------------------------------------------------------
# device phases

def _interface(H, lv, item=0):
    """Item `item` of level lv's interface: k, row/col skeletons, E, G1 or None."""
    L = H.levels[lv]
    k = int(L.k[item])
    rs = L.rskel[item, :k].to(torch.int64)
    cs = L.cskel[item, :k].to(torch.int64)
    E = L.E[item, :k, :k].contiguous()        # storage [col, row]
    G = getattr(L, "Gkeep", None)
    G1 = None if G is None else G[item // 2, :k, :k].contiguous()
    return k, rs, cs, E, G1


class _Couple:
    """vief_id_desc.couple for a top box whose row ID (side 0) and column ID
    (side 1) run on two ranks: every call swaps one int with the peer through
    `exchange(v) -> peer's v` and combines them (mode 0: either side still
    factoring; mode 1: group rank = max)."""

    def __init__(self, exchange):
        self.exchange = exchange
        self.error = None

        def cb(mode, value, ctx):
            try:
                other = int(self.exchange(int(value)))
            except BaseException as e:   # noqa: BLE001 -- re-raised by _id_batched
                self.error = e
                return 0
            return max(value, other) if mode == 1 else int(bool(value) or bool(other))

        self.fn = _lib.COUPLE_FN(cb)


class _ThreadPair:
    """Rendezvous of two host threads of one process (emulated ranks)."""

    def __init__(self):
        import threading
        self.bar = threading.Barrier(2)
        self.vals = [None, None]

    def exchange(self, side, v):
        self.vals[side] = v
        self.bar.wait(timeout=600)
        o = self.vals[1 - side]
        self.bar.wait(timeout=600)
        return o


def _virtual_level(Ht, lv, parts, dev):
    """Populate level `lv` of a top object with the children's interface
    data: parts = [(k, rskel, cskel, E, G1 or None)] for the level's boxes.
    The first child's G1 = E1^{-1} feeds the parent's block elimination."""
    V = Ht.levels[lv]
    V.virtual = True
    V.k = np.asarray([p[0] for p in parts], dtype=np.int32)
    V.kmax = max(int(V.k.max()), 1)
    V.k_d = sd._dev_i32(V.k, dev)
    P = len(parts)
    V.rskel = torch.zeros((P, V.kmax), dtype=_I32, device=dev)
    V.cskel = torch.zeros((P, V.kmax), dtype=_I32, device=dev)
    V.E = torch.zeros((P, V.kmax, V.kmax), dtype=_F64, device=dev)
    have_g = all(parts[g][4] is not None for g in range(0, P, 2))
    if have_g:
        V.Gkeep = torch.zeros((P // 2, V.kmax, V.kmax), dtype=_F64, device=dev)
    for g, (k, rs, cs, E, G1) in enumerate(parts):
        V.rskel[g, :k] = rs.to(dev, _I32)
        V.cskel[g, :k] = cs.to(dev, _I32)
        if E is not None:   # (a helper computing only a column ID has no E)
            V.E[g, :k, :k] = E.to(dev)
        if have_g and g % 2 == 0:
            V.Gkeep[g // 2, :k, :k] = G1.to(dev)
    return V


class ShardedInverse:
    """Subtree-sharded HSS-D factorization.  Construct with a communicator
    (TorchComm) for one-process-per-GPU runs, or with `emulate=True` to run
    all shards in this process (single-GPU validation of the sharded path)."""

    def __init__(self, spec, grid, tree, eps, opts, quad, world, comm=None, emulate=False,
                 support_mask=None, split_ids=True):
        self.spec, self.grid, self.tree, self.eps, self.opts, self.quad = spec, grid, tree, eps, opts, quad
        self.plan = plan = subtree_plan(tree, world)
        self.comm = comm
        self.emulate = emulate
        self.ranks = list(range(world)) if emulate else [comm.rank]
        self._lc = _LocalComm() if emulate else None
        self.local = {}
        # finite k_cut: the compressed path's a-priori skeletons (host annotation
        # is deterministic, so every rank derives the same splits)
        apriori = None
        if not (opts.k_cut is None or opts.k_cut == np.inf):
            from .solver_compressed import ensure_apriori_skeletons
            apriori = ensure_apriori_skeletons(spec, tree, opts, support_mask)
        self.apriori = apriori
        s = plan.split
        for g in self.ranks:
            # the subtree is factored like one GPU's problem: IDs and inversions
            # pipelined over the compression / inversion streams
            Hl = sd.Hss2dMatrix(spec, grid, tree, eps, opts, quad, level_slices=plan.slices[g])
            with sd._host_quiet():
                Hl, invl, _ = sd._factorize(spec, grid, tree, eps, opts, quad, apriori=apriori,
                                            H=Hl)
            self.local[g] = (Hl, invl)
        self.dev = next(iter(self.local.values()))[0].device
        # top boxes: the row ID on the owner, the column ID on the second child's
        # owner (idle at that level), ranks coupled per block (pivoted IDs of
        # non-symmetric problems; a symmetric problem has one ID per box)
        self.split_ids = (bool(split_ids) and apriori is None
                          and next(iter(self.local.values()))[0].group == 2)
        self.realified = next(iter(self.local.values()))[0].realified
        # top boxes: (lv, j) -> (object, inverse), on the owning rank
        self.top = {}
        for lv in range(s - 1, -1, -1):
            # second children's owners send their interface to the parent's owner
            for j in range(1 << lv):
                owner = top_owner(plan, lv, j)
                src = top_owner(plan, lv + 1, 2 * j + 1)
                if src in self.ranks:
                    self._send(self._iface(lv + 1, 2 * j + 1), src, owner, ("if", lv, j))
            for j in range(1 << lv):
                owner = top_owner(plan, lv, j)
                src = top_owner(plan, lv + 1, 2 * j + 1)
                if self.split_ids:
                    self._top_box_split(lv, j, owner, src)
                    continue
                if owner not in self.ranks:
                    continue
                first = self._iface(lv + 1, 2 * j)
                second = self._recv_iface(src, owner, ("if", lv, j))
                Ht = self._top_object(lv, j, [first, second])
                sd.compress_levels(Ht)
                self.top[(lv, j)] = (Ht, sd.invert_dense_block(Ht))
                self._drop_g1(lv + 1, 2 * j)   # copied into the virtual level, consumed

    def _top_object(self, lv, j, parts):
        Ht = sd.Hss2dMatrix(self.spec, self.grid, self.tree, self.eps, self.opts, self.quad,
                            level_slices={lv: (j, j + 1), lv + 1: (2 * j, 2 * j + 2)})
        _virtual_level(Ht, lv + 1, parts, self.dev)
        Ht.apriori = self.apriori
        return Ht

    def _top_box_split(self, lv, j, owner, helper):
        """Top box j of level lv factored by two ranks: `owner` runs the row ID
        and the whole inversion (F^-1 pipelined with its ID on the inversion
        stream, then W, G, E, C), `helper` (the second child's owner, idle at
        this level) runs the column ID; the IDs' ranks are coupled block by
        block through the library callback.  Messages: the first child's
        skeleton lists to the helper (k + 2k ints), the column ID's perm and T
        (m ints, k (m - k) doubles) back to the owner."""
        tag = ("top", lv, j)
        first_here = owner in self.ranks
        first = self._iface(lv + 1, 2 * j) if first_here else None
        second = None
        if first_here:
            # the helper's interface first (it sent it before this call), then
            # the first child's skeletons -> helper (no E: it only runs the ID)
            second = self._recv_iface(helper, owner, ("if", lv, j))
            k, rs, cs, _, _ = first
            self._send_skel((k, rs, cs), owner, helper, tag + ("skel",))
        if helper in self.ranks:
            fk, frs, fcs = self._recv_skel(owner, helper, tag + ("skel",))
        roles = []
        if first_here:
            roles.append(("owner", owner))
        if helper in self.ranks:
            roles.append(("helper", helper))
        pair = _ThreadPair() if self.emulate else None
        box = {}

        def exch_for(side):
            if self.emulate:
                return lambda v: pair.exchange(side, v)
            peer = helper if side == 0 else owner
            return lambda v: self._swap_int(v, peer, first=(side == 0))

        def run_owner():
            Ht = self._top_object(lv, j, [first, second])
            cp = _Couple(exch_for(0))
            Ht.id_split = (0, cp, None, lambda: self._recv_col(helper, owner, tag))
            with sd._host_quiet():
                Ht, inv, _ = sd._factorize(self.spec, self.grid, self.tree, self.eps, self.opts,
                                           self.quad, apriori=self.apriori, H=Ht)
            Ht.id_split = None
            box["owner"] = (Ht, inv)

        def run_helper():
            second = self._iface(lv + 1, 2 * j + 1)
            Hh = self._top_object(lv, j, [(fk, frs, fcs, None, None), second])
            cp = _Couple(exch_for(1))
            Hh.id_split = (1, cp, lambda perm, T: self._send_col(perm, T, helper, owner, tag),
                           None)
            st = torch.cuda.Stream(self.dev)
            # the top object's virtual level (skeleton lists, padded copies) was built by
            # kernels on the caller's stream: the ID stream starts after them
            st.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(st):
                sd.compress_levels(Hh)
            st.synchronize()

        if len(roles) == 2:   # emulated: both sides in this process, one thread each
            import threading
            errs = []

            def guard(fn):
                try:
                    fn()
                except BaseException as e:   # noqa: BLE001
                    errs.append(e)
            th = threading.Thread(target=guard, args=(run_helper,))
            th.start()
            guard(run_owner)
            th.join()
            if errs:
                raise errs[0]
        elif roles and roles[0][0] == "owner":
            run_owner()
        elif roles:
            run_helper()
        if "owner" in box:
            self.top[(lv, j)] = box["owner"]
            self._drop_g1(lv + 1, 2 * j)

    # -- messaging (emulated or torch.distributed) -----------------------------
    def _iface(self, lv, j):
        """Interface of box j of level lv, from the object on this process
        that factored it (subtree root at lv == s, else a top box)."""
        if lv == self.plan.split:
            return _interface(self.local[j][0], lv, 0)
        return _interface(self.top[(lv, j)][0], lv, 0)

    def _drop_g1(self, lv, j):
        H = self.local[j][0] if lv == self.plan.split else self.top[(lv, j)][0]
        H.levels[lv].Gkeep = None

    def _send(self, iface, src, dst, tag):
        if src == dst:
            return
        if self.emulate:
            self._lc.send(iface, src, dst, tag)
            return
        k, rs, cs, E, _ = iface
        for t in (torch.tensor([k], dtype=torch.int64, device=self.dev), rs, cs, E):
            self.comm.send(t, dst)

    def _recv_iface(self, src, dst, tag):
        if self.emulate:
            k, rs, cs, E, _ = self._lc.recv(src, dst, tag)
            return k, rs, cs, E, None
        k = int(self.comm.recv(src, torch.int64, self.dev).item())
        rs = self.comm.recv(src, torch.int64, self.dev)
        cs = self.comm.recv(src, torch.int64, self.dev)
        E = self.comm.recv(src, _F64, self.dev)
        return k, rs, cs, E, None

    def _send_skel(self, skel, src, dst, tag):
        if src == dst:
            return
        if self.emulate:
            self._lc.send(skel, src, dst, tag)
            return
        k, rs, cs = skel
        for t in (torch.tensor([k], dtype=torch.int64, device=self.dev), rs, cs):
            self.comm.send(t, dst)

    def _recv_skel(self, src, dst, tag):
        if self.emulate:
            return self._lc.recv(src, dst, tag)
        k = int(self.comm.recv(src, torch.int64, self.dev).item())
        rs = self.comm.recv(src, torch.int64, self.dev)
        cs = self.comm.recv(src, torch.int64, self.dev)
        return k, rs, cs

    def _send_col(self, perm, T, src, dst, tag):
        if self.emulate:
            self._lc.send((perm, T), src, dst, tag + ("col",))
            return
        self.comm.send(perm, dst)
        self.comm.send(T, dst)

    def _recv_col(self, src, dst, tag):
        if self.emulate:
            return self._lc.wait_recv(src, dst, tag + ("col",))
        perm = self.comm.recv(src, torch.int32, self.dev)
        T = self.comm.recv(src, _F64, self.dev)
        return perm, T

    def _swap_int(self, v, peer, first):
        """One int each way with `peer` (side 0 sends first)."""
        dist = self.comm.dist
        dev = "cpu" if self.comm.backend == "gloo" else self.dev
        out = torch.tensor([v], dtype=torch.int64, device=dev)
        got = torch.zeros(1, dtype=torch.int64, device=dev)
        if first:
            dist.send(out, peer)
            dist.recv(got, peer)
        else:
            dist.recv(got, peer)
            dist.send(out, peer)
        return int(got.item())

    def _xfer(self, t, src, dst, tag):
        """Move tensor t (present on src) to dst; returns it on dst."""
        if src == dst:
            return t
        if self.emulate:
            self._lc.send(t, src, dst, tag)
            return self._lc.recv(src, dst, tag)
        if self.comm.rank == src:
            self.comm.send(t, dst)
            return None
        if self.comm.rank == dst:
            return self.comm.recv(src, _F64, self.dev)
        return None

    # -- solve ----------------------------------------------------------------
    def apply_device(self, fd, gather="all"):
        """fd: (r, N') right-hand sides on the device (only the rows of this
        rank's grid points are read).  Returns the (r, N') solution: complete
        on every rank (gather="all"), on rank 0 only ("root"; other ranks get
        their owned rows), or owned rows only ("none")."""
        r = fd.shape[0]
        plan = self.plan
        s, world = plan.split, plan.world
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

        def ups_of(lv, j):  # this process's ups of box j at level lv (r x k)
            if lv == s:
                return st[j][1][s]
            return self._tst[(lv, j)][1][lv]

        # up: level s-1 .. 0 (second child's ups travel to the parent's owner)
        self._tst = {}
        for lv in range(s - 1, -1, -1):
            moved = {}
            for j in range(1 << lv):
                owner = top_owner(plan, lv, j)
                src = top_owner(plan, lv + 1, 2 * j + 1)
                if self.emulate or self.comm.rank in (owner, src):
                    have = src in self.ranks
                    moved[j] = self._xfer(ups_of(lv + 1, 2 * j + 1) if have else None, src, owner,
                                          ("up", lv, j))
            for j in range(1 << lv):
                owner = top_owner(plan, lv, j)
                if owner not in self.ranks:
                    continue
                Ht, _ = self.top[(lv, j)]
                V = Ht.levels[lv + 1]
                kk = V.kmax
                U = torch.zeros((r, 2 * kk), dtype=_F64, device=self.dev)
                u1 = ups_of(lv + 1, 2 * j)
                U[:, :int(V.k[0])] = u1[:, :int(V.k[0])]
                U[:, kk:kk + int(V.k[1])] = moved[j][:, :int(V.k[1])]
                phi_t, ups_t = {}, {lv + 1: U}
                sd._sweep_up(Ht, fd, phi_t, ups_t)
                self._tst[(lv, j)] = (phi_t, ups_t)
        # down: level 0 .. s-1 (second child's phi_dn travels to its owner)
        pd_of = {}   # (lv, j) -> phi_dn (r x k) of box j at level lv, on its owner
        for lv in range(s):
            sent = {}
            for j in range(1 << lv):
                owner = top_owner(plan, lv, j)
                if owner in self.ranks:
                    Ht, _ = self.top[(lv, j)]
                    phi_t, ups_t = self._tst[(lv, j)]
                    sd._sweep_down(Ht, phi_t, ups_t, torch.zeros_like(fd), pd_top=pd_of.get((lv, j)))
                    V = Ht.levels[lv + 1]
                    pd = sd._phi_dn(Ht, V, phi_t, r)          # (r, 2 * kk)
                    kk = V.kmax
                    pd_of[(lv + 1, 2 * j)] = pd[:, :int(V.k[0])].contiguous()
                    sent[j] = pd[:, kk:kk + int(V.k[1])].contiguous()
            for j in range(1 << lv):
                owner = top_owner(plan, lv, j)
                dst = top_owner(plan, lv + 1, 2 * j + 1)
                if self.emulate or self.comm.rank in (owner, dst):
                    got = self._xfer(sent.get(j), owner, dst, ("dn", lv, j))
                    if dst in self.ranks:
                        pd_of[(lv + 1, 2 * j + 1)] = got
        for g in self.ranks:
            Hl, _ = self.local[g]
            phi, ups = st[g]
            sd._sweep_down(Hl, phi, ups, out, pd_top=pd_of[(s, g)].contiguous())
        self._tst = None
        if self.emulate or gather == "none":
            return out
        return self._assemble(out, gather)

    def _owned_cols(self, g):
        cols = getattr(self, "_own_cache", {}).get(g)
        if cols is None:
            pts = owned_points(self.tree, self.plan, g)
            if self.realified:  # (Re, Im) interleaved per point
                pts = np.stack([2 * pts, 2 * pts + 1], 1).ravel()
            cols = torch.as_tensor(pts, dtype=torch.int64, device=self.dev)
            self.__dict__.setdefault("_own_cache", {})[g] = cols
        return cols

    def _assemble(self, out, gather):
        """Full solution from every rank's owned columns (equal counts per rank
        for the uniform trees this plan accepts)."""
        comm = self.comm
        mine = out[:, self._owned_cols(comm.rank)].contiguous()
        if gather == "all":
            parts = comm.all_gather(mine)
        else:
            parts = comm.gather0(mine)
            if parts is None:
                return out
        full = torch.zeros_like(out)
        for g, p in enumerate(parts):
            full[:, self._owned_cols(g)] = p.to(full.device)
        return full

    def apply(self, f, gather="all"):
        """Host or device right-hand sides (N,) / (N, r).  Only this rank's
        grid points are uploaded (H2D bytes ~ N / P per rank)."""
        n = self.grid.n
        if isinstance(f, torch.Tensor) and f.is_cuda:
            fd, single = sd._as_device_rhs(f, n, self.dev, self.realified)
        else:
            arr = f.numpy() if isinstance(f, torch.Tensor) else np.asarray(f)
            a2 = arr[:, None] if arr.ndim == 1 else arr
            pts = np.concatenate([owned_points(self.tree, self.plan, g) for g in self.ranks])
            rows = torch.from_numpy(np.ascontiguousarray(a2[pts]))
            if torch.cuda.is_available():
                rows = rows.pin_memory()
            full = torch.zeros((n, a2.shape[1]), dtype=rows.dtype, device=self.dev)
            full[torch.as_tensor(pts, device=self.dev)] = rows.to(self.dev, non_blocking=True)
            fd, single = sd._as_device_rhs(full[:, 0] if arr.ndim == 1 else full, n, self.dev,
                                           self.realified)
        return sd._from_device(self.apply_device(fd, gather), f, single, self.realified)

    def nbytes_local(self):
        tot = sum(inv.nbytes() for _, inv in self.local.values())
        tot += sum(inv.nbytes() for _, inv in self.top.values())
        return tot
