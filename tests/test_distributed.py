"""The sharded (multi-GPU) path's host logic on CPU with gloo, world_size 2
and 4: subtree partition, the ragged gather / broadcast / all-reduce
collectives of distributed.TorchComm, and an end-to-end sharded solve whose
per-box arithmetic is the CPU oracle's — it must reproduce the
single-process solution to rounding (the exchange is pure data movement)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1303_5466_b200 import Grid, build_tree
from paper_1303_5466_b200.distributed import TorchComm, owned_points, subtree_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_subtree_plan_partitions_every_level():
    tree = build_tree(Grid(64), 64)
    for world in (1, 2, 4, 8):
        plan = subtree_plan(tree, world)
        assert plan.split == world.bit_length() - 1
        for lv in range(plan.split, tree.depth + 1):
            cover = []
            for g in range(world):
                lo, hi = plan.slices[g][lv]
                cover.extend(tree.ids[lv][lo:hi])
                # children of a rank's boxes stay on that rank
                if lv < tree.depth:
                    for i in tree.ids[lv][lo:hi]:
                        c1, c2 = tree.nodes[i].children
                        lo2, hi2 = plan.slices[g][lv + 1]
                        assert c1 in tree.ids[lv + 1][lo2:hi2] and c2 in tree.ids[lv + 1][lo2:hi2]
            assert sorted(cover) == sorted(tree.ids[lv])
        pts = np.concatenate([owned_points(tree, plan, g) for g in range(world)])
        np.testing.assert_array_equal(np.sort(pts), np.arange(tree.grid.n))
    with pytest.raises(ValueError):
        subtree_plan(tree, 3)
    with pytest.raises(ValueError):
        subtree_plan(build_tree(Grid(16), 64), 16)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        # ragged gather / broadcast / allreduce
        t = torch.arange((rank + 1) * 3, dtype=torch.float64).reshape(rank + 1, 3)
        got = comm.gather0(t)
        if rank == 0:
            assert [g.shape[0] for g in got] == list(range(1, world + 1))
            for g, x in enumerate(got):
                assert torch.equal(x, torch.arange((g + 1) * 3, dtype=torch.float64).reshape(g + 1, 3))
        b = torch.full((2, 5), 7.0, dtype=torch.float64) if rank == 0 else None
        shape = comm.bcast_shape0(None if b is None else b.shape, "cpu")
        b = comm.bcast0(b, shape=shape, dtype=torch.float64, device="cpu")
        assert torch.equal(b, torch.full((2, 5), 7.0, dtype=torch.float64))
        s = comm.allreduce_sum(torch.ones(4, dtype=torch.float64) * (rank + 1))
        assert float(s[0]) == world * (world + 1) / 2
        q.put((rank, _sharded_oracle_solve(comm)))
    finally:
        dist.destroy_process_group()


def _sharded_oracle_solve(comm):
    """The ShardedInverse phase structure with the oracle's per-box kernels."""
    import oracle.hssd as O
    n, leaf, eps = 32, 64, 1e-10
    P = O.Problem(n, "laplace2d", 0.0, ("one", ()), ("gaussian_bump", ()), ("one", ()), "none")
    otree = O.make_tree(n, leaf)
    ptree = build_tree(Grid(n), leaf)
    plan = subtree_plan(ptree, comm.world)
    s, g = plan.split, comm.rank
    # local subtree: levels depth..s of this rank's slice
    boxes = [int(i) for lv in range(ptree.depth, s - 1, -1)
             for i in ptree.ids[lv][plan.slices[g][lv][0]:plan.slices[g][lv][1]]]
    H = O.compress(P, otree, eps, 2, boxes=boxes)
    inv = O.invert(H, boxes=boxes)
    root = boxes[-1]
    # interface: skeletons and E of the subtree root -> rank 0
    rs = comm.gather0(torch.from_numpy(H.rskel[root]))
    cs = comm.gather0(torch.from_numpy(H.cskel[root]))
    E = comm.gather0(torch.from_numpy(inv.E[root]))
    roots = [int(i) for i in ptree.ids[s]]
    top = [int(i) for lv in range(s - 1, -1, -1) for i in ptree.ids[lv]]
    if g == 0:
        for r, b in enumerate(roots):
            H.rskel[b], H.cskel[b] = rs[r].numpy(), cs[r].numpy()
            inv.E[b] = E[r].numpy()
        O.compress(P, otree, eps, 2, boxes=top, H=H)
        O.invert(H, boxes=top, inv=inv)
    # solve
    f = np.random.default_rng(4).standard_normal((n * n, 2))
    ups, uin = {}, {}
    O.apply_up(inv, f, boxes, ups, uin)
    U = comm.gather0(torch.from_numpy(ups[root]))
    dn = {0: None}
    if g == 0:
        for r, b in enumerate(roots):
            ups[b] = U[r].numpy()
        O.apply_up(inv, f, top, ups, uin)
        O.apply_down(inv, list(reversed(top)), ups, uin, dn, np.zeros_like(f))
        pd = torch.from_numpy(np.concatenate([dn[b] for b in roots]))
        ks = torch.tensor([dn[b].shape[0] for b in roots])
    else:
        pd, ks = None, None
    shape = comm.bcast_shape0(None if pd is None else pd.shape, "cpu")
    pd = comm.bcast0(pd, shape=shape, dtype=torch.float64, device="cpu")
    ks = comm.bcast0(ks, shape=(comm.world,), dtype=torch.int64, device="cpu")
    off = int(ks[:g].sum())
    dn_local = {root: pd[off:off + int(ks[g])].numpy()}
    out = np.zeros_like(f)
    O.apply_down(inv, list(reversed(boxes)), ups, uin, dn_local, out)
    out = comm.allreduce_sum(torch.from_numpy(out)).numpy()
    return out


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_solve_matches_single_process(world):
    import oracle.hssd as O
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 32
    P = O.Problem(n, "laplace2d", 0.0, ("one", ()), ("gaussian_bump", ()), ("one", ()), "none")
    f = np.random.default_rng(4).standard_normal((n * n, 2))
    x, _, _ = O.solve(P, 64, 1e-10, f)
    for r in range(world):
        # the exchange is pure data movement; only BLAS's layout-dependent
        # summation order (gathered copies are C-ordered) separates the results
        assert np.linalg.norm(res[r] - x) <= 1e-14 * np.linalg.norm(x)


def test_top_level_owner_tree():
    """Top boxes form a binary reduction tree: box j of level l < s is owned
    by rank j 2^(s-l), the owner of its first child; every top box has exactly
    one owner; rank 0 owns the root."""
    from paper_1303_5466_b200.distributed import top_boxes, top_owner
    tree = build_tree(Grid(64), 64)
    for world in (2, 4, 8):
        plan = subtree_plan(tree, world)
        s = plan.split
        owned = {}
        for g in range(world):
            for lv, j in top_boxes(plan, g):
                assert top_owner(plan, lv, j) == g
                owned[(lv, j)] = g
        assert sorted(owned) == sorted((lv, j) for lv in range(s) for j in range(1 << lv))
        for lv in range(s):
            for j in range(1 << lv):
                assert top_owner(plan, lv, j) == top_owner(plan, lv + 1, 2 * j)
                assert top_owner(plan, lv + 1, 2 * j + 1) != top_owner(plan, lv, j)
        assert top_owner(plan, 0, 0) == 0
        # level s owners are the subtree ranks
        assert [top_owner(plan, s, g) for g in range(world)] == list(range(world))
