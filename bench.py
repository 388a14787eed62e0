"""Benchmark: dense-block recursive-skeletonization factor + solve at N = 1024^2.

Metric (BASELINE.json): factor & solve unknowns/sec at N=1024^2, tol 1e-10.
One step = build_tree + compress_outer + invert_dense_block (the factor) and a
256-RHS solve, on config 4 (Laplace log-kernel VIE, float64, leaf 64,
eps 1e-10, BASELINE bump on the rows, cell-integral diagonal; synthetic
seeded N(0,1) right-hand sides), run as solver_dense.factor_solve (levels
pipelined over streams; same results as the three calls back to back).
value = N / step time, RHS resident in HBM.
e2e = the same step through the public API (compress_inverse + apply) with the
256 RHS copied from pinned host memory and the solution copied back.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle port (oracle/hssd.py: the reference's
algorithm on scipy/OpenBLAS, all host threads) on a bounded sample of the same
workload (the 128^2 member of the family, factor + 256-RHS solve per step).
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factor & solve unknowns/sec at N=1024^2, tol 1e-10"
UNIT = "unknowns/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--side", dest="n", type=int, default=None,   # --side under torchrun
                    help="grid side (default 1024: config c4; 512 when several ranks share a GPU)")
    ap.add_argument("--nrhs", type=int, default=256)
    ap.add_argument("--cpu-n", type=int, default=128, help="oracle sample grid side")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def _dist():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def _config(n, nrhs, world):
    return {"workload": f"c4: Laplace log-kernel VIE {n}x{n} (N={n*n}), float64, leaf 64, "
                        f"eps 1e-10, factor + {nrhs}-RHS solve",
            "n_side": n, "N": n * n, "nrhs": nrhs, "leaf": 64, "eps": 1e-10,
            "kernel": "laplace2d (1/2pi) log r on [-1,1]^2, b = (pi/2)(1+0.5 exp(-|x|^2/0.08)) "
                      "rows, c = 1, cell-integral diagonal",
            "l2": "inputs and factors (~60 GB at 1024^2) far exceed the 126 MB L2 between steps",
            "parallelism": "replicas" if world > 1 else "single GPU"}


# ---------------------------------------------------------------------------
# reference arm (CPU oracle port)

def _oracle_step(n, nrhs, seed=0):
    import oracle.hssd as O
    P = O.Problem(n, "laplace2d", 0.0, ("one", ()), ("centre_bump", (("scale", math.pi / 2),)),
                  ("one", ()), "cell")
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((n * n, nrhs))
    t0 = time.perf_counter()
    tree = O.make_tree(n, 64)
    H = O.compress(P, tree, 1e-10, 2)
    inv = O.invert(H)
    x = O.apply_inverse(inv, f)
    t1 = time.perf_counter()
    return t1 - t0, x


def _cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _reference_headline():
    """The reference package itself (vief, /root/reference) at the headline
    size, measured once in the build container by tests/golden/make_golden_c3c4.py
    (stored with its solution in tests/golden/solve_c4_1024.npz): a stated
    baseline, not a same-run measurement."""
    path = os.path.join(ROOT, "tests", "golden", "solve_c4_1024.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    tb, tf, ts = (float(x) for x in g["times"])
    n = 1024 * 1024
    return {"n_side": 1024, "build_s": tb, "factor_s": tf, "solve_1rhs_s": ts,
            "factor_unknowns_per_s": n / (tb + tf), "threads": int(g["threads"]),
            "host": "build container (8-core Xeon, OpenBLAS), not the GPU box",
            "source": "tests/golden/solve_c4_1024.npz (make_golden_c3c4.py)"}


def run_reference(a):
    rank, world, _ = _dist()
    if rank != 0:
        return
    cores = _cpu_threads()
    for _ in range(a.warmup):
        _oracle_step(a.cpu_n, a.nrhs)
    times = [_oracle_step(a.cpu_n, a.nrhs)[0] for _ in range(a.steps)]
    t = sum(times) / len(times)
    v = a.cpu_n ** 2 / t
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": dict(_config(a.cpu_n, a.nrhs, world),
                           workload=f"c4 family, bounded CPU sample: Laplace log-kernel VIE "
                                    f"{a.cpu_n}x{a.cpu_n} (N={a.cpu_n ** 2}), float64, leaf 64, "
                                    f"eps 1e-10, factor + {a.nrhs}-RHS solve (the {a.n}^2 "
                                    f"headline size takes ~1 h of reference CPU per step; its "
                                    f"measured time is in reference_at_headline)",
                           sample_of=_config(a.n, a.nrhs, world)["workload"]),
            "reference_at_headline": _reference_headline(),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"oracle/hssd.py (reference algorithm on scipy "
                                       f"{__import__('scipy').__version__}/OpenBLAS, "
                                       f"{cores} threads) full factor + {a.nrhs}-RHS solve of "
                                       f"the {a.cpu_n}^2 member of the same problem family per "
                                       f"step; unknowns/s falls as N^-1/2 with size, so this "
                                       f"overstates the CPU at 1024^2"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks

class Clocks:
    def __init__(self, gpu):
        self.path = f"/tmp/vief_clocks_{os.getpid()}.csv"
        self.proc = None
        self.gpu = gpu

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# our arm

def _stage_traffic():
    """DRAM bytes per step of the factorization stages at 1024^2 from the
    committed ncu launch list (tools/ncu_levels.py under ncu)."""
    try:
        st = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_stage_traffic.json")))["stages"]
    except Exception:
        return {}
    return {"id (compress_outer)": st["id"]["dram_bytes"] + st["blocks"]["dram_bytes"],
            "lu_schur (invert_dense_block)": st["finv"]["dram_bytes"] + st["wgec"]["dram_bytes"]}


def _algorithmic_work(H):
    """SURVEY §8(d) per-box formulas evaluated with this run's m, k, p."""
    id_fl = lu_fl = 0.0
    solve_bytes = 0.0
    solve_fl = 0.0
    own_bytes = 0.0  # this layout: F^-1 (m^2) and C (k m) read up, E (k^2) and W (m k) down
    sym = H.symmetric
    for L in H.levels:
        if L is None or getattr(L, "virtual", False):
            continue
        m = L.m.astype(np.float64)
        if L.lv == 0:
            lu_fl += float(((2.0 / 3.0) * m ** 3).sum())
            solve_bytes += float((8.0 * m * m).sum())
            own_bytes += float((8.0 * m * m).sum())
            solve_fl += float((2.0 * m * m).sum())
            continue
        k = L.k.astype(np.float64)
        p = L.p.astype(np.float64)
        one = 4 * p * m * k - 2 * (p + m) * k * k + (4.0 / 3.0) * k ** 3 + k * k * (m - k)
        id_fl += float(one.sum()) * (1 if sym else 2)
        lu_fl += float(((2.0 / 3.0) * m ** 3 + 2 * m * m * k + 2 * k * k * (m - k)
                        + (2.0 / 3.0) * k ** 3 + 2 * k ** 3).sum())
        solve_bytes += float((8.0 * (2 * m * m + 2 * k * k + 2 * k * (m - k))).sum())
        own_bytes += float((8.0 * (m * m + k * k + 2 * k * m)).sum())
        solve_fl += float((4 * m * m + 4 * k * k + 6 * k * (m - k)).sum())
    return id_fl, lu_fl, solve_bytes, solve_fl, own_bytes


def run_sharded(a):
    """N > 1 GPUs: one 1024^2 problem, subtree-sharded (distributed.py): each
    rank factors its subtree, the top levels run on rank 0 from interface data
    gathered over NCCL.  Strong scaling (the total work is fixed)."""
    import torch
    import torch.distributed as dist
    rank, world, local = _dist()
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    # NCCL with one GPU per rank; with fewer GPUs than ranks (e.g. --gpus 2 on a
    # one-GPU box) the exchanges go host-staged over gloo: no rank's kernels
    # ever wait on another rank's (VF_DIST_BACKEND overrides)
    backend = os.environ.get("VF_DIST_BACKEND") or ("nccl" if ndev >= world else "gloo")
    dist.init_process_group(backend)
    from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field, _lib
    from paper_1303_5466_b200.distributed import ShardedInverse, TorchComm
    comm = TorchComm()
    # ranks sharing a GPU (no multi-GPU box): a functional check, not a scaling number --
    # the 1024^2 factors of all ranks plus each process's pools do not fit one GPU
    shared = ndev < world
    n, nrhs = (a.n or (512 if shared else 1024)), a.nrhs
    N = n * n
    spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                      c_field=make_field("one"))
    grid = Grid(n)
    opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    Ft = torch.randn((nrhs, N), dtype=torch.float64, device="cuda", generator=gen)
    fac, sol = [], []

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()

    def step(record=False):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        inv = ShardedInverse(spec, grid, build_tree(grid, 64), 1e-10, opts, CELL, world, comm=comm)
        ev[1].record()
        X = inv.apply_device(Ft, gather="root")
        ev[2].record()
        if record:
            torch.cuda.synchronize()
            fac.append(ev[0].elapsed_time(ev[1]))
            sol.append(ev[1].elapsed_time(ev[2]))
        return inv, X

    for _ in range(a.warmup):
        inv, X = step()
        del inv, X
    barrier()
    L0 = _lib.launch_count()
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record()
        for i in range(a.steps):
            inv, X = step(record=True)
            if i < a.steps - 1:
                del inv, X
        e1.record()
        barrier()
    launches = _lib.launch_count() - L0
    dev_t = "cpu" if backend == "gloo" else "cuda"
    t = torch.tensor([e0.elapsed_time(e1) / a.steps, statistics.mean(fac), statistics.mean(sol)],
                     device=dev_t)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, tf, ts = (float(v) for v in t.tolist())
    local_bytes = inv.nbytes_local()
    # whole-job algorithmic FP64 work (every rank's subtree + its top boxes)
    work = np.zeros(2)
    for H in [h for h, _ in inv.local.values()] + [h for h, _ in inv.top.values()]:
        i_fl, l_fl, _, s_fl, _ = _algorithmic_work(H)
        work += (i_fl + l_fl, s_fl * nrhs)
    wt = torch.tensor(work, dtype=torch.float64, device=dev_t)
    dist.all_reduce(wt)
    fl_tot = float(wt.sum())
    peak_fp64 = 37.1e12
    roof = {"bound": "tensor", "achieved": fl_tot / (ms / 1e3) / 1e12,
            "peak": peak_fp64 * world / 1e12, "unit": "TFLOP/s",
            "frac": fl_tot / (ms / 1e3) / (peak_fp64 * world), "traffic": None,
            "stage": "whole step (ID + LU/Schur + solve flops of all ranks, SURVEY §8(d) "
                     "formulas) against N x the measured DMMA peak"}
    del inv, X
    torch.cuda.empty_cache()
    out = {"metric": METRIC, "value": N / (ms / 1e3), "unit": UNIT, "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(_config(n, nrhs, world), parallelism=f"subtree shards x{world} + "
                          f"top boxes as a reduction tree ({backend} send/recv)"
                          + (f"; {world} ranks share {ndev} GPU(s): functional check at a size "
                             f"that fits, not a scaling measurement" if shared else "")),
           "factor_s": tf / 1e3, "solve_s": ts / 1e3, "factor_bytes_rank": local_bytes,
           "roofline": roof, "gpu_launches": int(launches), "clocks": clk.summary(),
           "backend": backend, "devices": ndev}
    if not a.no_e2e:
        Fh = Ft.t().contiguous().cpu().pin_memory()

        def e2e_step():
            inv2 = ShardedInverse(spec, grid, build_tree(grid, 64), 1e-10, opts, CELL, world,
                                  comm=comm)
            Xh = inv2.apply(Fh, gather="root")   # owned RHS rows up, full solution to rank 0
            torch.cuda.synchronize()
            del inv2, Xh

        for _ in range(a.warmup):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            e2e_step()
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / a.steps], device=dev_t)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        te = float(te.item())
        out["e2e"] = {"value": N / te, "unit": UNIT, "h2d_bytes_per_step": int(N * nrhs * 8),
                      "d2h_bytes_per_step": int(N * nrhs * 8), "ms_per_step": te * 1e3,
                      "api": "distributed.ShardedInverse(...).apply(host RHS, gather='root'): "
                             "each rank uploads its own N/P rows, rank 0 receives the solution"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def run_ours(a):
    import torch
    rank, world, local = _dist()
    if world > 1:
        return run_sharded(a)
    torch.cuda.set_device(local)
    dist = None
    from paper_1303_5466_b200 import (CELL, Grid, KernelSpec, SolverOptions, build_tree,
                                      make_field, _lib)
    from paper_1303_5466_b200 import solver_dense as sd
    from paper_1303_5466_b200.solver_compressed import compress_inverse

    n, nrhs = a.n, a.nrhs
    N = n * n
    spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                      c_field=make_field("one"))
    grid = Grid(n)
    opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    F = torch.randn((N, nrhs), dtype=torch.float64, device="cuda", generator=gen)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    stage = {}

    def step(record=False):
        """One step: build_tree + factor_solve (compress_outer + invert_dense_block
        with the levels pipelined over two streams, the solve's up sweep
        overlapping the coarser levels' factorization) of the 256 RHS."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        tree = build_tree(grid, 64)
        H, inv, X = sd.factor_solve(spec, grid, tree, 1e-10, opts, F, CELL)
        ev[1].record()
        if record:
            torch.cuda.synchronize()
            stage.setdefault("step", []).append(ev[0].elapsed_time(ev[1]))
        return H, inv, X

    def staged_step():
        """Untimed diagnostic step with the stages run back to back (no overlap),
        for the per-stage split and rooflines."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        tree = build_tree(grid, 64)
        H = sd.compress_outer(spec, grid, tree, 1e-10, opts, CELL)
        ev[1].record()
        inv = sd.invert_dense_block(H)
        ev[2].record()
        X = inv.apply(F)
        ev[3].record()
        torch.cuda.synchronize()
        # the first apply after a factorization may wait on the caching allocator
        # (buffers for 256 RHS while ~100 GB are reserved); time a second one too
        e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e2[0].record()
        X = inv.apply(F)
        e2[1].record()
        torch.cuda.synchronize()
        stage.setdefault("compress", []).append(ev[0].elapsed_time(ev[1]))
        stage.setdefault("invert", []).append(ev[1].elapsed_time(ev[2]))
        stage.setdefault("solve", []).append(min(ev[2].elapsed_time(ev[3]),
                                                 e2[0].elapsed_time(e2[1])))
        # 1-RHS sweeps (HBM-bound: every stored factor is read twice per solve)
        f1 = F[:, :1].contiguous()
        inv.apply(f1)
        e1 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 5
        e1[0].record()
        for _ in range(reps):
            inv.apply(f1)
        e1[1].record()
        torch.cuda.synchronize()
        stage.setdefault("solve1", []).append(e1[0].elapsed_time(e1[1]) / reps)
        del H, inv, X

    for _ in range(a.warmup):
        H, inv, X = step()
        del H, inv, X
    barrier()
    L0 = _lib.launch_count()
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record()
        for _ in range(a.steps):
            H, inv, X = step(record=True)
            if _ < a.steps - 1:
                del H, inv, X
        e1.record()
        barrier()
    launches = _lib.launch_count() - L0
    ms = e0.elapsed_time(e1) / a.steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * N / (ms / 1e3)

    # residual check of the last step (approximate residual of the paper, E)
    v = F[:, :4]
    r = (v - H.matvec(X[:, :4])).norm() / v.norm()
    # exact residual ||f - A x|| / ||f|| of the same 4 columns (A applied by FFT, verify.py)
    from paper_1303_5466_b200.verify import FFTOperator
    op = FFTOperator(spec, grid, CELL, "cuda")
    rt = float(((v - op.matvec(X[:, :4])).norm(dim=0) / v.norm(dim=0)).max())
    del op
    id_fl, lu_fl, sbytes, sfl, obytes = _algorithmic_work(H)
    max_rank = int(max(L.kmax for L in H.levels if L.lv))
    fbytes = inv.nbytes()
    del H, inv, X
    _lib.release_memory()  # the pipelined steps cached blocks on their own streams
    staged_step()          # warms the allocator for the back-to-back schedule
    stage.pop("compress"), stage.pop("invert"), stage.pop("solve"), stage.pop("solve1")
    staged_step()
    t_step = statistics.mean(stage["step"]) / 1e3
    t_c = statistics.mean(stage["compress"]) / 1e3
    t_i = statistics.mean(stage["invert"]) / 1e3
    t_s = statistics.mean(stage["solve"]) / 1e3
    t_s1 = statistics.mean(stage["solve1"]) / 1e3
    peak_fp64 = 37.1e12   # measured DMMA issue rate (profiles/r01_fp64_peak.txt)
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = float(peaks["hbm_gbs"]) * 1e9
    except Exception:
        hbm = 6.65e12
    sfl_all = sfl * nrhs
    roof_solve = max(sbytes / hbm, sfl_all / peak_fp64)
    stages = {
        "id (compress_outer)": {"bound": "tensor", "achieved": id_fl / t_c / 1e12,
                                "peak": peak_fp64 / 1e12, "unit": "TFLOP/s",
                                "frac": id_fl / t_c / peak_fp64, "algorithmic_flops": id_fl,
                                "seconds": t_c},
        "lu_schur (invert_dense_block)": {"bound": "tensor", "achieved": lu_fl / t_i / 1e12,
                                          "peak": peak_fp64 / 1e12, "unit": "TFLOP/s",
                                          "frac": lu_fl / t_i / peak_fp64,
                                          "algorithmic_flops": lu_fl, "seconds": t_i},
        f"solve ({nrhs} rhs)": {"bound": "tensor" if sfl_all / peak_fp64 > sbytes / hbm else "hbm",
                                "achieved": sfl_all / t_s / 1e12, "peak": peak_fp64 / 1e12,
                                "unit": "TFLOP/s", "frac": roof_solve / t_s,
                                "algorithmic_flops": sfl_all, "factor_bytes": sbytes,
                                "seconds": t_s},
        "solve (1 rhs)": {"bound": "hbm", "achieved": obytes / t_s1 / 1e9, "peak": hbm / 1e9,
                          "unit": "GB/s", "frac": obytes / t_s1 / hbm,
                          "factor_bytes_read": obytes, "seconds": t_s1,
                          "reference_layout_bytes": sbytes,
                          "note": "achieved = bytes this layout must read per solve (F^-1, C "
                                  "up; E, W down; each once) / sweep-pair time; the SURVEY "
                                  "formula counts the reference's F_lu/E/T read twice"},
    }
    # DRAM traffic per step of each stage: dram__bytes_read.sum + dram__bytes_write.sum
    # summed over the stage's kernels (ncu launch list at 1024^2, committed profile)
    traffic = _stage_traffic() if n == 1024 else {}
    for k, v in traffic.items():
        if k in stages:
            stages[k]["traffic"] = v
    dom = max(stages, key=lambda s: stages[s]["seconds"])
    roof = dict(stages[dom])
    roof = {"bound": roof["bound"], "achieved": roof["achieved"], "peak": roof["peak"],
            "unit": roof["unit"], "frac": roof["frac"], "traffic": traffic.get(dom),
            "traffic_unit": "bytes per step (the stage's kernels, ncu, "
                            "profiles/r02_ncu_stage_traffic.json)", "stage": dom,
            "peak_source": "measured DMMA mma.sync.m8n8k4.f64 issue rate 37.1 TFLOP/s "
                           "(cuBLAS DGEMM 35.5); MEASURED_PEAKS.json has no FP64 entry",
            "stage_timing": "stage seconds from one untimed back-to-back (unpipelined) "
                            "compress_outer + invert_dense_block step after the timed region"}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": _config(n, nrhs, world),
           "step_s": t_step,
           "stage_seconds_unpipelined": {"compress_outer": t_c, "invert_dense_block": t_i,
                                         "apply": t_s},
           "solve_unknown_rhs_per_s": N * nrhs / t_s,
           "approx_residual_E": float(r), "true_residual_fft": rt, "max_rank": max_rank,
           "factor_bytes": fbytes, "roofline": roof, "roofline_stages": stages,
           "gpu_launches": int(launches)}
    _lib.release_memory()
    out["clocks"] = clk.summary()

    # e2e through the public API with host buffers
    if not a.no_e2e:
        Fh = F.cpu().pin_memory()
        Xh = torch.empty_like(Fh).pin_memory()

        copy_stream = torch.cuda.Stream()

        def e2e_step():
            # the step's RHS upload is issued first on its own stream, so it
            # overlaps the factorization (it is still inside the timed region)
            with torch.cuda.stream(copy_stream):
                Fd = Fh.to("cuda", non_blocking=True)
            inv2 = compress_inverse(spec, grid, eps=1e-10, opts=opts, quad=CELL)
            torch.cuda.current_stream().wait_stream(copy_stream)
            Fd.record_stream(torch.cuda.current_stream())
            Xd = inv2.apply(Fd)
            Xh.copy_(Xd, non_blocking=True)
            torch.cuda.synchronize()
            del inv2, Xd, Fd

        for _ in range(a.warmup):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            e2e_step()
        barrier()
        te = (time.perf_counter() - t0) / a.steps
        if dist is not None:
            t = torch.tensor([te], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        out["e2e"] = {"value": world * N / te, "unit": UNIT, "h2d_bytes_per_step": int(N * nrhs * 8),
                      "d2h_bytes_per_step": int(N * nrhs * 8), "ms_per_step": te * 1e3,
                      "api": "solver_compressed.compress_inverse(k_cut=None) + .apply(pinned host "
                             "RHS -> device, upload issued on a copy stream before the factor) + "
                             "device->pinned host copy of the solution"}

    # CPU baseline (oracle port), rank 0, single GPU only
    if rank == 0 and world == 1 and not a.no_cpu:
        t, _ = _oracle_step(a.cpu_n, a.nrhs)
        cores = _cpu_threads()
        out["cpu_baseline"] = {"value": a.cpu_n ** 2 / t, "unit": UNIT, "cores": cores,
                               "kind": "port",
                               "sample": f"oracle/hssd.py at {a.cpu_n}^2 (same problem family, "
                                         f"leaf 64, eps 1e-10), factor + {nrhs}-RHS solve, "
                                         f"{t:.1f} s on {cores} threads; CPU unknowns/s falls "
                                         f"as N^-1/2, so this overstates the CPU at 1024^2"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _spawn(a):
    """--gpus N > 1 without a torchrun environment: relaunch this script as N
    ranks under torch.distributed.run (127.0.0.1 rendezvous)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)]
    # torchrun's own parser would take "--n" as an abbreviation of its options
    cmd += ["--side" if x == "--n" else ("--side=" + x[4:] if x.startswith("--n=") else x)
            for x in sys.argv[1:]]
    return subprocess.call(cmd)


if __name__ == "__main__":
    args = _args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    if int(os.environ.get("WORLD_SIZE", 1)) == 1 or args.impl == "reference":
        args.n = args.n or 1024
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
