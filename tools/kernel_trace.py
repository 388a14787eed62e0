"""Kernel timeline of one bench step (the c4 factor + 256-RHS solve) from
CUPTI via torch.profiler -- the nsys-style breakdown (nsys is not in the
image).  Every kernel of the process is recorded, ours (libvief_b200.so) and
torch's, with device start/end timestamps.

Reports: kernel time by name (sum of durations), the GPU-busy fraction (union
of kernel intervals over the step), how much of the step has 1 / 2 / 3+
kernels in flight, and busy time per 100 ms window.  Writes a JSON summary.

    python tools/kernel_trace.py [--n 1024] [--nrhs 256] [--out profiles/r02_kernel_trace.json]
"""
import argparse
import collections
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=256)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--out", default="gpurun_out/kernel_trace.json")
ap.add_argument("--dump", default="", help="also write every kernel (name, stream, start, dur, grid) here (.json.gz)")
a = ap.parse_args()

spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                  c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
F = torch.randn((grid.n, a.nrhs), dtype=torch.float64, device="cuda")


def step():
    tree = build_tree(grid, 64)
    H, inv, X = sd.factor_solve(spec, grid, tree, 1e-10, opts, F, CELL)
    return H, inv, X


for _ in range(a.warmup):
    r = step()
    del r
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    r = step()
    ev1.record()
    torch.cuda.synchronize()
step_ms = ev0.elapsed_time(ev1)
if a.dump:
    import gzip
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".json") as tf:
        prof.export_chrome_trace(tf.name)
        tr = json.load(open(tf.name))
    rows = [(e["name"][:80], e["args"].get("stream"), e["ts"], e["dur"], e["args"].get("grid"),
             e["args"].get("block"))
            for e in tr["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    with gzip.open(a.dump, "wt") as fo:
        json.dump(rows, fo)
kern = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0:
        name = e.name
        if name.startswith("Memcpy") or name.startswith("Memset"):
            kind = "copy"
        else:
            kind = "kernel"
        kern.append((e.time_range.start, e.time_range.end, name, kind))
kern.sort()
t0 = min(k[0] for k in kern)
t1 = max(k[1] for k in kern)
# per-name totals
tot = collections.defaultdict(lambda: [0.0, 0])
for s, e, n, kind in kern:
    short = n.split("(")[0]
    tot[short][0] += (e - s) / 1e3
    tot[short][1] += 1
# concurrency profile: sweep over interval endpoints
pts = []
for s, e, n, kind in kern:
    if kind == "kernel":
        pts.append((s, 1))
        pts.append((e, -1))
pts.sort()
conc = collections.Counter()
cur, last = 0, pts[0][0]
for t, d in pts:
    conc[min(cur, 3)] += t - last
    cur += d
    last = t
span = (t1 - t0)
busy = sum(v for c, v in conc.items() if c > 0)
# busy per 100 ms window
win = collections.Counter()
for s, e, n, kind in kern:
    if kind != "kernel":
        continue
    a_, b_ = s - t0, e - t0
    w = int(a_ // 100000)
    while a_ < b_:
        end = min(b_, (w + 1) * 100000)
        win[w] += end - a_
        a_ = end
        w += 1
ours = sum(v[0] for k, v in tot.items() if k.startswith("void vf::") or k.startswith("vf::"))
allk = sum(v[0] for k, v in tot.items())
top = sorted(tot.items(), key=lambda kv: -kv[1][0])[:40]
summary = {
    "workload": f"bench step at {a.n}^2, {a.nrhs} RHS (factor_solve), one step after {a.warmup} warm-ups",
    "step_ms_events": step_ms,
    "trace_span_ms": span / 1e3,
    "launches": len(kern),
    "kernel_ms_sum": allk,
    "ours_kernel_ms_sum": ours,
    "gpu_busy_ms": busy / 1e3,
    "gpu_busy_frac": busy / span,
    "concurrency_ms": {"0": conc[0] / 1e3, "1": conc[1] / 1e3, "2": conc[2] / 1e3, "3+": conc[3] / 1e3},
    "busy_ms_per_100ms_window (sum of kernel durations)": [round(win[w] / 1e3, 1) for w in range(int(span // 100000) + 1)],
    "top_kernels": [{"name": k, "ms": round(v[0], 3), "launches": v[1],
                     "share_of_kernel_time": round(v[0] / allk, 4)} for k, v in top],
}
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
json.dump(summary, open(a.out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "top_kernels"}, indent=1))
for t in summary["top_kernels"][:25]:
    print(f"{t['ms']:9.2f} ms {t['launches']:6d}  {100 * t['share_of_kernel_time']:5.1f}%  {t['name'][:100]}")
