"""A/B timing of module-level knobs of solver_dense on the bench step
(factor_solve at 1024^2, 256 RHS): each setting runs W warm-ups and K timed
steps (CUDA events), settings interleaved.

    python tools/ab_step.py _ID_PRIORITY=0 _ID_PRIORITY=-100 [--steps 3]
    python tools/ab_step.py "env:VF_AB_D=16,8,4,2" "env:VF_AB_D=16,16,8,4"
(settings: ';'-separated key=value; env:NAME sets an environment variable)
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, build_tree, make_field
from paper_1303_5466_b200 import solver_dense as sd

ap = argparse.ArgumentParser()
ap.add_argument("settings", nargs="+")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--rounds", type=int, default=2)
a = ap.parse_args()

spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                  c_field=make_field("one"))
grid = Grid(a.n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
F = torch.randn((grid.n, 256), dtype=torch.float64, device="cuda")


def apply(setting):
    for kv in setting.split(";"):
        k, v = kv.split("=", 1)
        if k.startswith("env:"):   # library knob read from the environment per call
            os.environ[k[4:]] = v
        else:
            setattr(sd, k, type(getattr(sd, k))(eval(v)))
    sd._SIDE.clear()
    sd._WORKERS.clear()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def step():
    r = sd.factor_solve(spec, grid, build_tree(grid, 64), 1e-10, opts, F, CELL)
    del r


res = {s: [] for s in a.settings}
for rnd in range(a.rounds):
    for s in a.settings:
        apply(s)
        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        for _ in range(a.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize()
            res[s].append(e0.elapsed_time(e1))
            print(f"{s}: {res[s][-1]:.1f} ms, reserved {torch.cuda.memory_reserved() / 1e9:.1f} GB",
                  flush=True)
for s, v in res.items():
    v = sorted(v)
    print(f"{s:40s} median {v[len(v) // 2]:8.1f} ms  min {v[0]:8.1f}  all {[round(x) for x in v]}")
