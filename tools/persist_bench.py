"""Save / load throughput of a factorization (persist.py) and a bitwise check
that the loaded factors solve like the saved ones.

python tools/persist_bench.py --n 512 [--dir /tmp]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math  # noqa: E402
from paper_1303_5466_b200 import CELL, Grid, KernelSpec, SolverOptions, make_field  # noqa: E402
from paper_1303_5466_b200 import solver_compressed as sc  # noqa: E402
from paper_1303_5466_b200.solver_compressed import CompressedInverse  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--dir", default="/tmp")
    a = ap.parse_args()
    # the bench problem (bench.py run_ours)
    spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2),
                      c_field=make_field("one"))
    grid = Grid(a.n)
    opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
    inv = sc.compress_inverse(spec, grid, eps=1e-10, opts=opts, quad=CELL)
    f = np.random.default_rng(0).standard_normal(grid.n)
    x0 = inv.apply(f)
    path = os.path.join(a.dir, f"vief_{a.n}.vief")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inv.save(path)
    os.sync()
    t1 = time.perf_counter()
    size = os.path.getsize(path)
    del inv
    torch.cuda.empty_cache()
    t2 = time.perf_counter()
    inv2 = CompressedInverse.load(path)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    x1 = inv2.apply(f)
    os.remove(path)
    print(json.dumps({"n_side": a.n, "file_bytes": size, "save_s": t1 - t0,
                      "save_GBps": size / (t1 - t0) / 1e9, "load_s": t3 - t2,
                      "load_GBps": size / (t3 - t2) / 1e9,
                      "bitwise_equal_solution": bool(np.array_equal(x0, x1))}))


if __name__ == "__main__":
    main()
