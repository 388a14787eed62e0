"""GPU timeline of the pipelined factorize(): per level, when each of the four
phases (compress blocks / IDs on the main stream, F inversion / W,G,E,C on the
side stream) starts and ends (CUDA events, ms from the first event)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, CELL
from paper_1303_5466_b200 import solver_dense as sd

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
rec = []


def wrap(name):
    f = getattr(sd, name)

    def g(*a, **k):
        L = a[1]
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        r = f(*a, **k)
        h1 = time.perf_counter()
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        rec.append((name, L.lv, e0, e1, h0, h1))
        return r
    setattr(sd, name, g)


for nm in ["_compress_level_blocks", "_compress_level_id", "_invert_level_F", "_invert_level_rest"]:
    wrap(nm)
reps = []
for rep in range(int(os.environ.get("REPS", "3"))):
    rec.clear()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    hs = time.perf_counter()
    tree = build_tree(grid, 64)
    H, inv = sd.factorize(spec, grid, tree, 1e-10, opts, CELL)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: {t0.elapsed_time(t1):.1f} ms", flush=True)
    reps.append({(name, lv): e0.elapsed_time(e1) for name, lv, e0, e1, h0, h1 in rec})
    del H, inv
ms = torch.cuda.memory_stats()
print(f"total {t0.elapsed_time(t1):.1f} ms; torch reserved {torch.cuda.memory_reserved() / 1e9:.1f} GB "
      f"(max {torch.cuda.max_memory_reserved() / 1e9:.1f}), max allocated "
      f"{torch.cuda.max_memory_allocated() / 1e9:.1f} GB, alloc retries {ms.get('num_alloc_retries')}, "
      f"cudaMalloc calls {ms.get('num_device_alloc')}, cudaFree calls {ms.get('num_device_free')}")
short = {"_compress_level_blocks": "blocks", "_compress_level_id": "ID", "_invert_level_F": "F^-1", "_invert_level_rest": "WGEC"}
for name, lv, e0, e1, h0, h1 in rec:
    print(f"L{lv:02d} {short[name]:>6s}  gpu {t0.elapsed_time(e0):8.1f} -> {t0.elapsed_time(e1):8.1f}  ({e0.elapsed_time(e1):7.1f})"
          f"   host {(h0 - hs) * 1e3:8.1f} -> {(h1 - hs) * 1e3:8.1f}")

# phases whose duration varies across the warm reps (> 20 ms spread)
if len(reps) > 2:
    print("unstable phases (gpu ms per rep 1..):")
    for key in reps[1]:
        vals = [r.get(key, 0.0) for r in reps[1:]]
        if max(vals) - min(vals) > 20.0:
            print(f"  L{key[1]:02d} {key[0]:>24s} " + " ".join(f"{v:7.1f}" for v in vals))
