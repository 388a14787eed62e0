"""Device memory over repeated factorize()+solve steps (allocated / reserved by
torch, device free memory)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1303_5466_b200 import Grid, KernelSpec, SolverOptions, build_tree, make_field, CELL
from paper_1303_5466_b200 import solver_dense as sd
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = KernelSpec("laplace2d", b_field=make_field("centre_bump", scale=math.pi / 2), c_field=make_field("one"))
grid = Grid(n)
opts = SolverOptions(eps=1e-10, leaf_size=64, k_cut=None)
F = torch.randn((n * n, 256), dtype=torch.float64, device="cuda")
G = 1 << 30
def rep(tag):
    torch.cuda.synchronize()
    free, tot = torch.cuda.mem_get_info()
    print(f"{tag:>12s}: alloc {torch.cuda.memory_allocated()/G:6.1f}  reserved {torch.cuda.memory_reserved()/G:6.1f}  "
          f"peak {torch.cuda.max_memory_allocated()/G:6.1f}  device free {free/G:6.1f} / {tot/G:6.1f} GiB", flush=True)
rep("start")
for i in range(6):
    tree = build_tree(grid, 64)
    H, inv = sd.factorize(spec, grid, tree, 1e-10, opts, CELL)
    rep(f"factor {i}")
    X = inv.apply(F)
    rep(f"solve {i}")
    del H, inv, X
    rep(f"freed {i}")
