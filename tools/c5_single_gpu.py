"""Config c5's problem size (Laplace VIE, 2048^2 = 4.2 M unknowns, eps 1e-10,
1 RHS) on ONE B200: compressed path (a-priori skeletons, k_cut = 64) with the
low-memory schedule -- every level converted to 1-D HSS / lean storage as soon
as its parent is factored, the source blocks freed as they are consumed.
Prints times, resident bytes and the true residual (FFT operator).

    python tools/c5_single_gpu.py [--n 2048] [--nrhs 1] [--frac 0.95]
"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# growing segments instead of fixed blocks: at ~160 of 178 GB the caching allocator's
# fragmentation (tens of GB reserved but unusable) is what runs out first
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import numpy as np
import torch
import paper_1303_5466_b200 as P
from paper_1303_5466_b200 import solver_dense as sd
from paper_1303_5466_b200.solver_compressed import ensure_apriori_skeletons
from paper_1303_5466_b200.verify import FFTOperator

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--frac", type=float, default=0.92)
ap.add_argument("--storage", default="hss1d")
ap.add_argument("--trace", action="store_true")
ap.add_argument("--kcut", type=int, default=64, help="0: the pivoted-ID path (k_cut = None)")
a = ap.parse_args()
torch.cuda.set_per_process_memory_fraction(a.frac)   # an over-commit raises here, not on the box
spec = P.KernelSpec("laplace2d", b_field=P.make_field("centre_bump", scale=math.pi / 2),
                    c_field=P.make_field("one"))
grid = P.Grid(a.n)
opts = P.SolverOptions(eps=1e-10, leaf_size=64, k_cut=a.kcut or None)


def sync_t():
    torch.cuda.synchronize()
    return time.time()


t0 = sync_t()
tree = P.build_tree(grid, 64)
H = sd.Hss2dMatrix(spec, grid, tree, 1e-10, opts, P.CELL)
if a.kcut:
    H.apriori = ensure_apriori_skeletons(spec, tree, opts)
t1 = sync_t()
t2 = sync_t()
mem_c = torch.cuda.max_memory_allocated()
if a.trace:
    from paper_1303_5466_b200 import compressed_store as cs
    _cl = cs.compact_level
    def _traced(H_, L_, *aa, **kw):
        r = _cl(H_, L_, *aa, **kw)
        print(f"level {L_.lv}: {r}, allocated {torch.cuda.memory_allocated() / 1e9:.1f} GB, "
              f"peak {torch.cuda.max_memory_allocated() / 1e9:.1f} GB, t {time.time() - t2:.1f} s",
              file=sys.stderr, flush=True)
        return r
    cs.compact_level = _traced
    # synchronised wall time per phase (compression / inversion / storage conversion / cache release)
    from paper_1303_5466_b200 import _lib as lib
    phase = {}
    def _timed(mod, name, key):
        fn = getattr(mod, name)
        def w(*aa, **kw):
            torch.cuda.synchronize(); t = time.time()
            r = fn(*aa, **kw)
            torch.cuda.synchronize()
            lv = next((x.lv for x in aa if hasattr(x, "lv")), -1)
            phase.setdefault(lv, {}).setdefault(key, 0.0)
            phase[lv][key] += time.time() - t
            return r
        setattr(mod, name, w)
    _timed(sd, "_compress_level", "compress")
    _timed(sd, "_invert_level", "invert")
    _timed(cs, "compact_level", "convert")
    _timed(lib, "release_memory_if_low", "release")
    import atexit
    atexit.register(lambda: print("phase seconds per level: " + json.dumps(
        {k: {a: round(b, 3) for a, b in v.items()} for k, v in sorted(phase.items())}), file=sys.stderr))
# each level is compressed just before it is inverted: one level's sources resident at a time
inv = sd.invert_dense_block(H, free_source=True, storage=a.storage, compress=True)
t3 = sync_t()
mem_f = torch.cuda.max_memory_allocated()
torch.cuda.empty_cache()
F = torch.randn(grid.n, a.nrhs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
X = inv.apply(F)
t4 = sync_t()
X = inv.apply(F)
t5 = sync_t()
op = FFTOperator(spec, grid, P.CELL, "cuda")
res = float(((F - op.matvec(X)).norm(dim=0) / F.norm(dim=0)).max())
kinds = {L.lv: getattr(L, "hss_kind", "dense") for L in H.levels if L is not None}
print(json.dumps({"n_side": a.n, "N": grid.n, "nrhs": a.nrhs, "storage": a.storage, "k_cut": a.kcut or None,
                  "tree_s": t1 - t0, "compress_invert_convert_s": t3 - t2,
                  "solve_first_s": t4 - t3, "solve_s": t5 - t4, "true_residual_fft": res,
                  "factor_bytes": inv.nbytes(), "peak_alloc_compress": mem_c,
                  "peak_alloc_factor": mem_f, "resident_after": torch.cuda.memory_allocated(),
                  "level_storage": kinds}))
