"""Factor persistence: save a factorization once, solve with it in later runs
(SURVEY.md §8(f) row 4).

The reference has two related mechanisms: `_Spill` (solver_dense.py:37-55)
backs large blocks by `.npy` memmaps in a temporary directory, and the 1-D HSS
debug blob `to_blob`/`from_blob` (hss1d/ops.py:218-267) writes a JSON
structure header plus the blocks.  Here the factors live in HBM as per-level
batches, so the file is a dump of those batches, not of per-box blocks:

    [0:8)    magic  b"VIEFB200"
    [8:16)   u64 little-endian length of the JSON header
    [16:..)  JSON header, then zero padding to a 4096-byte boundary
    ...      storages, each starting on a 4096-byte boundary

The header records the problem (spec, quadrature rule, options, eps, grid side,
leaf size, level slices -- as plain JSON values, see `_problem_json`), every storage (file offset, byte
count, whether it lives on the device) and, per tree level, every attribute
of the level's state: tensors and numpy arrays as (storage, offset, shape,
stride, dtype) views -- aliasing between tensors (the root's block-form factors
are views of level buffers) is preserved exactly -- and plain scalars/tuples
as JSON.  Device storages stream through two pinned staging buffers in
`_CHUNK`-byte pieces (the copy of one overlaps the file I/O of the other), so
saving/loading the ~50 GB 1024^2 factorization needs no host copy of the
whole thing.

Loading rebuilds the host objects (grid, tree, assembler) from the problem
description and uploads the storages; `load(...).apply(f)` is bitwise
identical to the saved object's `apply(f)` (tests).  Nothing in the file is
executed: the header is JSON decoded into the package's own frozen dataclasses
(field presets and kernel families are validated by their constructors), and
every storage is a raw byte range.
"""

import dataclasses
import json
import os
import struct

import numpy as np
import torch

from . import _lib

MAGIC = b"VIEFB200"
VERSION = 2
_ALIGN = 4096
_CHUNK = 256 << 20

_DT = {torch.float64: "float64", torch.float32: "float32", torch.int64: "int64",
       torch.int32: "int32", torch.int16: "int16", torch.int8: "int8",
       torch.uint8: "uint8", torch.bool: "bool", torch.complex128: "complex128"}
_TD = {v: k for k, v in _DT.items()}


def _align(x):
    return (x + _ALIGN - 1) // _ALIGN * _ALIGN


class _Writer:
    """Collects the storages behind every tensor / array of the state."""

    def __init__(self):
        self.storages = []      # (kind, object) in file order
        self._seen = {}

    def _sid(self, key, kind, obj):
        sid = self._seen.get(key)
        if sid is None:
            sid = self._seen[key] = len(self.storages)
            self.storages.append((kind, obj))
        return sid

    def encode(self, v):
        if v is None or isinstance(v, (bool, int, float, str)):
            return {"t": "py", "v": v}
        if isinstance(v, (np.integer, np.floating, np.bool_)):
            return {"t": "py", "v": v.item()}
        if isinstance(v, torch.Tensor):
            st = v.untyped_storage()
            sid = self._sid(("t", st.data_ptr(), st.device.type), "dev" if v.is_cuda else "host",
                            st)
            return {"t": "tensor", "s": sid, "o": v.storage_offset(), "shape": list(v.shape),
                    "stride": list(v.stride()), "dtype": _DT[v.dtype]}
        if isinstance(v, np.ndarray):
            a = np.ascontiguousarray(v)
            sid = self._sid(("n", id(v)), "nd", a)
            return {"t": "nd", "s": sid, "shape": list(a.shape), "dtype": a.dtype.str}
        if isinstance(v, (tuple, list)):
            return {"t": "tuple" if isinstance(v, tuple) else "list",
                    "v": [self.encode(x) for x in v]}
        if isinstance(v, dict):
            return {"t": "dict", "v": [[self.encode(k), self.encode(x)] for k, x in v.items()]}
        # lean / 1-D HSS block storage of a level (compressed_store.py): L.hss = (hF, hE)
        from .hss1d import Hss1dBatch, _HLevel
        if isinstance(v, Hss1dBatch):
            return {"t": "hss1d", "v": {k: self.encode(getattr(v, k))
                                        for k in ("nb", "n", "tree", "depth", "lv", "dense")}}
        if isinstance(v, _HLevel):
            return {"t": "hlevel", "v": {k: self.encode(getattr(v, k))
                                         for k in _HLevel.__slots__ if hasattr(v, k)}}
        raise TypeError(f"cannot persist a {type(v).__name__}")


def _level_state(L):
    # attributes starting with "_" are caches rebuilt on demand
    return {k: v for k, v in vars(L).items() if not k.startswith("_")}


def _nbytes(kind, obj):
    return obj.nbytes() if kind in ("dev", "host") else obj.nbytes


class _Stager:
    """Two pinned staging buffers on a private stream: the device<->host copy
    of one chunk overlaps the file I/O of the other."""

    def __init__(self, nbytes):
        n = min(_CHUNK, max(nbytes, 1))
        self.buf = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.ev = [torch.cuda.Event(), torch.cuda.Event()]
        self.stream = torch.cuda.Stream()
        self.busy = [False, False]

    def write(self, f, src):
        """src: uint8 CUDA tensor -> file, chunk by chunk."""
        n = src.numel()
        chunks = [(lo, min(n, lo + _CHUNK)) for lo in range(0, n, _CHUNK)]

        def issue(c):
            lo, hi = chunks[c]
            with torch.cuda.stream(self.stream):
                self.buf[c % 2][:hi - lo].copy_(src[lo:hi], non_blocking=True)
                self.ev[c % 2].record(self.stream)

        self.stream.wait_stream(torch.cuda.current_stream())
        if chunks:
            issue(0)
        for c, (lo, hi) in enumerate(chunks):
            if c + 1 < len(chunks):
                issue(c + 1)
            self.ev[c % 2].synchronize()
            f.write(self.buf[c % 2][:hi - lo].numpy().data)

    def read(self, f, dst):
        """file -> dst (uint8 CUDA tensor), chunk by chunk."""
        n = dst.numel()
        for c, lo in enumerate(range(0, n, _CHUNK)):
            hi = min(n, lo + _CHUNK)
            i = c % 2
            if self.busy[i]:
                self.ev[i].synchronize()          # the buffer's previous upload is done
            f.readinto(self.buf[i][:hi - lo].numpy().data)
            with torch.cuda.stream(self.stream):
                dst[lo:hi].copy_(self.buf[i][:hi - lo], non_blocking=True)
                self.ev[i].record(self.stream)
            self.busy[i] = True

    def finish(self):
        self.stream.synchronize()
        self.busy = [False, False]


def _write_storage(f, kind, obj, stage):
    if kind == "nd":
        f.write(memoryview(obj).cast("B"))
        return
    src = torch.empty(0, dtype=torch.uint8, device=obj.device).set_(obj)
    if kind == "host":
        f.write(src.numpy().data)
        return
    stage.write(f, src)


def _field_json(f):
    return {"name": f.name, "params": [[k, v] for k, v in f.params]}


def _problem_json(pb):
    """problem dict (spec, quad, opts, ...) -> JSON-safe dict."""
    sp = pb["spec"]
    out = {"spec": {"family": sp.family, "k": float(sp.k),
                    "a_field": _field_json(sp.a_field), "b_field": _field_json(sp.b_field),
                    "c_field": _field_json(sp.c_field)},
           "quad": pb["quad"].order,
           "opts": dataclasses.asdict(pb["opts"])}
    for k in ("eps", "n_side", "n_max", "ti_mode", "apriori"):
        if k in pb:
            out[k] = pb[k]
    sl = pb.get("level_slices")
    out["level_slices"] = None if sl is None else [[int(lv), list(v)] for lv, v in sl.items()]
    return out


def _problem_from_json(d):
    from .config import SolverOptions
    from .kernels import Field, KernelSpec, QuadratureCorrection, make_field

    def field(e):
        f = make_field(e["name"], **{k: v for k, v in e["params"]})  # validates the preset
        assert isinstance(f, Field)
        return f

    sp = d["spec"]
    spec = KernelSpec(str(sp["family"]), k=float(sp["k"]), a_field=field(sp["a_field"]),
                      b_field=field(sp["b_field"]), c_field=field(sp["c_field"]))
    fields = {f.name for f in dataclasses.fields(SolverOptions)}
    opts = SolverOptions(**{k: v for k, v in d["opts"].items() if k in fields})
    out = {"spec": spec, "quad": QuadratureCorrection(str(d["quad"])), "opts": opts,
           "eps": float(d["eps"]), "n_side": int(d["n_side"]), "n_max": int(d["n_max"])}
    if "ti_mode" in d:
        out["ti_mode"] = bool(d["ti_mode"])
    if d.get("apriori") is not None:
        out["apriori"] = int(d["apriori"])
    sl = d.get("level_slices")
    out["level_slices"] = None if sl is None else {int(lv): tuple(int(x) for x in v)
                                                   for lv, v in sl}
    return out


def write_state(path, problem, kind, levels):
    """Write `levels` (list of per-level attribute dicts or None) and the
    `problem` description (spec, quad, opts, eps, n_side, n_max, level_slices)
    to `path`."""
    w = _Writer()
    enc_levels = [None if st is None else {k: w.encode(v) for k, v in st.items()}
                  for st in levels]
    sizes = [_nbytes(k, o) for k, o in w.storages]
    header = {"version": VERSION, "kind": kind,
              "problem": _problem_json(problem) if "spec" in problem else problem,
              "levels": enc_levels, "storages": []}
    # offsets depend on the header length; iterate until it is stable
    hlen = 0
    while True:
        off = _align(16 + hlen)
        header["storages"] = []
        for (k, _), nb in zip(w.storages, sizes):
            header["storages"].append({"offset": off, "nbytes": nb, "device": k == "dev"})
            off = _align(off + nb)
        blob = json.dumps(header).encode()
        if len(blob) == hlen:
            break
        hlen = len(blob)
    need_stage = any(k == "dev" for k, _ in w.storages)
    stage = _Stager(max(sizes + [1])) if need_stage else None
    if need_stage:
        torch.cuda.synchronize()
    tmp = f"{path}.tmp{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", hlen))
        f.write(blob)
        for (k, o), s in zip(w.storages, header["storages"]):
            f.seek(s["offset"])
            _write_storage(f, k, o, stage)
        f.truncate(_align(f.tell()))
    os.replace(tmp, path)


def read_header(path):
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError(f"{path}: not a vief_b200 factor file")
        (hlen,) = struct.unpack("<Q", f.read(8))
        header = json.loads(f.read(hlen).decode())
    if header.get("version") != VERSION:
        raise ValueError(f"{path}: factor file version {header.get('version')}, "
                         f"this build reads {VERSION}")
    return header


def read_state(path, device):
    """-> (kind, problem, levels) with device storages uploaded to `device`."""
    header = read_header(path)
    device = torch.device(device)
    stor = []
    with open(path, "rb") as f:
        dev_sizes = [s["nbytes"] for s in header["storages"] if s["device"]]
        stage = None
        if dev_sizes and device.type == "cuda":
            with torch.cuda.device(device):
                stage = _Stager(max(dev_sizes))
        for s in header["storages"]:
            f.seek(s["offset"])
            nb = s["nbytes"]
            if s["device"]:
                buf = torch.empty(nb, dtype=torch.uint8, device=device)
                if stage is None:
                    f.readinto(buf.numpy().data)
                else:
                    stage.read(f, buf)
            else:
                buf = np.empty(nb, dtype=np.uint8)
                f.readinto(buf.data)
            stor.append(buf)
        if stage is not None:
            stage.finish()

    def decode(e):
        t = e["t"]
        if t == "py":
            return e["v"]
        if t in ("tuple", "list"):
            v = [decode(x) for x in e["v"]]
            return tuple(v) if t == "tuple" else v
        if t == "nd":
            return stor[e["s"]].view(np.dtype(e["dtype"])).reshape(e["shape"])
        if t == "tensor":
            base = stor[e["s"]]
            if isinstance(base, np.ndarray):
                base = torch.from_numpy(base)
            typed = base.view(_TD[e["dtype"]])
            return torch.as_strided(typed, e["shape"], e["stride"], e["o"])
        if t == "dict":
            return {decode(k): decode(x) for k, x in e["v"]}
        if t == "hss1d":
            from .hss1d import Hss1dBatch
            d = {k: decode(x) for k, x in e["v"].items()}
            h = Hss1dBatch(d["nb"], d["n"], d["tree"], device)
            h.lv, h.dense = d["lv"], d["dense"]
            return h
        if t == "hlevel":
            from .hss1d import _HLevel
            h = _HLevel()
            for k, x in e["v"].items():
                setattr(h, k, decode(x))
            return h
        raise ValueError(f"bad entry type {t!r}")

    levels = [None if st is None else {k: decode(v) for k, v in st.items()}
              for st in header["levels"]]
    pb = header["problem"]
    return header["kind"], (_problem_from_json(pb) if "spec" in pb else pb), levels


# ---------------------------------------------------------------------------
# solver objects

def _problem_of(H):
    sl = None
    if H.sharded:
        sl = {L.lv: tuple(int(x) for x in L.sl) for L in H.levels if L is not None}
    return {"spec": H.spec, "quad": H.quad, "opts": H.opts, "eps": H.eps,
            "n_side": H.grid.n_side, "n_max": H.tree.n_max, "level_slices": sl}


def save(obj, path):
    """Write an `Hss2dMatrix`, a `DenseBlockInverse` or a `CompressedInverse`
    (either path; dense, lean or 1-D HSS block storage) to `path`.  The factors
    stay where they are (HBM)."""
    from .solver_compressed import CompressedInverse
    from .solver_dense import DenseBlockInverse, Hss2dMatrix
    if isinstance(obj, CompressedInverse):
        if obj.ti_mode and any(getattr(L, "ti", False) for L in obj.dense_matvec_source.levels
                               if L is not None):
            raise NotImplementedError("saving TI-mode (shared-record) factors is not supported")
        kind, H = "CompressedInverse", obj.dense_matvec_source
    elif isinstance(obj, DenseBlockInverse):
        kind, H = "DenseBlockInverse", obj.H
    elif isinstance(obj, Hss2dMatrix):
        kind, H = "Hss2dMatrix", obj
    else:
        raise TypeError(f"cannot save a {type(obj).__name__}")
    torch.cuda.synchronize(H.device)
    problem = _problem_of(H)
    if kind == "CompressedInverse":
        problem["ti_mode"] = obj.ti_mode
    if getattr(H, "apriori", None):   # the finite-k_cut path: the a-priori band width
        problem["apriori"] = int(H.apriori)
    write_state(path, problem, kind,
                [None if L is None else _level_state(L) for L in H.levels])


def load(path, device=None):
    """Read a file written by `save`; returns an object of the saved type with
    its factors resident on `device` (default: the current CUDA device)."""
    from .kernels import Grid
    from .solver_compressed import CompressedInverse
    from .solver_dense import DenseBlockInverse, Hss2dMatrix
    from .tree import build_tree
    _lib.require_cuda()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    kind, pb, levels = read_state(path, device)
    grid = Grid(pb["n_side"])
    tree = build_tree(grid, pb["n_max"])
    with torch.cuda.device(device):
        H = Hss2dMatrix(pb["spec"], grid, tree, pb["eps"], pb["opts"], pb["quad"],
                        level_slices=pb["level_slices"])
    H.apriori = pb.get("apriori")
    for L, st in zip(H.levels, levels):
        if (L is None) != (st is None):
            raise ValueError(f"{path}: level layout does not match the rebuilt tree")
        if L is not None:
            for k, v in st.items():
                setattr(L, k, v)
    if kind == "Hss2dMatrix":
        return H
    inv = DenseBlockInverse(H)
    if kind == "DenseBlockInverse":
        return inv
    ci = CompressedInverse(pb["spec"], grid, tree, pb["eps"], pb["opts"], pb["quad"],
                           pb.get("ti_mode", False))
    ci.dense_delegate, ci.dense_matvec_source = inv, H
    if H.apriori:   # the compressed path's factor views (factor_of, record_count) read these
        from .solver_compressed import ensure_apriori_skeletons
        ensure_apriori_skeletons(pb["spec"], tree, pb["opts"])   # (a support mask is not recorded)
        ci.factors = inv
        ci.hss_levels = sum(getattr(L, "hss_kind", None) == "hss" for L in H.levels if L is not None)
    return ci
