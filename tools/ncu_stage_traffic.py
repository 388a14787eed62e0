"""ncu --csv launch list of tools/ncu_levels.py (metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum, with --nvtx) -> the per-stage /
per-level / top-kernel JSON bench.py reads for roofline.traffic.

    python tools/ncu_stage_traffic.py gpurun_out/ncu_levels.csv profiles/r02_ncu_stage_traffic.json
"""
import collections
import csv
import json
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src, errors="replace")) if len(r) > 10]
hdr = rows[0]
ix = {n: i for i, n in enumerate(hdr)}
nvtx_col = next(i for i, n in enumerate(hdr) if "NVTX" in n or "nvtx" in n.lower()) \
    if any("nvtx" in n.lower() for n in hdr) else 4
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ix["ID"]], {"range": re.findall(r"(\w+_L\d\d)", r[nvtx_col]),
                                        "name": r[ix["Kernel Name"]]})
    try:
        v = float(r[ix["Metric Value"]].replace(",", ""))
    except ValueError:
        continue
    unit = r[ix["Metric Unit"]]
    name = r[ix["Metric Name"]]
    if name == "gpu__time_duration.sum":
        v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1e-6)       # -> ms
    else:
        v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    d[name] = v
stages = collections.defaultdict(lambda: {"kernel_ms": 0.0, "dram_bytes": 0.0, "launches": 0})
levels = collections.defaultdict(lambda: {"kernel_ms": 0.0, "dram_bytes": 0.0})
kern = collections.defaultdict(lambda: {"launches": 0, "kernel_ms": 0.0, "dram_bytes": 0.0})
for d in launch.values():
    if not d["range"]:
        continue
    rng = d["range"][-1]
    st = rng.split("_")[0]
    ms = d.get("gpu__time_duration.sum", 0.0)
    by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    for tgt in (stages[st], levels[rng]):
        tgt["kernel_ms"] += ms
        tgt["dram_bytes"] += by
    stages[st]["launches"] += 1
    k = kern[(st, re.sub(r"\(.*", "", d["name"]).replace("void ", ""))]
    k["launches"] += 1
    k["kernel_ms"] += ms
    k["dram_bytes"] += by
top = sorted(({"stage": s, "kernel": n, **v} for (s, n), v in kern.items()),
             key=lambda e: -e["kernel_ms"])[:40]
out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none --nvtx, python tools/ncu_levels.py (c4 operator at 1024^2, "
                 "sequential compress_outer + invert_dense_block, one ID slice); per-launch values "
                 "summed per NVTX range (serialised, cold-cache); tools/ncu_stage_traffic.py",
       "stages": {k: {a: (round(b, 3) if a == "kernel_ms" else int(b)) for a, b in v.items()}
                  for k, v in stages.items()},
       "levels": {k: {"kernel_ms": round(v["kernel_ms"], 3), "dram_bytes": int(v["dram_bytes"])}
                  for k, v in sorted(levels.items())},
       "top_kernels": [{**e, "kernel_ms": round(e["kernel_ms"], 3), "dram_bytes": int(e["dram_bytes"])}
                       for e in top]}
json.dump(out, open(dst, "w"), indent=1)
for k, v in out["stages"].items():
    print(f"{k:8s} {v['kernel_ms']:10.1f} ms  {v['dram_bytes'] / 1e9:9.1f} GB  {v['launches']:6d} launches")
for e in out["top_kernels"][:16]:
    print(f"{e['stage']:6s} {e['kernel'][:52]:52s} {e['launches']:6d} {e['kernel_ms']:9.1f} ms {e['dram_bytes'] / 1e9:8.1f} GB")
