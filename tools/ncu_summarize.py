"""Summarise an ncu --csv launch list with NVTX ranges (tools/ncu_levels.py):
per range and kernel name: launches, device time, DRAM bytes, FP64-pipe
activity.  Usage: python tools/ncu_summarize.py gpurun_out/ncu_L01.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {n: i for i, n in enumerate(hdr)}
launch = collections.OrderedDict()
for r in rows[1:]:
    key = r[ix["ID"]]
    d = launch.setdefault(key, {"range": re.findall(r":(\w+_L\d\d):", r[ix[hdr[4]]]),
                                "name": r[ix["Kernel Name"]]})
    v = r[ix["Metric Value"]].replace(",", "")
    try:
        d[r[ix["Metric Name"]]] = float(v)
    except ValueError:
        pass
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for d in launch.values():
    rng = d["range"][-1] if d["range"] else "?"
    name = re.sub(r"\(.*", "", d["name"]).replace("void ", "")[:48]
    a = agg[(rng, name)]
    a["n"] += 1
    a["ns"] += d.get("gpu__time_duration.sum", 0.0)
    a["bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a["fp64_inst"] += d.get("sm__inst_executed_pipe_fp64.sum", 0.0)
    a["pipe_x_ns"] += d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * \
        d.get("gpu__time_duration.sum", 0.0)
tot = collections.defaultdict(lambda: [0.0, 0.0])
print(f"{'range':10s} {'kernel':48s} {'n':>6s} {'ms':>9s} {'GB':>8s} {'GB/s':>7s} {'fp64%':>6s}")
for (rng, name), a in sorted(agg.items(), key=lambda kv: (kv[0][0], -kv[1]["ns"])):
    tot[rng][0] += a["ns"]
    tot[rng][1] += a["bytes"]
    if a["ns"] < 0.005 * 1e6:
        continue
    print(f"{rng:10s} {name:48s} {int(a['n']):6d} {a['ns'] / 1e6:9.3f} {a['bytes'] / 1e9:8.3f} "
          f"{a['bytes'] / max(a['ns'], 1):7.0f} {a['pipe_x_ns'] / max(a['ns'], 1):6.1f}")
print()
for rng, (ns, b) in tot.items():
    print(f"{rng:10s} total {ns / 1e6:9.3f} ms (serialised, cold)  DRAM {b / 1e9:8.3f} GB")
