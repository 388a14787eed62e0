"""Key metrics of every launch in an ncu report (.ncu-rep), with units:
duration, DRAM bytes, DMMA / FP64 pipe utilisation, warps active, registers,
grid, DRAM throughput.  python tools/ncu_report.py <file.ncu-rep> ..."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
     "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
SHORT = ["time", "dram_rd", "dram_wr", "tensor%", "dmma_inst%", "fp64%", "warps%", "regs", "grid",
         "dram%"]
for f in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ix = {n: i for i, n in enumerate(h)}
    print(f"== {f}")
    for r in rows[2:]:
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")[:40]
        cells = []
        for m, s in zip(M, SHORT):
            if m in ix:
                cells.append(f"{s}={r[ix[m]]}{units[ix[m]]}")
        print(f"{name:40s} " + " ".join(cells))
