"""Compact per-kernel table of an ncu --set full report: python ncu_table.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "launch__occupancy_limit_registers", "smsp__average_warp_latency_per_inst_issued.ratio"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
cols = ["ID", "Kernel Name", "Grid Size"] + [m for m in M if m in h]
idx = [h.index(c) for c in cols]
short = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
         "launch__registers_per_thread": "reg", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
         "smsp__inst_executed.sum": "inst", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
         "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem%",
         "launch__occupancy_limit_registers": "lim_reg", "smsp__average_warp_latency_per_inst_issued.ratio": "lat"}
print(" | ".join(short.get(c, c) for c in cols))
print(" | ".join(r[1][i] for i in idx))
for row in r[2:]:
    v = [row[i] for i in idx]
    v[1] = v[1].split("(DevMesh")[0].split("(int")[0].replace("void ldgb::<unnamed>::", "")[:30] + \
        (row[idx[1]].split("(int)")[1].split(">")[0] if "(int)" in row[idx[1]] else "")
    print(" | ".join(v))
