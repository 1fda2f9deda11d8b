"""Per-launch DRAM traffic and duration of the kernels in an ncu --set full report,
as JSON (profiles/): python ncu_traffic.py rep.ncu-rep out.json [p] [dim]"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
p = int(sys.argv[3]) if len(sys.argv) > 3 else None
dim = int(sys.argv[4]) if len(sys.argv) > 4 else None
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
     "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6,
         "us": 1e-3, "ms": 1.0, "ns": 1e-6}
res = []
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    e = {"kernel": name.split("::")[-1].replace("(int)", ""),
         "grid": r[h.index("Grid Size")]}
    for m in M:
        if m not in h:
            continue
        i = h.index(m)
        v = float(r[i].replace(",", "")) if r[i] else None
        u = units[i]
        if m.startswith("dram__bytes"):
            v = v * scale.get(u, 1)
        if m == "gpu__time_duration.sum":
            v = v * scale.get(u, 1)  # -> ms
            m = "ms"
        e[m] = v
    if "dram__bytes_read.sum" in e and "dram__bytes_write.sum" in e:
        e["dram_bytes"] = e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"]
    res.append(e)
json.dump({"report": rep, "p": p, "dim": dim, "note": "one ncu --set full capture (cold caches, serialised "
           "launches, --clock-control none); per-launch figures", "kernels": res}, open(out, "w"), indent=1)
for e in res:
    print(f"{e['kernel'][:40]:40s} {e['grid']:>14s} {e.get('ms', 0) * 1e3:9.1f} us  dram {e.get('dram_bytes', 0) / 1e6:9.1f} MB")
