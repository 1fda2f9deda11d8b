"""Per (kernel, grid size) breakdown of an ncu launch list (gpu__time_duration)."""
import collections
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("(anonymous namespace)::", "")
    rows.append((name, r.get("Grid Size", ""), float(r["Metric Value"].replace(",", ""))))
agg = collections.defaultdict(list)
for n, g, v in rows:
    agg[(n, g)].append(v)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for (n, g), vs in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:top]:
    print(f"{n[-44:]:44s} grid {g:>16s} n {len(vs):5d} avg {sum(vs)/len(vs)/1e3:9.2f} us total {sum(vs)/1e6:8.2f} ms")
