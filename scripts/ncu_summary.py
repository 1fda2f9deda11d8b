"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
per-kernel launch counts, total time and share of the profiled range."""
from __future__ import annotations

import csv
import re
import sys
from collections import defaultdict


def main(path: str):
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        rows.append((name, val * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"ldgb::\(anonymous namespace\)::", "", short)
        agg[short][0] += 1
        agg[short][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total / 1e3:.3f} ms of kernel time")
    print(f"{'kernel':60s} {'launches':>9s} {'total us':>12s} {'share':>7s} {'avg us':>9s}")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {n:9d} {us:12.1f} {100 * us / total:6.1f}% {us / n:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
