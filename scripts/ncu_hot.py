"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report.
python ncu_hot.py rep.ncu-rep KERNEL_REGEX LAUNCH_SKIP [N]"""
import csv
import io
import subprocess
import sys

rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
ist = h.index("Warp Stall Sampling (All Samples)")
isrc = h.index("Source")
tot = sum(int(r[ist] or 0) for r in body)
print("samples", tot, "sass lines", len(body))
for r in sorted(body, key=lambda r: -int(r[ist] or 0))[:n]:
    print(f"{int(r[ist]):6d} {100.0 * int(r[ist]) / max(tot, 1):5.1f}%  {r[0][-5:]}  {r[isrc].strip()[:100]}")
