"""Registers / spills per kernel from a ptxas -v log: python regs.py build/ldg_obj/X.ptxas.log"""
import re
import subprocess
import sys

cur = None
for line in open(sys.argv[1]).read().splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        d = subprocess.run(["cu++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = d.split("(DevMesh")[0].split("(int")[0].split("(long")[0].replace("ldgb::(anonymous namespace)::", "")
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:45s} regs {m.group(1)}")
    if "spill" in line and " 0 bytes spill stores" not in line:
        print("   SPILL", line.strip())
