"""Registers / spills per kernel from `nvcc -Xptxas -v` output: python tools/ptxas_regs.py PTXAS.txt [REGEX]"""
import re
import subprocess
import sys

txt = open(sys.argv[1]).read().splitlines()
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cur, spill = None, ""
for l in txt:
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur, spill = m.group(1), ""
        continue
    if "spill" in l:
        spill = l.split(":")[-1].strip() if ":" in l else l.strip()
    if "Used" in l and cur:
        dem = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("jtk::", "").replace("(int)", "").replace("(bool)", "")
        dem = dem[:dem.find("(AxisDev")] if "(AxisDev" in dem else dem
        if pat is None or pat.search(dem):
            regs = re.search(r"Used (\d+) registers", l).group(1)
            print(f"{regs:>4} regs  {spill:60s} {dem}")
