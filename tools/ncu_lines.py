"""Attribute ncu warp-stall samples and executed instructions of one kernel to CUDA source lines.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX LIB.so [launch_skip] [top]

ncu's CSV source page has no SASS->line correlation, so this joins it with `nvdisasm -g` of the same
library (the .so that was profiled: copy it next to the report on the GPU box).  Rows are matched by
offset from the kernel's first instruction.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def sass_rows(rep, kregex, skip):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kregex,
                          "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    kname = next(csv.reader([lines[0]]))[1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    data = []
    for r in rows[1:]:
        if r and r[0] == "Address":  # a second copy of the listing follows: keep the first
            break
        if len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return kname, data


def line_map(lib, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
        sec = None
        cur_line = None
        m = {}
        for ln in dis.splitlines():
            if ln.startswith("//---------------------") and ".text." in ln:
                sec = ln.split(".text.")[1].split()[0]
                continue
            if sec is None or not re.search(mangled_hint, sec):
                continue
            mm = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
            if mm:
                cur_line = f"{os.path.basename(mm.group(1))}:{mm.group(2)}"
                continue
            mi = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if mi and cur_line:
                m.setdefault(sec, {})[int(mi.group(1), 16)] = cur_line
        if m:
            return m
    return {}


def main(rep, kregex, lib, skip=0, top=40):
    kname, rows = sass_rows(rep, kregex, skip)
    # mangled-name hint: template args of Cfg<N, R, MAXR>
    cfg = re.search(r"Cfg<([^>]*)>", kname)
    nums = re.findall(r"\(int\)(\d+)", cfg.group(1))
    cbools = re.findall(r"\(bool\)(\d)", cfg.group(1))                 # Cfg's INV [, WG]
    kbools = re.findall(r"\(bool\)(\d)", kname[cfg.end():].split(">(")[0])  # the kernel's SPLIT, TSPLIT
    base = "fwd_axis_kernel" if "fwd_axis" in kname else "inv_axis_kernel"
    hint = base + r"INS_3CfgILi" + r"ELi".join(nums) + "E"
    if cbools:
        hint += "".join("Lb" + b + "E" for b in cbools) + "EE" + "".join("Lb" + b + "E" for b in kbools) + "E"
    maps = line_map(lib, hint)
    if not maps:
        print("no line map for", hint)
        return
    sec, lm = next(iter(maps.items()))
    a0 = int(rows[0]["Address"], 16)

    def f(d, k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    agg = defaultdict(lambda: defaultdict(float))
    tot = 0.0
    for d in rows:
        off = int(d["Address"], 16) - a0
        line = lm.get(off, "?")
        s = f(d, "Warp Stall Sampling (All Samples)")
        tot += s
        a = agg[line]
        a["samples"] += s
        a["inst"] += f(d, "Instructions Executed")
        for k in ("stall_wait", "stall_long_sb", "stall_short_sb", "stall_math", "stall_mio", "stall_barrier",
                  "stall_selected", "stall_not_selected"):
            a[k] += f(d, k)
    print(kname[:120])
    print(f"{'line':28s} {'stall%':>6s} {'warp_inst':>12s}  wait  lsb  ssb  math  mio  bar  sel")
    for line, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        s = max(a["samples"], 1)
        print(f"{line:28s} {100*a['samples']/tot:6.1f} {a['inst']:12.0f} " +
              " ".join(f"{100*a[k]/s:4.0f}" for k in ("stall_wait", "stall_long_sb", "stall_short_sb", "stall_math",
                                                        "stall_mio", "stall_barrier", "stall_selected")))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0,
         int(sys.argv[5]) if len(sys.argv) > 5 else 40)
