"""Resource usage of the built sm_100a kernels (CPU: cuobjdump on the in-tree libjt.so, no GPU needed).
The bench workload's kernel (512^3: the N = 512, radix-32 forward over plain layouts) must not spill: a
register-allocation regression there shows up as local-memory traffic in the hot loop.  Its inverse
may keep a few bytes of stack: with its twiddles in TMEM (tuning.h JT_TWT_INV32) ptxas spills 16 bytes and the
pass is still 0.5 % faster than with the shared-memory twiddle table (profiles/ab_r02zn.txt)."""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1901_07275_b200", "libjt.so")


def res_usage():
    if not shutil.which("cuobjdump") or not os.path.exists(LIB):
        pytest.skip("cuobjdump or libjt.so missing")
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    res, name = {}, None
    for ln in out.splitlines():
        m = re.match(r"\s*Function (\S+):", ln)
        if m:
            name = m.group(1)
            continue
        if name and "REG:" in ln:
            res[name] = {k: int(v) for k, v in re.findall(r"(\w+):(\d+)", ln)}
            name = None
    return res


@pytest.mark.parametrize("direction,inv,pair", [("fwd", 0, 1), ("fwd", 0, 0), ("inv", 1, 0)])
def test_bench_kernels_do_not_spill(direction, inv, pair):
    """(Cfg<N, R, MAXR, INV, WG, PAIR>: the bench's forward is the PAIR kernel; the unpaired forward stays for the
    few-line launches and JT_PAIR=0.)"""
    res = res_usage()
    key = f"{direction}_axis_kernelINS_3CfgILi512ELi32ELi2ELb{inv}ELb0ELb{pair}EEELb0ELb0EE"
    hits = [v for k, v in res.items() if key in k]
    assert len(hits) == 1, key
    r = hits[0]
    assert r["REG"] <= 255 and r["STACK"] <= (0 if direction == "fwd" else 32) and r["LOCAL"] == 0, r


def test_every_axis_kernel_fits_the_register_file():
    res = res_usage()
    kernels = {k: v for k, v in res.items() if "axis_kernel" in k}
    assert len(kernels) > 50
    for k, v in kernels.items():
        assert v["REG"] <= 255, (k, v)
        assert v["STACK"] <= 512, (k, v)  # small spills only (the N > 1024 and MAXR = 4 kernels)
