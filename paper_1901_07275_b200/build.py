"""Build libjt.so in-tree for sm_100a (host plan in g++/OpenMP, kernels + C ABI in nvcc), and its bounds-checked
twin libjt_checks.so (-DJT_CHECKS=1: every kernel index checked, include/jt_debug.h jt_debug_checks).

    python -m paper_1901_07275_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libjt.so")
LIB_CHECKS = os.path.join(HERE, "libjt_checks.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _run_parallel(cmds):
    procs = []
    for cmd in cmds:
        print("+", " ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)


def build(verbose_ptxas: bool = False, out: str = LIB, defines=(), tag: str = "", checks: bool = True) -> str:
    """Compile libjt.so (or a variant: `out` path, extra -D `defines`, object-file `tag`); with `checks` (default,
    only for the default build) also libjt_checks.so, compiled in parallel."""
    nvcc = _nvcc()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    build_dir = os.path.join(HERE, "_build")
    os.makedirs(build_dir, exist_ok=True)
    plan_o = os.path.join(build_dir, "plan.o")
    _run(["g++", "-std=c++17", "-O2", "-fPIC", "-fopenmp", *inc, "-c", os.path.join(CSRC, "plan.cpp"),
          "-o", plan_o])
    base = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", *inc]
    if verbose_ptxas:
        base += ["-Xptxas", "-v"]
    api_o = os.path.join(build_dir, f"jt_api{tag}.o")
    jobs = [(out, api_o, [f"-D{d}" for d in defines])]
    if checks and out == LIB and not defines:
        jobs.append((LIB_CHECKS, os.path.join(build_dir, "jt_api_checks.o"), ["-DJT_CHECKS=1"]))
    _run_parallel([[nvcc, *base, *dfl, "-c", os.path.join(CSRC, "jt_api.cu"), "-o", obj] for _, obj, dfl in jobs])
    for lib, obj, _ in jobs:
        _run([nvcc, *ARCH, "-shared", "-o", lib, obj, plan_o, "-Xcompiler", "-fopenmp", "-lgomp"])
    return out


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv, checks="--no-checks" not in sys.argv)
