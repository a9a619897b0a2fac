"""Build libjt.so in-tree for sm_100a (host plan in g++/OpenMP, kernels + C ABI in nvcc).

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
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose_ptxas: bool = False, out: str = LIB, defines=(), tag: str = "") -> str:
    """Compile libjt.so (or a variant: `out` path, extra -D `defines`, object-file `tag`)."""
    nvcc = _nvcc()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    build_dir = os.path.join(HERE, "_build")
    os.makedirs(build_dir, exist_ok=True)
    plan_o = os.path.join(build_dir, "plan.o")
    api_o = os.path.join(build_dir, f"jt_api{tag}.o")
    _run(["g++", "-std=c++17", "-O2", "-fPIC", "-fopenmp", *inc, "-c", os.path.join(CSRC, "plan.cpp"),
          "-o", plan_o])
    flags = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", *inc, *[f"-D{d}" for d in defines]]
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    _run([nvcc, *flags, "-c", os.path.join(CSRC, "jt_api.cu"), "-o", api_o])
    _run([nvcc, *ARCH, "-shared", "-o", out, api_o, plan_o, "-Xcompiler", "-fopenmp", "-lgomp"])
    return out


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv)
