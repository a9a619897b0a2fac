"""Build libjt.so in-tree for sm_100a (host plan in g++/OpenMP, kernels + C ABI in nvcc), and its bounds-checked
twin libjt_checks.so (-DJT_CHECKS=1: every kernel index checked, include/jt_debug.h jt_debug_checks).

    python -m paper_1901_07275_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

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


def _run_parallel(cmds, jobs=None):
    """Run the commands, at most `jobs` (default: CPU count) at a time."""
    jobs = jobs or os.cpu_count() or 4
    pending, running = list(cmds), []
    while pending or running:
        while pending and len(running) < jobs:
            cmd = pending.pop(0)
            print("+", " ".join(cmd), flush=True)
            running.append((cmd, subprocess.Popen(cmd)))
        cmd, p = running.pop(0)
        if p.wait() != 0:
            for _, q in running:
                q.kill()
            raise subprocess.CalledProcessError(p.returncode, cmd)


# translation units of the CUDA side: the C ABI (jt_api.cu) and one unit per FFT length (launch_<N>.cu: that
# length's kernel instantiations), largest first so the parallel compile ends sooner
UNITS = ["launch_4096", "launch_512", "launch_2048", "launch_1024", "launch_256", "launch_128", "launch_64",
         "launch_32", "launch_16", "jt_api"]


def build(verbose_ptxas: bool = False, out: str = LIB, defines=(), tag: str = "", checks: bool = True,
          extra=()) -> str:
    """Compile libjt.so (or a variant: `out` path, extra -D `defines`, extra nvcc flags `extra`, object-file `tag`);
    with `checks` (default, only for the default build) also libjt_checks.so.  All translation units compile in
    parallel."""
    nvcc = _nvcc()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    # object files outside the repository (they need not travel to the GPU box with the libraries)
    build_dir = os.environ.get("JT_BUILD_DIR") or os.path.join(tempfile.gettempdir(), "jt_build")
    os.makedirs(build_dir, exist_ok=True)
    plan_o = os.path.join(build_dir, "plan.o")
    # (compressed fatbins: one translation unit per FFT length repeats the line tables, 45 -> ~15 MB per library)
    base = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "-Xfatbin=-compress-all", *inc, *extra]
    if verbose_ptxas:
        base += ["-Xptxas", "-v"]
    variants = [(out, tag, [f"-D{d}" for d in defines])]
    if checks and out == LIB and not defines and not extra:
        variants.append((LIB_CHECKS, "_checks", ["-DJT_CHECKS=1"]))
    cmds = [["g++", "-std=c++17", "-O2", "-fPIC", "-fopenmp", *inc, "-c", os.path.join(CSRC, "plan.cpp"), "-o", plan_o]]
    objs = {}
    for lib, tg, dfl in variants:
        objs[lib] = []
        for u in UNITS:
            obj = os.path.join(build_dir, f"{u}{tg}.o")
            objs[lib].append(obj)
            cmds.append([nvcc, *base, *dfl, "-c", os.path.join(CSRC, f"{u}.cu"), "-o", obj])
    _run_parallel(cmds)
    for lib, _, _ in variants:
        _run([nvcc, *ARCH, "-shared", "-o", lib, *objs[lib], plan_o, "-Xcompiler", "-fopenmp", "-lgomp"])
    return out


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv, checks="--no-checks" not in sys.argv)
