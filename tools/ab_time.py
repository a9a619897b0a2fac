"""A/B timing of several libjt builds on the same box (dev tool; raw ctypes so older builds load too).

    python tools/ab_time.py LIB1.so LIB2.so ... [--configs cfg5_3d_512,cfg4_3d_256,grid:2048x2048] [--reps 20]
                            [--rounds 2]

Each library is loaded in its own subprocess; per config prints forward / inverse ms (CUDA events, mean
of `reps` after 3 warm-ups), libraries interleaved `rounds` times to expose box drift.
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, configs, reps, k0=None):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import seeded_inputs as si
    L = ctypes.CDLL(lib)
    P = ctypes.c_void_p
    L.jt_plan.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_double, ctypes.c_void_p]
    for f in ("jt_forward", "jt_inverse", "jt_adjoint"):
        getattr(L, f).argtypes = [P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.jt_destroy.argtypes = [P]
    out = {}
    for name in configs:
        if name.startswith("grid:"):  # ad hoc grid "grid:2048x2048": (a, b) = (0.25, -0.25) per axis, eps 1e-12
            shp = tuple(int(v) for v in name[5:].split("x"))
            c = {"n": shp, "a": (0.25,) * len(shp), "b": (-0.25,) * len(shp), "eps": 1e-12}
        else:
            c = si.CONFIGS[name]
        d = len(c["n"])
        n = (ctypes.c_int64 * d)(*c["n"])
        a = (ctypes.c_double * d)(*c["a"])
        b = (ctypes.c_double * d)(*c["b"])
        h = P()
        opts = None
        if k0 is not None:  # jt_opts {seed, k0, rmax_init, q, sweeps, device}
            class O(ctypes.Structure):
                _fields_ = [("seed", ctypes.c_uint64), ("k0", ctypes.c_int), ("rmax_init", ctypes.c_int),
                            ("q", ctypes.c_int), ("sweeps", ctypes.c_int), ("device", ctypes.c_int)]
            opts = ctypes.byref(O(0, k0, 0, 3, 2, -1))
        pts = si.config_points(c)
        if pts is None and c.get("kind", 0) == 0:
            assert L.jt_plan(ctypes.byref(h), d, n, a, b, c["eps"], opts) == 0
        else:  # nonuniform / second kind: jt_plan_ex (include/jt.h)
            L.jt_plan_ex.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
            keep = [np.ascontiguousarray(q, dtype=np.float64) for q in pts] if pts is not None else []
            arr = (ctypes.c_void_p * d)(*[q.ctypes.data for q in keep]) if pts is not None else None
            assert L.jt_plan_ex(ctypes.byref(h), d, n, a, b, arr, c.get("kind", 0), c["eps"], opts) == 0
        x = torch.from_numpy(si.gaussian(c["n"], 0)).cuda()
        y = torch.empty_like(x)
        s = torch.cuda.current_stream().cuda_stream
        fns = ("jt_forward", "jt_inverse") if (pts is None and c.get("kind", 0) == 0) else ("jt_forward", "jt_adjoint")
        for fn in fns:
            f = getattr(L, fn)
            for _ in range(3):
                f(h, x.data_ptr(), y.data_ptr(), s)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f(h, x.data_ptr(), y.data_ptr(), s)
            e1.record()
            torch.cuda.synchronize()
            out[f"{name}:{fn[3:]}"] = round(e0.elapsed_time(e1) / reps, 4)
        L.jt_destroy(h)
    print("RESULT " + json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--configs", default="cfg5_3d_512,cfg4_3d_256,cfg3_2d_4096")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--k0", type=int, default=None)
    args = ap.parse_args()
    configs = args.configs.split(",")
    if args.child:
        child(args.libs[0], configs, args.reps, args.k0)
        return
    res = {}
    for rnd in range(args.rounds):
        for lib in args.libs:
            lib_k0 = lib.split("@")
            cmd = [sys.executable, __file__, lib_k0[0], "--child", "--configs", args.configs, "--reps", str(args.reps)]
            if len(lib_k0) > 1:
                cmd += ["--k0", lib_k0[1]]
            p = subprocess.run(cmd, capture_output=True, text=True)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("RESULT ")]
            if not line:
                print(lib, "FAILED", p.stderr[-2000:])
                continue
            r = json.loads(line[0][7:])
            for k, v in r.items():
                res.setdefault(k, {}).setdefault(os.path.basename(lib), []).append(v)
    names = [os.path.basename(l) for l in args.libs]  # LIB.so@K0 runs the library with jt_opts.k0 = K0
    print(f"{'case':28s} " + " ".join(f"{n:>22s}" for n in names))
    for k, d in res.items():
        print(f"{k:28s} " + " ".join(f"{'/'.join(f'{v:.3f}' for v in d.get(n, [])):>22s}" for n in names))


if __name__ == "__main__":
    main()
