"""Phase trace of the latency-bound configs (dev tool): with a library built with -DJT_PHASES=1 (JT_LIB=...), every
CTA's thread 0 prints clock64 phase boundaries of its first batch (axis_kernels.cuh `Phases`).  This runs a few
calls per config and direction and summarises the LAST call: per launch, the kernel's globaltimer span and the
median / max over CTAs of each phase end (microseconds at the clock the box reports).

    JT_LIB=paper_1901_07275_b200/libjt_phases.so python tools/phases.py [config ...] > out.txt
Phases: 1 start (TMEM, twiddles, ring issue)  2 input loads + state  3 batch-start W V block  4 rank terms
        5 stores  6 TMEM free  7-9 cluster reduction (first barrier, remote loads + sums + stores, second barrier)
        10 reduction done  11 end.
"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(name, fn_name, calls=4):
    import torch
    import paper_1901_07275_b200 as jt
    import seeded_inputs as si
    libc = ctypes.CDLL(None)
    c = si.CONFIGS[name]
    p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
    x = torch.from_numpy(si.gaussian(c["n"], 0)).cuda()
    y = torch.empty_like(x)
    fn = getattr(jt, fn_name)
    for i in range(calls):
        libc.printf(b"CALL %d\n", ctypes.c_int(i))
        libc.fflush(None)
        fn(p.handle, x, y)
        torch.cuda.synchronize()
        libc.fflush(None)


def summarise(text, mhz):
    calls = text.split("CALL ")
    last = calls[-1].splitlines()[1:]
    rows = []
    for ln in last:
        if not ln.startswith("PH "):
            continue
        t = ln.split()
        rec = dict(kind=t[1], n=t[2], cta=int(t[3][3:]), sm=t[4], terms=int(t[5][5:]), g0=int(t[7]), g1=int(t[9]),
                   d=[int(v) for v in t[11:22]])
        rows.append(rec)
    if not rows:
        return ["(no PH lines)"]
    rows.sort(key=lambda r: r["g0"])
    # one launch per (direction, FFT length, line stride): the passes of a call overlap under PDL
    launches = {}
    for r in rows:
        launches.setdefault((r["kind"], r["n"]), []).append(r)
    launches = sorted(launches.values(), key=lambda ls: min(q["g0"] for q in ls))
    out = []
    t_first = launches[0][0]["g0"]
    for ls in launches:
        g0 = min(r["g0"] for r in ls) - t_first
        g1 = max(r["g1"] for r in ls) - t_first
        out.append(f"launch {ls[0]['kind']} {ls[0]['n']}: {len(ls)} CTAs, terms {sorted(set(r['terms'] for r in ls))}, "
                   f"globaltimer {g0 / 1e3:.2f} .. {g1 / 1e3:.2f} us (CTA starts spread "
                   f"{(max(r['g0'] for r in ls) - min(r['g0'] for r in ls)) / 1e3:.2f} us)")
        names = ["start", "loads", "W V", "terms", "stores", "TMEM free", "cl.bar1", "cl.loads", "cl.bar2", "reduce",
                 "end"]
        for i in range(len(ls[0]["d"])):
            vals = sorted(r["d"][i] for r in ls if r["d"][i] > 0)
            if vals:
                out.append(f"   phase {i + 1:2d} {names[i]:9s} end: median {vals[len(vals) // 2] / mhz:7.2f} us, max {vals[-1] / mhz:7.2f} us")
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        sys.exit(0)
    import torch
    mhz = torch.cuda.get_device_properties(0).clock_rate / 1e3 if hasattr(torch.cuda.get_device_properties(0),
                                                                          "clock_rate") else 1965.0
    names = sys.argv[1:] or ["cfg1_1d_1024", "cfg2_2d_256"]
    for name in names:
        for fn in ("jt_forward", "jt_inverse"):
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", name, fn], capture_output=True,
                               text=True)
            print(f"== {name} {fn} (rc {r.returncode})")
            if r.returncode:
                print(r.stderr[-2000:])
            for ln in summarise(r.stdout, mhz):
                print(ln)
            sys.stdout.flush()
