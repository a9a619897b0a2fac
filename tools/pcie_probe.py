"""Host<->device copy bandwidth on the GPU box (context for bench.py's e2e number): pinned host
buffers of the 512^3 step's size, H2D alone, D2H alone, and both directions at once on two streams.
usage: python tools/pcie_probe.py [OUT.json] [GiB]"""
import json
import sys

import torch

nbytes = int(float(sys.argv[2] if len(sys.argv) > 2 else 1.0) * (1 << 30))
h_in = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def d2h_pitched():
    # the e2e pipeline's D2H pattern (jt_api.cu transform_host): 8 column blocks of a (512, cols) row-major array,
    # each one cudaMemcpy2DAsync (cuda-python; torch's strided host copies do not use it)
    from cuda.bindings import runtime as rt
    rows = 512
    cols = (nbytes // 8) // rows
    st = torch.cuda.current_stream().cuda_stream
    for c in range(8):
        c0, c1 = cols * c // 8, cols * (c + 1) // 8
        off = c0 * 8
        rt.cudaMemcpy2DAsync(h_out.data_ptr() + off, cols * 8, d_out.data_ptr() + off, cols * 8, (c1 - c0) * 8, rows,
                             rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, st)


res = {"bytes": nbytes}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("d2h_pitched", d2h_pitched)):
    ms = timed(fn)
    res[name + "_ms"] = ms
    res[name + "_GBps"] = (2 if name == "both" else 1) * nbytes / ms / 1e6
print(json.dumps(res))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=1)
