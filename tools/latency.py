"""Latency of the small (launch-bound) configs: host enqueue cost per call, back-to-back stream time per call,
and the same call replayed from a CUDA graph (GPU time without host overhead).  Dev tool.

    python tools/latency.py OUT.json [config ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402

names = sys.argv[2:] or ["cfg1_1d_1024", "cfg2_2d_256"]
out = {}
reps = 200
for name in names:
    c = si.CONFIGS[name]
    p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
    x = torch.from_numpy(si.gaussian(c["n"], 0)).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    for fn_name in ("jt_forward", "jt_inverse"):
        fn = getattr(jt, fn_name)
        with torch.cuda.stream(s):
            for _ in range(5):
                fn(p.handle, x, y, s)
            s.synchronize()
            launches = jt.jt_last_launches(p)
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                fn(p.handle, x, y, s)
            host_us = (time.perf_counter() - t0) / reps * 1e6
            e1.record(s)
            s.synchronize()
            stream_us = e0.elapsed_time(e1) / reps * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            fn(p.handle, x, y, s)
        with torch.cuda.stream(s):
            for _ in range(5):
                g.replay()
            s.synchronize()
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
            s.synchronize()
            graph_us = e0.elapsed_time(e1) / reps * 1e3
        # the graph replays compute the same result
        y_ref = torch.empty_like(y)
        fn(p.handle, x, y_ref, s)
        s.synchronize()
        ok = bool(torch.equal(y, y_ref))
        out[f"{name}:{fn_name[3:]}"] = {"host_us_per_call": round(host_us, 2), "stream_us_per_call": round(stream_us, 2),
                                        "graph_us_per_call": round(graph_us, 2), "kernels_per_call": launches,
                                        "graph_result_equal": ok}
        print(name, fn_name, out[f"{name}:{fn_name[3:]}"], flush=True)
    p.close()
json.dump(out, open(sys.argv[1], "w"), indent=1)
