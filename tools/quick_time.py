"""Quick CUDA-event timing of jt_forward / jt_inverse per BASELINE config (dev tool, not the bench)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_07275_b200 as jt
import seeded_inputs as si
res = {}
for name, c in si.CONFIGS.items():
    t0 = time.time(); p = jt.Plan(c["n"], c["a"], c["b"], c["eps"], points=si.config_points(c), kind=c.get("kind", 0)); tp = time.time() - t0
    x = torch.from_numpy(si.gaussian(c["n"], 0)).cuda(); y = torch.empty_like(x)
    for fn in ("fwd", "inv"):
        f = jt.jt_forward if fn == "fwd" else jt.jt_adjoint
        for _ in range(3): f(p.handle, x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps): f(p.handle, x, y)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        npts = int(np.prod(c["n"]))
        res[f"{name}_{fn}"] = dict(ms=round(ms, 4), coeff_per_s=npts / ms * 1e3, ranks=[p.rank(i) for i in range(len(c["n"]))], plan_s=round(tp, 2))
        print(name, fn, res[f"{name}_{fn}"], flush=True)
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/quick_time.json", "w"), indent=1)
