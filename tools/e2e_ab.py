"""e2e A/B: a stream of jt_forward_host_async calls (bench.py's e2e loop) with the library named by JT_LIB (dev tool).

    JT_LIB=... python tools/e2e_ab.py [config] [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_3d_512"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = si.CONFIGS[name]
p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
xs = [torch.from_numpy(si.gaussian(c["n"], seed=k)).pin_memory().numpy() for k in range(2)]
ys = [torch.empty(c["n"], dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
s = torch.cuda.current_stream()
for k in range(2):
    p.forward_host_async(xs[k], ys[k], s)
p.wait_host()
res = []
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        p.forward_host_async(xs[k % 2], ys[k % 2], s)
    p.wait_host()
    res.append((time.perf_counter() - t0) * 1e3 / steps)
yd = torch.empty(c["n"], dtype=torch.float64, device="cuda")
jt.jt_forward(p.handle, torch.from_numpy(xs[1]).cuda(), yd)
torch.cuda.synchronize()
err = float(np.linalg.norm(ys[1] - yd.cpu().numpy()) / np.linalg.norm(ys[1]))
print(f"{os.path.basename(jt.LIB_PATH)} {name} e2e ms/step {['%.2f' % v for v in res]} rel-diff vs device {err:.1e}")
