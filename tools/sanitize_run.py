"""Small forward + inverse + adjoint runs of several FFT lengths / kinds for compute-sanitizer (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402

cases = [((64, 40), (0.1, -0.3), (0.2, 0.4), None, 0), ((300,), (0.5,), (-0.2,), None, 0),
         ((16, 512), (0.25, 0.25), (-0.25, -0.25), None, 0), ((8, 1024), (0.2, 0.1), (0.1, 0.0), None, 0),
         ((4, 4096), (0.45, 0.0), (-0.45, 0.0), None, 0), ((48, 33), (0.4, 0.4), (0.4, 0.4), "random", 0),
         ((64, 64), (0.2, -0.4), (-0.2, 0.3), None, 1)]
for shape, a, b, pts, kind in cases:
    points = None if pts is None else [si.points(n, 5 + i) for i, n in enumerate(shape)]
    p = jt.Plan(shape, a, b, 1e-12, points=points, kind=kind)
    x = torch.from_numpy(si.gaussian(shape, 1)).cuda()
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    jt.jt_forward(p.handle, x, y)
    jt.jt_adjoint(p.handle, y, z)
    torch.cuda.synchronize()
    print("ok", shape, kind, pts, flush=True)
