"""Repeat-determinism probe (dev tool): run a forward / inverse many times and report bitwise mismatches, their size,
parity against the oracle and (checks build) bounds violations.  JT_LIB selects the library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402

ALL = [((3000,), (0.2,), (0.2,)), ((4096,), (0.45,), (-0.45,)), ((2000, 3), (0.1, 0.2), (0.3, -0.4)),
       ((1024,), (0.25,), (-0.3,)), ((2048,), (-0.3,), (0.6,)), ((512, 4096), (0.1, 0.45), (0.2, -0.45)),
       ((8, 4096), (0.1, 0.45), (0.2, -0.45)), ((600, 4096), (0.1, 0.45), (0.2, -0.45))]
sel = [int(v) for v in sys.argv[1:]]
cases = [ALL[i] for i in sel] if sel else ALL
for shape, a, b in cases:
    p = jt.Plan(shape, a, b, 1e-12)
    x = torch.from_numpy(si.gaussian(shape, seed=7)).cuda()
    for fn in (jt.jt_forward, jt.jt_inverse):
        outs = []
        for _ in range(12):
            y = torch.empty_like(x)
            fn(p.handle, x, y)
            outs.append(y)
        torch.cuda.synchronize()
        ref = (oracle.forward if fn is jt.jt_forward else oracle.inverse)(x.cpu().numpy(), a, b)
        errs = [float(np.linalg.norm(o.cpu().numpy() - ref) / np.linalg.norm(ref)) for o in outs]
        mism = sum(not torch.equal(outs[0], o) for o in outs[1:])
        md = max(float((outs[0] - o).abs().max()) for o in outs[1:])
        try:
            ck = jt.jt_debug_checks()
        except Exception:
            ck = None
        print(shape, fn.__name__, "mismatching runs", mism, "max diff %.2e" % md, "relerr range %.1e..%.1e" % (min(errs), max(errs)),
              "launches", jt.jt_last_launches(p), "checks", ck, flush=True)
    p.close()
