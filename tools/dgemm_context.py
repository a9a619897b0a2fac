"""Context only (SURVEY.md §8(d) comparator ii): one axis pass as a dense cuBLAS DGEMM (the definition
Y = Phi X, 2 n flop/point) at the BASELINE axis lengths, vs the factored fused axis pass of libjt.
The product is the factored method; this quantifies where it pays off on B200's FP64 tensor cores."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1901_07275_b200 as jt  # noqa: E402

out = {}
for n, lines, a, b in [(256, 256 * 256, 0.2, -0.2), (512, 512 * 512, 0.25, -0.25), (1024, 16384, 0.25, -0.3),
                       (4096, 4096, 0.45, -0.45)]:
    phi = torch.randn(n, n, dtype=torch.float64, device="cuda")
    x = torch.randn(n, lines, dtype=torch.float64, device="cuda")
    for _ in range(3):
        y = phi @ x
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y = phi @ x
    e1.record()
    torch.cuda.synchronize()
    t_gemm = e0.elapsed_time(e1) / 10
    p = jt.Plan(n, a, b, 1e-12)
    xl = torch.randn(lines, n, dtype=torch.float64, device="cuda")  # lines contiguous along the axis
    yl = torch.empty_like(xl)
    for _ in range(3):
        jt.jt_axis_pass(p.handle, 0, False, xl, yl, lines, 1)
    torch.cuda.synchronize()
    # the fused pass over `lines` contiguous lines: (outer = lines, n, inner = 1)
    e0.record()
    for _ in range(10):
        jt.jt_axis_pass(p.handle, 0, False, xl, yl, lines, 1)
    e1.record()
    torch.cuda.synchronize()
    t_fast = e0.elapsed_time(e1) / 10
    out[n] = {"lines": lines, "dgemm_ms": round(t_gemm, 4), "dgemm_tflops": 2 * n * n * lines / t_gemm / 1e9,
              "factored_ms": round(t_fast, 4), "rank": p.rank(), "k0": p.info()["k0"]}
    print(n, out[n], flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/dgemm_context.json", "w"), indent=1)
