"""One forward + one inverse of a BASELINE config through the C ABI (for ncu captures; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_3d_512"
c = si.CONFIGS[name]
p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
x = torch.from_numpy(si.gaussian(c["n"], 0)).cuda()
y = torch.empty_like(x)
jt.jt_forward(p.handle, x, y)
jt.jt_inverse(p.handle, y, x)
torch.cuda.synchronize()
print("ok", name, [p.rank(i) for i in range(len(c["n"]))])
