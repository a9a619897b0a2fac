"""Dev tool: full-array parity of jt_forward / jt_inverse vs the oracle for one shape."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import oracle  # noqa: E402
import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


shape = tuple(int(v) for v in sys.argv[1].split('x'))
a = (0.25,) * len(shape)
b = (-0.25,) * len(shape)
p = jt.Plan(shape, a, b, 1e-12)
x = si.gaussian(shape, 0)
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)
jt.jt_forward(p.handle, xd, yd)
zd = torch.empty_like(xd)
jt.jt_inverse(p.handle, yd, zd)
torch.cuda.synchronize()
y, z = yd.cpu().numpy(), zd.cpu().numpy()
ref = oracle.forward(x, a, b)
print("forward", rel(y, ref), "roundtrip", rel(z, x), flush=True)
e = np.abs(y - ref)
bad = np.argwhere(e > 1e-9)
print("fwd nbad", len(bad), bad[:12].tolist(), flush=True)
if len(bad):
    ax = [np.unique(bad[:, i]).size for i in range(bad.shape[1])]
    print("distinct per axis", ax, "lines (i0 fixed)?", np.unique(bad[:, 1:], axis=0).shape[0], flush=True)
refi = oracle.inverse(y, a, b)
print("inverse", rel(z, refi))
e = np.abs(z - refi)
bad = np.argwhere(e > 1e-8)
print("nbad", len(bad), bad[:10].tolist())
