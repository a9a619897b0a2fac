import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle, paper_1901_07275_b200 as jt, seeded_inputs as si
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
shape = (64, n, n) if len(sys.argv) < 3 else tuple(int(v) for v in sys.argv[2].split('x'))
a = (0.25,) * 3; b = (-0.25,) * 3
p = jt.Plan(shape, a, b, 1e-12)
x = si.gaussian(shape, 0)
phis = [oracle.phi(shape[i], a[i], b[i]) for i in range(3)]
xd = torch.from_numpy(x).cuda()
for ax in range(3):
    outer = int(np.prod(shape[:ax])); inner = int(np.prod(shape[ax+1:]))
    for inv, inplace in ((False, False), (True, False), (False, True)):
        yd = xd.clone() if inplace else torch.empty_like(xd)
        src = yd if inplace else xd
        (jt.jt_inverse_axis if inv else jt.jt_forward_axis)(p.handle, ax, src, yd, outer, inner)
        torch.cuda.synchronize()
        y = yd.cpu().numpy()
        M = phis[ax].T if inv else phis[ax]
        ref = np.moveaxis(np.tensordot(M, x, axes=([1], [ax])), 0, ax)
        err = np.abs(y - ref)
        bad = np.argwhere(err > 1e-9 * np.abs(ref).max())
        print(f"axis {ax} {'inv' if inv else 'fwd'} inplace={inplace} rel {rel(y, ref):.3e} nbad {len(bad)} first {bad[:3].tolist()}", flush=True)
