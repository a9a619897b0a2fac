"""GPU parity of SURVEY.md §8(f) NEXT-1 (nonuniform forward) and NEXT-3 (second-kind Q~) transforms: the
CUDA path through the C ABI (jt_plan_ex / jt_forward / jt_adjoint) against the oracle (oracle.forward_ex /
oracle.adjoint_ex), element by element on the same seeded inputs; bar: relative l2 <= 1e-10 (north star).
The same fused axis-pass kernels run these plans: only the host plan differs."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si
from test_next import random_points

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1901_07275_b200 as jt

TOL = 1e-10


def relerr(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / np.linalg.norm(np.ravel(ref)))


def run(fn, plan, x_np):
    x = torch.from_numpy(x_np).cuda()
    y = torch.empty_like(x)
    fn(plan.handle, x, y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


CASES = [  # shape, a, b, which axes are nonuniform (clustered?), kind
    ((512,), (0.4,), (0.4,), [False], 0),
    ((1000,), (0.25,), (-0.3,), [True], 0),
    ((333,), (-0.6,), (0.2,), [False], 1),
    ((64, 96), (0.4, 0.1), (0.4, -0.2), [False, None], 0),
    ((128, 128), (0.2, -0.3), (0.3, 0.25), [True, False], 0),
    ((40, 48, 33), (0.4, 0.4, 0.4), (0.4, 0.4, 0.4), [False, False, False], 0),
    ((32, 24, 40), (0.1, -0.5, 0.3), (0.2, 0.5, -0.1), [None, None, None], 1),
    ((24, 32, 20), (0.3, 0.0, -0.2), (-0.1, 0.0, 0.6), [True, None, False], 1),
]


@pytest.mark.parametrize("shape,a,b,nu,kind", CASES)
def test_forward_and_adjoint_vs_oracle(shape, a, b, nu, kind):
    pts = [None if c is None else random_points(n, 100 + i, c) for i, (n, c) in enumerate(zip(shape, nu))]
    p = jt.Plan(shape, a, b, 1e-12, points=pts, kind=kind)
    x = si.gaussian(shape, seed=21)
    y = run(jt.jt_forward, p, x)
    assert relerr(y, oracle.forward_ex(x, a, b, pts, kind)) <= TOL
    z = run(jt.jt_adjoint, p, x)
    assert relerr(z, oracle.adjoint_ex(x, a, b, pts, kind)) <= TOL
    if all(q is None for q in pts) and kind == 0:
        return
    with pytest.raises(jt.JTError) as ei:  # not orthogonal: no inverse
        run(jt.jt_inverse, p, x)
    assert ei.value.status == jt.JT_ERR_ARG


def test_uniform_adjoint_equals_inverse():
    shape, a, b = (64, 80), (0.1, -0.3), (0.2, 0.4)
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=3)
    np.testing.assert_array_equal(run(jt.jt_adjoint, p, x), run(jt.jt_inverse, p, x))


def test_nonuniform_3d_256_paper_setting_sampled():
    """The paper's nonuniform experiment setting (a = b = 0.4 on every axis; random points),
    at 256^3: sampled outputs computed one by one by the oracle."""
    n = 256
    shape, a, b = (n, n, n), (0.4,) * 3, (0.4,) * 3
    pts = [random_points(n, 7 + i) for i in range(3)]
    p = jt.Plan(shape, a, b, 1e-12, points=pts)
    x = si.gaussian(shape, seed=0)
    y = run(jt.jt_forward, p, x)
    mats = [oracle.phi_points(pts[i], n, a[i], b[i]) for i in range(3)]
    idx = si.sample_indices(shape, 64)
    ref = np.array([np.einsum("i,j,k,ijk->", mats[0][i0], mats[1][i1], mats[2][i2], x) for i0, i1, i2 in idx])
    got = y[tuple(idx.T)]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= TOL
