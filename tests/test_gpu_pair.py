"""GPU parity of the paired forward kernels (Cfg::PAIR; DESIGN.md §6 "Two real rank terms per FFT"; eq:oneJ,
PAPER.md:610, applied with a factorisation of eq:approxA whose v'_l are real) against the CPU oracle, and of the
unpaired forward kernels of the same FFT lengths (JT_PAIR=0 at plan time), which the library still uses for the
few-line launches, the inverse and the transpose.  Same bar as tests/test_gpu.py: relative l2 <= 1e-10."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1901_07275_b200 as jt

TOL = 1e-10
MIN_LINES = 2400  # csrc/tuning.h JT_PAIR_MIN_LINES
PAIR_N = (256, 512, 2048, 4096)  # FFT lengths with paired kernels (csrc/launch.cuh pair_length)


def fft_length(n):
    """The plan's FFT length: the power of two >= max(n, 16) (R18)."""
    N = 16
    while N < n:
        N *= 2
    return N


def relerr(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / np.linalg.norm(np.ravel(ref)))


def fwd(p, x):
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    jt.jt_forward(p.handle, xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


# shapes whose axes of FFT length 256 / 512 / 2048 / 4096 are transformed in launches of >= MIN_LINES lines (paired kernels),
# with ragged line counts (not multiples of the CTA's line tile), every axis position, other axis lengths mixed in, and
# axis lengths below their FFT length (n = 2403 -> N = 4096, 200 -> 256, 300 -> 512: zero-padded v, sparser bins)
CASES = [((512, 2403), (0.25, 0.1), (-0.25, -0.3)),
         ((2501, 512), (0.3, -0.45), (0.2, 0.45)),
         ((50, 512, 49), (0.2, 0.0, -0.4), (-0.2, 0.0, 0.3)),
         ((256, 2410), (0.35, -0.2), (0.1, 0.3)),
         ((61, 256, 41), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
         ((4096, 2401), (0.45, 0.25), (-0.45, -0.3)),
         ((2405, 4096), (0.1, 0.0), (-0.1, 0.0)),
         ((200, 300, 41), (0.3, -0.2, 0.1), (0.2, 0.4, -0.3)),
         ((2048, 2405), (-0.3, 0.2), (0.6, 0.1)),
         ((2409, 2000), (0.15, 0.4), (-0.35, -0.4))]


@pytest.mark.parametrize("shape,a,b", CASES)
def test_paired_forward_vs_oracle(shape, a, b, monkeypatch):
    x = si.gaussian(shape, seed=11)
    idx = np.stack([np.random.default_rng(5).integers(0, s, 96) for s in shape], axis=1)
    ref = oracle.forward_at(x, a, b, idx)
    sel = tuple(idx[:, i] for i in range(len(shape)))
    p = jt.Plan(shape, a, b, 1e-12)
    paired_axes = [i for i in range(len(shape)) if jt.jt_debug_pair_factors(p.handle, i) is not None]
    # (every eligible axis of these cases pairs -- checked on the GPU box, r03i; an axis whose nodes do not fit two per
    # half-integer bin may keep only its unpaired set, so the test insists on eligibility and on at least one)
    eligible = [i for i, n in enumerate(shape) if fft_length(n) in PAIR_N]
    assert paired_axes and set(paired_axes) <= set(eligible)
    for i in paired_axes:  # fewer FFTs than rank terms
        assert jt.jt_debug_pair_factors(p.handle, i)[1].shape[0] < p.rank(i)
    # at least one paired axis is transformed in a launch large enough to use the paired kernels
    assert any(int(np.prod(shape)) // shape[i] >= MIN_LINES for i in paired_axes)
    y = fwd(p, x)
    assert relerr(y[sel], ref) <= TOL
    # the inverse (its large launches: the transposed paired operator) undoes the forward, and matches the oracle
    yd = torch.from_numpy(y).cuda()
    zd = torch.empty_like(yd)
    jt.jt_inverse(p.handle, yd, zd)
    torch.cuda.synchronize()
    assert relerr(zd.cpu().numpy(), x) <= TOL
    xd = torch.from_numpy(x).cuda()
    jt.jt_inverse(p.handle, xd, zd)
    torch.cuda.synchronize()
    iref = oracle.inverse_at(x, a, b, idx)
    z = zd.cpu().numpy()
    assert relerr(z[sel], iref) <= TOL
    p.close()
    # the unpaired kernels on the same input: same values to the plan's eps
    monkeypatch.setenv("JT_PAIR", "0")
    q = jt.Plan(shape, a, b, 1e-12)
    assert all(jt.jt_debug_pair_factors(q.handle, i) is None for i in range(len(shape)))
    y0 = fwd(q, x)
    jt.jt_inverse(q.handle, xd, zd)
    torch.cuda.synchronize()
    q.close()
    assert relerr(y0[sel], ref) <= TOL
    assert relerr(y, y0) <= 1e-11
    assert relerr(zd.cpu().numpy(), z) <= 1e-11


def test_paired_forward_full_compare():
    """Element by element over the whole output (several CTA batches and a ragged tail of lines)."""
    shape, a, b = (2437, 512), (0.1, 0.25), (-0.3, -0.25)
    x = si.gaussian(shape, seed=3)
    p = jt.Plan(shape, a, b, 1e-12)
    assert jt.jt_debug_pair_factors(p.handle, 1) is not None
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    jt.jt_forward_axis(p.handle, 1, xd, yd, shape[0], 1, None)  # the 512 axis alone: 2437 lines
    torch.cuda.synchronize()
    ref = x @ oracle.phi(512, a[1], b[1]).T
    assert relerr(yd.cpu().numpy(), ref) <= TOL
    err_rows = np.linalg.norm(yd.cpu().numpy() - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err_rows.max() <= TOL
    # deterministic: a second run is bit-identical
    y2 = torch.empty_like(xd)
    jt.jt_forward_axis(p.handle, 1, xd, y2, shape[0], 1, None)
    torch.cuda.synchronize()
    assert torch.equal(yd, y2)
    # the paired inverse pass of the same axis, element by element against the oracle's transpose product
    jt.jt_inverse_axis(p.handle, 1, xd, y2, shape[0], 1, None)
    torch.cuda.synchronize()
    iref = x @ oracle.phi(512, a[1], b[1])
    assert relerr(y2.cpu().numpy(), iref) <= TOL
    assert (np.linalg.norm(y2.cpu().numpy() - iref, axis=1) / np.linalg.norm(iref, axis=1)).max() <= TOL
    p.close()


def test_few_line_launches_stay_unpaired():
    """Launches below JT_PAIR_MIN_LINES lines run the unpaired kernels (term split): same results as JT_PAIR=0."""
    shape, a, b = (256, 256), (0.1, -0.25), (-0.4, 0.35)
    x = si.gaussian(shape, seed=0)
    p = jt.Plan(shape, a, b, 1e-12)
    y = fwd(p, x)
    p.close()
    assert relerr(y, oracle.forward(x, a, b)) <= TOL
