"""SURVEY.md §8(f) NEXT-2 (grids beyond the configs' sizes) and the "maximum sizes" edge case: the largest cube
one B200 holds, 2048^3 fp64 (8.6e9 coefficients, 68.7 GB per copy, element offsets past 2^32).  The fused build
needs only the caller's input and output arrays (O(n^d) memory; the paper's MATLAB apply keeps O(r n^d)),
so forward and inverse run in 2 x 68.7 GB.

The check holds at any size and is exact up to rounding: the operator is the Kronecker product
of the per-axis matrices (eq:TJ3), so for a rank-one input alpha = beta (x) gamma (x) delta the forward
output is the outer product of the three 1D transforms Phi_0 beta, Phi_1 gamma, Phi_2 delta, which the oracle
computes (oracle.forward on each vector).  The whole output array is compared, plane by plane on the device,
against that outer product (relative l2 <= 1e-10, north star); then the inverse of the output is compared the
same way against beta (x) gamma (x) delta (round trip).  Different (a, b) per axis make an axis mix-up visible.

Skipped when the GPU has less free memory than the two arrays need (JT_CAPACITY_N selects another n; with
JT_CAPACITY_OUT set the errors and timings are written there as JSON, e.g. profiles/capacity_r01.json)."""
import json
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1901_07275_b200 as jt

A = (0.25, -0.4, 0.1)
B = (-0.25, 0.3, 0.2)


def _outer_relerr(arr, f0, f1, f2):
    """Relative l2 distance of the (n0, n1, n2) device array from f0 (x) f1 (x) f2, plane by plane."""
    plane = torch.outer(f1, f2)
    num = torch.zeros((), dtype=torch.float64, device=arr.device)
    den = torch.zeros((), dtype=torch.float64, device=arr.device)
    for i in range(arr.shape[0]):
        ref = plane * f0[i]
        num += torch.sum((arr[i] - ref) ** 2)
        den += torch.sum(ref ** 2)
    return float(torch.sqrt(num / den))


def test_largest_cube_rank_one():
    n = int(os.environ.get("JT_CAPACITY_N", "2048"))
    shape = (n, n, n)
    need = 2 * 8 * n ** 3
    free, _ = torch.cuda.mem_get_info()
    if free < need + (4 << 30):
        pytest.skip(f"needs {need / 1e9:.1f} GB free, {free / 1e9:.1f} GB available")
    vecs = [si.gaussian((n,), seed=40 + i) for i in range(3)]
    fwd1 = [oracle.forward(v, A[i], B[i]) for i, v in enumerate(vecs)]  # Phi_i v_i (oracle)
    d_vecs = [torch.from_numpy(v).cuda() for v in vecs]
    d_fwd = [torch.from_numpy(v).cuda() for v in fwd1]

    p = jt.Plan(shape, A, B, 1e-12)
    x = torch.einsum("i,j,k->ijk", *d_vecs)  # alpha = beta (x) gamma (x) delta
    y = torch.empty_like(x)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    jt.jt_forward(p.handle, x, y)
    ev[1].record()
    torch.cuda.synchronize()
    e_fwd = _outer_relerr(y, *d_fwd)
    ev[2].record()
    jt.jt_inverse(p.handle, y, x)  # overwrite alpha: the reference is the rank-one outer product
    ev[3].record()
    torch.cuda.synchronize()
    e_rt = _outer_relerr(x, *d_vecs)
    rec = {"shape": list(shape), "a": list(A), "b": list(B), "eps": 1e-12,
           "ranks": [p.rank(i) for i in range(3)], "k0": [p.info(i)["k0"] for i in range(3)],
           "device_bytes_in_out": need, "forward_relerr": e_fwd, "roundtrip_relerr": e_rt,
           "forward_ms": ev[0].elapsed_time(ev[1]), "inverse_ms": ev[2].elapsed_time(ev[3]),
           "check": "rank-one input; whole output vs the outer product of the oracle's 1D transforms",
           "note": "first call on the plan (cold: includes TMEM/ring setup); timings are context, not bench values"}
    out = os.environ.get("JT_CAPACITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)
    del x, y
    p.close()
    torch.cuda.empty_cache()
    assert e_fwd <= 1e-10, rec
    assert e_rt <= 1e-10, rec
