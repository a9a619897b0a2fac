"""Accuracy of the GPU path against the oracle at every BASELINE config (and the NEXT-row configs), with the
bar of the north star (relative l2 <= 1e-10 forward, round trip <= 1e-10).  Full arrays where the oracle is
fast (<= 256^3, 4096^2), sampled outputs computed one by one by the oracle at 512^3.  With JT_ACCURACY_OUT set,
the per-config errors are written there as JSON (profiles/accuracy_r01.json comes from this test)."""
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

RESULTS = {}


def relerr(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / np.linalg.norm(np.ravel(ref)))


@pytest.mark.parametrize("name", list(si.CONFIGS))
def test_config_accuracy(name):
    c = si.CONFIGS[name]
    shape, a, b = c["n"], c["a"], c["b"]
    pts, kind = si.config_points(c), c.get("kind", 0)
    p = jt.Plan(shape, a, b, c["eps"], points=pts, kind=kind)
    x = si.gaussian(shape, seed=0)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    jt.jt_forward(p.handle, xd, yd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    rec = {"shape": list(shape), "ranks": [p.rank(i) for i in range(len(shape))],
           "k0": [p.info(i)["k0"] for i in range(len(shape))]}
    if np.prod(shape) <= 256 ** 3 or (pts is None and kind == 0 and np.prod(shape) <= 4096 ** 2):
        rec["forward_relerr"] = relerr(y, oracle.forward_ex(x, a, b, pts, kind))
        rec["forward_check"] = "full array"
    else:
        idx = si.sample_indices(shape, 48)
        ref = oracle.forward_at(x, a, b, idx)
        rec["forward_relerr"] = relerr(y[tuple(idx.T)], ref)
        rec["forward_check"] = "48 sampled outputs (oracle one by one)"
    assert rec["forward_relerr"] <= 1e-10
    if pts is None and kind == 0:
        zd = torch.empty_like(xd)
        jt.jt_inverse(p.handle, yd, zd)
        torch.cuda.synchronize()
        rec["roundtrip_relerr"] = relerr(zd.cpu().numpy(), x)
        assert rec["roundtrip_relerr"] <= 1e-10
    RESULTS[name] = rec
    out = os.environ.get("JT_ACCURACY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(RESULTS, f, indent=1)
    p.close()
