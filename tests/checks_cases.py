"""Run by tests/test_gpu_dist.py::test_checks_build_parity_and_no_violations with JT_LIB = libjt_checks.so (the
bounds-checked, schedule-fuzzed build, include/jt_debug.h jt_debug_checks): small cases of every kernel family and
schedule against the oracle, each single-GPU case twice (bitwise equal: the fuzzed schedules expose races), then the
violation counter must read zero; finally the negative control.  Prints "CHECKS OK"."""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1901_07275_b200 as jt  # noqa: E402
import seeded_inputs as si  # noqa: E402
from paper_1901_07275_b200.dist import LibSlabPlan  # noqa: E402

TOL = 1e-10


def relerr(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / np.linalg.norm(np.ravel(ref)))


def dev(plan, x, inverse=False, adjoint=False):
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    (jt.jt_adjoint if adjoint else jt.jt_inverse if inverse else jt.jt_forward)(plan.handle, xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def expect_clean(what):
    enabled, count, line = jt.jt_debug_checks()
    assert enabled, "JT_LIB is not the checks build"
    assert count == 0, f"{what}: {count} bounds violations, first at axis_kernels.cuh:{line}"


def single_gpu_cases():
    cases = [((2,), (0.1,), (-0.2,)), ((28,), (0.25,), (-0.3,)), ((100,), (-0.75,), (0.2,)),
             ((512,), (0.25,), (-0.25,)), ((777,), (0.0,), (0.0,)), ((1024,), (0.25,), (-0.3,)),
             ((3000,), (0.2,), (0.2,)), ((4096,), (0.45,), (-0.45,)),
             ((256, 256), (0.1, -0.25), (-0.4, 0.35)), ((33, 7), (0.0, 0.5), (0.0, -0.5)),
             ((17, 2048), (-0.2, 0.7), (0.1, 0.3)), ((64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
             ((5, 130, 9), (0.25, 0.25, 0.25), (-0.25, -0.25, -0.25)), ((128, 96), (0.25, -0.3), (-0.1, 0.4)),
             ((64, 64, 64), (0.1, 0.2, 0.3), (-0.1, -0.2, -0.3)), ((2000, 3), (0.1, 0.2), (0.3, -0.4)),
             # launches of >= 2400 lines on FFT lengths 256 / 512 / 4096: the paired kernels (Cfg::PAIR), forward and
             # inverse, incl. n below the FFT length; the host pipelines mix paired and unpaired chunk launches
             ((2410, 256), (0.35, -0.2), (0.1, 0.3)), ((300, 2403), (0.3, -0.2), (0.2, 0.4)),
             ((4096, 2401), (0.45, 0.25), (-0.45, -0.3))]
    for shape, a, b in cases:
        p = jt.Plan(shape, a, b, 1e-12)
        x = si.gaussian(shape, seed=7)
        y1, y2 = dev(p, x), dev(p, x)  # (the checks build fuzzes the schedule: a race makes the two runs differ)
        assert np.array_equal(y1, y2), f"forward {shape}: two runs differ"
        assert relerr(y1, oracle.forward(x, a, b)) <= TOL, shape
        z1, z2 = dev(p, x, inverse=True), dev(p, x, inverse=True)
        assert np.array_equal(z1, z2), f"inverse {shape}: two runs differ"
        assert relerr(z1, oracle.inverse(x, a, b)) <= TOL, shape
        if len(shape) >= 2:  # the pipelined host paths (row chunks, column blocks)
            assert relerr(p.forward_host(x), oracle.forward(x, a, b)) <= TOL, shape
            assert relerr(p.inverse_host(x), oracle.inverse(x, a, b)) <= TOL, shape
        p.close()
        expect_clean(f"single GPU {shape}")
    # nonuniform random points (cap-3 bins: the MAXR = 3 kernels), clustered points (MAXR = 4), the second kind
    shape, a, b = (96, 80), (0.4, 0.4), (0.4, 0.4)
    pts = [si.points(n, 100 + i) for i, n in enumerate(shape)]
    p = jt.Plan(shape, a, b, 1e-12, points=pts)
    x = si.gaussian(shape, seed=8)
    assert relerr(dev(p, x), oracle.forward_ex(x, a, b, pts, 0)) <= TOL
    assert relerr(dev(p, x, adjoint=True), oracle.adjoint_ex(x, a, b, pts, 0)) <= TOL
    p.close()
    rng = np.random.default_rng(4)  # clustered: half the points in a narrow window
    tc = np.sort(np.concatenate([rng.uniform(0.01, 3.13, 40), rng.uniform(1.0, 1.05, 40)]))
    pc = jt.Plan((80,), (0.2,), (0.2,), 1e-12, points=[tc])
    xc = si.gaussian((80,), seed=9)
    assert relerr(dev(pc, xc), oracle.forward_ex(xc, (0.2,), (0.2,), [tc], 0)) <= TOL
    pc.close()
    q = jt.Plan(shape, a, b, 1e-12, kind=jt.JT_KIND_Q)
    assert relerr(dev(q, x), oracle.forward_ex(x, a, b, None, 1)) <= TOL
    q.close()
    expect_clean("nonuniform / second kind")


def run_ranks(G, fn):
    errs = [None] * G
    out = [None] * G

    def body(g):
        try:
            out[g] = fn(g)
        except BaseException as ex:  # noqa: BLE001
            errs[g] = ex
    th = [threading.Thread(target=body, args=(g,)) for g in range(G)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    for e in errs:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    return out


def distributed_cases():
    for G, shape, a, b in [(2, (64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
                           (4, (96, 64, 33), (0.25, -0.1, 0.0), (-0.25, 0.6, 0.0)),
                           (4, (256, 256), (0.1, -0.25), (-0.4, 0.35))]:
        for flags in (0, jt.JT_DIST_LOWMEM, jt.JT_DIST_NCCL_A2A):
            g = jt.jt_debug_vgroup_create(G, 60000)
            plans = [LibSlabPlan(shape, a, b, 1e-12, vgroup=g, rank=r, flags=flags) for r in range(G)]
            streams = [torch.cuda.Stream() for _ in range(G)]
            x = si.gaussian(shape, seed=9)
            xs = [p.local_input(torch.from_numpy(x)) for p in plans]
            torch.cuda.synchronize()
            ys = run_ranks(G, lambda r: plans[r].forward(xs[r], stream=streams[r]))
            y = np.concatenate([t.cpu().numpy() for t in ys], axis=1)
            assert relerr(y, oracle.forward(x, a, b)) <= TOL, (G, shape, flags)
            zs = run_ranks(G, lambda r: plans[r].inverse(ys[r], stream=streams[r]))
            assert relerr(np.concatenate([t.cpu().numpy() for t in zs], axis=0), x) <= TOL, (G, shape, flags)
            xh = [torch.from_numpy(np.ascontiguousarray(x[p.local_box(0)[0][0]:p.local_box(0)[1][0]])).pin_memory()
                  for p in plans]
            yh = [torch.empty(p.y_shape, dtype=torch.float64).pin_memory() for p in plans]
            run_ranks(G, lambda r: plans[r].forward_host(xh[r], yh[r], stream=streams[r]))
            assert relerr(np.concatenate([t.numpy() for t in yh], axis=1), oracle.forward(x, a, b)) <= TOL
            for p in plans:
                p.close()
            jt.jt_debug_vgroup_destroy(g)
            expect_clean(f"distributed G={G} {shape} flags={flags}")


def negative_control():
    """An axis pass whose output extent is declared one line short: the last line's stores must be counted as
    violations and skipped (the sentinel after the declared extent survives)."""
    shape, a, b = (64, 48), (0.1, 0.2), (0.3, -0.1)
    p = jt.Plan(shape, a, b, 1e-12)
    x = torch.from_numpy(si.gaussian(shape, seed=3)).cuda()
    y = torch.full_like(x, 12345.0)
    total = x.numel()
    jt.jt_debug_axis_pass_lim(p.handle, 1, False, x, y, 64, 1, total, total - 48)  # axis 1: 64 lines of 48
    torch.cuda.synchronize()
    enabled, count, line = jt.jt_debug_checks()
    assert enabled and count > 0 and line > 0, (enabled, count, line)
    yy = y.cpu().numpy()
    assert np.all(yy[-1] == 12345.0), "the stores beyond the declared extent were not skipped"
    ref = oracle.forward_axes(x.cpu().numpy(), a, b, axes=[1])
    assert relerr(yy[:-1], ref[:-1]) <= TOL
    p.close()
    print(f"negative control: {count} violations caught, first at axis_kernels.cuh:{line}")


if __name__ == "__main__":
    torch.cuda.set_device(0)
    assert jt.LIB_PATH.endswith("libjt_checks.so"), jt.LIB_PATH
    expect_clean("start")
    single_gpu_cases()
    distributed_cases()
    negative_control()
    print("CHECKS OK")
