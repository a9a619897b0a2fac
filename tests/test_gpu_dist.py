"""GPU parity of the LIBRARY's distributed slab transform at G = 2, 4, 8 ranks on one B200 (SURVEY.md §8(a) row A7,
§8(e)).

The G ranks are virtual (include/jt_debug.h): each is a real distributed plan of libjt.so (jt_debug_plan_virtual =
jt_plan_dist_ex without NCCL), driven by its own host thread and CUDA stream, running the product schedule
(transform_dist / the distributed transform_host: the axis passes writing and reading the chunk-major all-to-all
layouts, pipelined in row chunks with `ostride > outer`); only the all-to-all itself is an in-process exchange
(one cudaMemcpyAsync per peer block, cross-stream events, a host barrier) instead of grouped ncclSend / ncclRecv.
No kernel waits on another.

Each rank's y-slab (forward) / x-slab (inverse) is compared with the oracle's full transform restricted to the
rank's box (relative l2 <= 1e-10; the independence of the lines that makes the slab split exact is the paper's
"n 2D transforms and n^2 1D transforms", PAPER.md:716-724 eq:TJ3, inverse PAPER.md:731-737 eq:invTJ3), and with the
Python twin dist.SlabPlan (same kernels, same launches) bit for bit.
"""
import threading

import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1901_07275_b200 as jt
    from paper_1901_07275_b200.dist import LibSlabPlan, SlabPlan

TOL = 1e-10

SHAPES = [  # (world, shape, a, b): 3D and 2D, ragged n2, rows per rank from 6 to 256
    (2, (64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
    (4, (64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
    (8, (64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
    (8, (96, 64, 33), (0.25, -0.1, 0.0), (-0.25, 0.6, 0.0)),
    (8, (512, 64, 16), (0.25, 0.25, 0.25), (-0.25, -0.25, -0.25)),
    (2, (256, 256), (0.1, -0.25), (-0.4, 0.35)),
    (4, (256, 256), (0.1, -0.25), (-0.4, 0.35)),
    (8, (256, 256), (0.1, -0.25), (-0.4, 0.35)),
]


def relerr(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / np.linalg.norm(np.ravel(ref)))


def run_ranks(G, fn):
    """fn(rank) on G host threads at once (the virtual group's exchanges need every rank in its call)."""
    out, errs = [None] * G, [None] * G

    def body(g):
        try:
            torch.cuda.set_device(0)
            out[g] = fn(g)
        except BaseException as ex:  # noqa: BLE001 (re-raised below)
            errs[g] = ex
    th = [threading.Thread(target=body, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    return out


class Group:
    """G virtual-rank LibSlabPlans of one shape (closed in the right order)."""

    def __init__(self, G, shape, a, b, flags=0, timeout_ms=120000):
        self.G = G
        self.g = jt.jt_debug_vgroup_create(G, timeout_ms)
        self.plans = [LibSlabPlan(shape, a, b, 1e-12, vgroup=self.g, rank=r, flags=flags) for r in range(G)]
        self.streams = [torch.cuda.Stream() for _ in range(G)]

    def close(self):
        for p in self.plans:
            p.close()
        jt.jt_debug_vgroup_destroy(self.g)


def x_slabs(grp, x):
    return [p.local_input(torch.from_numpy(x)) for p in grp.plans]


def y_slabs(grp, y):
    return [p.local_output(torch.from_numpy(y)) for p in grp.plans]


def gather_y(ys):
    return np.concatenate([y.cpu().numpy() for y in ys], axis=1)


def gather_x(xs):
    return np.concatenate([x.cpu().numpy() for x in xs], axis=0)


MODES = [0, 2]  # the fused exchange (default: blocks stored straight into the peers' receive buffers) and
#                 JT_DIST_NCCL_A2A (the chunked all-to-all pipelined with the axis-1 pass; here the in-process copies)


@pytest.mark.parametrize("flags", MODES)
@pytest.mark.parametrize("world,shape,a,b", SHAPES)
def test_library_slab_transform_virtual_ranks(world, shape, a, b, flags):
    """jt_forward / jt_inverse on G distributed plans (transform_dist: the fused exchange, or the pipelined axis-1 pass
    + all-to-all in row chunks with ostride > outer) against the oracle; the round trip; repeat determinism."""
    grp = Group(world, shape, a, b, flags=flags)
    try:
        x = si.gaussian(shape, seed=11)
        xs = x_slabs(grp, x)
        torch.cuda.synchronize()
        ys = run_ranks(world, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        y = gather_y(ys)
        assert relerr(y, oracle.forward(x, a, b)) <= TOL
        ys2 = run_ranks(world, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        assert all(torch.equal(p, q) for p, q in zip(ys, ys2))  # no atomics, same schedule: bitwise repeatable
        zs = run_ranks(world, lambda g: grp.plans[g].inverse(ys[g], stream=grp.streams[g]))
        assert relerr(gather_x(zs), x) <= TOL
        # inverse alone on independent values
        yv = si.gaussian(shape, seed=12)
        yvs = y_slabs(grp, yv)
        torch.cuda.synchronize()
        ws = run_ranks(world, lambda g: grp.plans[g].inverse(yvs[g], stream=grp.streams[g]))
        assert relerr(gather_x(ws), oracle.inverse(yv, a, b)) <= TOL
        for p in grp.plans:  # one fused pass per axis (+ term-split reductions): kernels only, no copies counted
            assert jt.jt_last_launches(p.handle) >= len(shape)
    finally:
        grp.close()


@pytest.mark.parametrize("flags", MODES)
@pytest.mark.parametrize("world,shape,a,b", [SHAPES[1], SHAPES[4], SHAPES[6]])
def test_library_slab_host_paths_virtual_ranks(world, shape, a, b, flags):
    """The distributed host-buffer paths: jt_forward_host (x-slab copied in row chunks feeding the local passes and
    the chunked exchange, y-slab copied back in column blocks), two jt_forward_host_async calls in flight through the
    staging slots, and jt_inverse_host, against the device-pointer path (equal up to rounding: a row chunk may take
    a term-split launch) and the oracle."""
    grp = Group(world, shape, a, b, flags=flags)
    try:
        x = si.gaussian(shape, seed=21)
        xs = x_slabs(grp, x)
        torch.cuda.synchronize()
        ys = run_ranks(world, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        y_dev = gather_y(ys)
        xh = [x_.cpu().pin_memory() for x_ in xs]
        yh = [[torch.empty(p.y_shape, dtype=torch.float64).pin_memory() for _ in range(3)] for p in grp.plans]

        def host(g):
            p, s = grp.plans[g], grp.streams[g]
            p.forward_host(xh[g], yh[g][0], stream=s)
            for k in (1, 2):
                p.forward_host_async(xh[g], yh[g][k], stream=s)
            p.wait_host()
        run_ranks(world, host)
        for k in range(3):
            yk = np.concatenate([yh[g][k].numpy() for g in range(world)], axis=1)
            assert relerr(yk, y_dev) <= 1e-14, k
        assert relerr(y_dev, oracle.forward(x, a, b)) <= TOL
        zh = [torch.empty(p.x_shape, dtype=torch.float64).pin_memory() for p in grp.plans]
        run_ranks(world, lambda g: grp.plans[g].inverse_host(yh[g][0], zh[g], stream=grp.streams[g]))
        assert relerr(np.concatenate([z.numpy() for z in zh], axis=0), x) <= TOL
        # the pipelined distributed inverse (y-slab row chunks -> axis 2 -> axis 0 -> chunked exchange -> axis 1 per
        # chunk -> x-slab rows copied back): two calls in flight, equal to the device path up to rounding
        ys_dev = [torch.from_numpy(yh[g][0].numpy()).cuda() for g in range(world)]
        torch.cuda.synchronize()
        zs_dev = run_ranks(world, lambda g: grp.plans[g].inverse(ys_dev[g], stream=grp.streams[g]))
        za = [[torch.empty(p.x_shape, dtype=torch.float64).pin_memory() for _ in range(2)] for p in grp.plans]

        def inv_async(g):
            p, s = grp.plans[g], grp.streams[g]
            for k in range(2):
                p.inverse_host_async(yh[g][k], za[g][k], stream=s)
            p.wait_host()
        run_ranks(world, inv_async)
        z_dev = gather_x(zs_dev)
        for k in range(2):
            assert relerr(np.concatenate([za[g][k].numpy() for g in range(world)], axis=0), z_dev) <= 1e-14, k
    finally:
        grp.close()


class _VirtualDist:
    def __init__(self, rank, world):
        self.r, self.w = rank, world

    def get_world_size(self, group=None):
        return self.w

    def get_rank(self, group=None):
        return self.r


@pytest.mark.parametrize("world,shape,a,b", [SHAPES[1], SHAPES[3], SHAPES[7]])
def test_library_schedule_equals_python_twin_bitwise(world, shape, a, b):
    """dist.SlabPlan (the schedule in Python: whole-slab chunk-major passes, a tensor-copy exchange between the
    phases) and the library's pipelined transform_dist issue the same per-line kernel arithmetic: bit-identical
    y-slabs and x-slabs."""
    grp = Group(world, shape, a, b)
    sps = [SlabPlan(shape, a, b, 1e-12, _VirtualDist(g, world)) for g in range(world)]
    try:
        x = si.gaussian(shape, seed=31)
        xs = x_slabs(grp, x)
        torch.cuda.synchronize()
        ys = run_ranks(world, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        c = sps[0].count // world

        def exchange():
            for g in range(world):
                sps[g]._recv.copy_(torch.cat([sps[q]._send[g * c:(g + 1) * c] for q in range(world)]))
        outs = [sp.forward_local(sp.local_input(x)) for sp in sps]
        exchange()
        ys_twin = [sp.forward_finish(o) for sp, o in zip(sps, outs)]
        torch.cuda.synchronize()
        for g in range(world):
            assert torch.equal(ys[g], ys_twin[g]), g
        zs = run_ranks(world, lambda g: grp.plans[g].inverse(ys[g], stream=grp.streams[g]))
        outs = [sp.inverse_local(y) for sp, y in zip(sps, ys_twin)]
        exchange()
        zs_twin = [sp.inverse_finish(o) for sp, o in zip(sps, outs)]
        torch.cuda.synchronize()
        for g in range(world):
            assert torch.equal(zs[g], zs_twin[g]), g
    finally:
        for sp in sps:
            sp.close()
        grp.close()


@pytest.mark.parametrize("world,shape,a,b", [SHAPES[0], SHAPES[2], SHAPES[4], SHAPES[7]])
def test_lowmem_capacity_mode_virtual_ranks(world, shape, a, b):
    """JT_DIST_LOWMEM (NEXT-2 capacity mode): no plan-owned slabs, the input slab is the workspace; same results as
    the pipelined mode (bitwise: the same launches over whole slabs vs row chunks of the same lines) and the oracle;
    the *_host variants through one staging pair."""
    grp = Group(world, shape, a, b, flags=jt.JT_DIST_LOWMEM)
    ref_grp = Group(world, shape, a, b)
    try:
        x = si.gaussian(shape, seed=41)
        xs = x_slabs(grp, x)
        xs_ref = x_slabs(ref_grp, x)
        torch.cuda.synchronize()
        ys = run_ranks(world, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        ys_ref = run_ranks(world, lambda g: ref_grp.plans[g].forward(xs_ref[g], stream=ref_grp.streams[g]))
        y = gather_y(ys)
        assert relerr(y, oracle.forward(x, a, b)) <= TOL
        assert relerr(y, gather_y(ys_ref)) <= 1e-14
        y_keep = [t.clone() for t in ys]  # (the inverse destroys its input)
        zs = run_ranks(world, lambda g: grp.plans[g].inverse(ys[g], stream=grp.streams[g]))
        assert relerr(gather_x(zs), x) <= TOL
        # host variants (staging pair, copy in / transform / copy out)
        xh = [torch.from_numpy(np.ascontiguousarray(x[p.local_box(0)[0][0]:p.local_box(0)[1][0]])).pin_memory()
              for p in grp.plans]
        yh = [torch.empty(p.y_shape, dtype=torch.float64).pin_memory() for p in grp.plans]
        zh = [torch.empty(p.x_shape, dtype=torch.float64).pin_memory() for p in grp.plans]
        run_ranks(world, lambda g: grp.plans[g].forward_host(xh[g], yh[g], stream=grp.streams[g]))
        assert relerr(np.concatenate([t.numpy() for t in yh], axis=1), gather_y(y_keep)) <= 1e-14
        run_ranks(world, lambda g: grp.plans[g].inverse_host(yh[g], zh[g], stream=grp.streams[g]))
        assert relerr(np.concatenate([t.numpy() for t in zh], axis=0), x) <= TOL
        assert np.array_equal(xh[0].numpy(), x[:xh[0].shape[0]])  # host inputs are never modified
    finally:
        grp.close()
        ref_grp.close()


def test_lowmem_footprint():
    """Per-rank device memory of a capacity-mode plan: the plan's factors only (no slab-sized buffer), i.e. the
    caller's two slabs + the factors (~0.1 MB per axis here) per GPU; the fused-exchange mode adds one receive slab,
    the NCCL all-to-all mode two (send + receive).  Measured with cudaMemGetInfo around plan creation and one forward per rank, at 256^3 over 2
    virtual ranks (64 MiB slabs), against G single-GPU plans of the same shape (the same factor allocations)."""
    shape, a, b, G = (256, 256, 256), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1), 2
    slab_bytes = 8 * int(np.prod(shape)) // G
    x = si.gaussian(shape, seed=5)

    def measure(make):
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        free0 = torch.cuda.mem_get_info()[0]
        closer = make()
        torch.cuda.synchronize()
        used = free0 - torch.cuda.mem_get_info()[0]
        closer()
        return used

    def dist_group(flags):
        def make():
            grp = Group(G, shape, a, b, flags=flags)
            xs = x_slabs(grp, x)
            ys = [torch.empty(p.y_shape, dtype=torch.float64, device="cuda") for p in grp.plans]
            torch.cuda.synchronize()
            run_ranks(G, lambda g: grp.plans[g].forward(xs[g], ys[g], stream=grp.streams[g]))
            return lambda: (grp.close(), xs.clear(), ys.clear())
        return measure(make) - 2 * G * slab_bytes  # minus the caller's x- and y-slabs (torch allocations)

    def single_plans():
        ps = [jt.Plan(shape, a, b, 1e-12) for _ in range(G)]
        return lambda: [p.close() for p in ps]
    base = measure(single_plans)
    lowmem = dist_group(jt.JT_DIST_LOWMEM)
    fused = dist_group(0)
    a2a = dist_group(jt.JT_DIST_NCCL_A2A)
    assert lowmem - base <= 0.05 * G * slab_bytes, (lowmem, base, slab_bytes)
    assert 0.95 * G * slab_bytes <= fused - lowmem <= 1.05 * G * slab_bytes, (fused, lowmem, slab_bytes)
    assert a2a - lowmem >= 1.9 * G * slab_bytes, (a2a, lowmem, slab_bytes)


def test_virtual_exchange_failure_aborts():
    """A peer that never reaches the exchange: the waiting rank's call returns JT_ERR_NCCL after the group's timeout
    (the communicator-abort path) and every later call on its plan is refused with JT_ERR_NCCL."""
    shape, a, b = (32, 32, 8), (0.1, 0.2, 0.3), (0.0, -0.1, 0.2)
    grp = Group(2, shape, a, b, timeout_ms=1500)
    try:
        x0 = grp.plans[0].local_input(torch.from_numpy(si.gaussian(shape, seed=1)))
        with pytest.raises(jt.JTError) as ei:
            grp.plans[0].forward(x0)
        assert ei.value.status == jt.JT_ERR_NCCL
        with pytest.raises(jt.JTError) as ei:
            grp.plans[0].forward(x0)
        assert ei.value.status == jt.JT_ERR_NCCL
        torch.cuda.synchronize()
    finally:
        grp.close()


def test_profile_phases():
    """jt_profile / jt_last_profile (bench.py's per-axis and all-to-all split): a single-GPU 3D transform reports
    three axis passes inside the call; a distributed one also the exchange."""
    shape, a, b = (128, 128, 128), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)
    p = jt.Plan(shape, a, b, 1e-12)
    x = torch.from_numpy(si.gaussian(shape, seed=2)).cuda()
    y = torch.empty_like(x)
    jt.jt_profile(p.handle, True)
    jt.jt_forward(p.handle, x, y)
    prof = jt.jt_last_profile(p.handle)
    assert all(t > 0 for t in prof["axis_ms"]) and prof["exchange_ms"] == 0.0
    assert sum(prof["axis_ms"]) <= prof["total_ms"] * 1.001 + 1e-3
    p.close()
    grp = Group(2, shape, a, b)
    try:
        for q in grp.plans:
            jt.jt_profile(q.handle, True)
        xs = x_slabs(grp, si.gaussian(shape, seed=2))
        torch.cuda.synchronize()
        run_ranks(2, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        for q in grp.plans:
            pr = jt.jt_last_profile(q.handle)
            assert all(t > 0 for t in pr["axis_ms"]) and pr["exchange_ms"] > 0 and pr["total_ms"] > 0
    finally:
        grp.close()


def test_checks_build_parity_and_no_violations():
    """The bounds-checked build (libjt_checks.so) on small cases of every kernel family and schedule (1D-3D, term
    split, chunk-major virtual ranks at G = 2 and 4 in both modes, host paths, nonuniform, second kind): parity with
    the oracle and zero violations; plus the negative control (a declared-too-small output extent is caught and the
    elements beyond it are left untouched).  Runs in a subprocess (the library is chosen at import, JT_LIB)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_1901_07275_b200", "libjt_checks.so")
    assert os.path.exists(lib), "build() makes libjt_checks.so"
    env = dict(os.environ, JT_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "checks_cases.py")], env=env, cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "CHECKS OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.parametrize("name,world,flags", [("cfg5_3d_512", 8, 0), ("cfg3_2d_4096", 8, 0), ("cfg4_3d_256", 4, 0),
                                              ("cfg5_3d_512", 8, 1), ("cfg5_3d_512", 8, 2)])
def test_full_size_distributed_virtual_ranks(name, world, flags):
    """The BASELINE multi-GPU configs at full size through the library's distributed schedule (the launch
    configuration bench.py runs under torchrun, G virtual ranks; flags 1 = JT_DIST_LOWMEM): the assembled y-slabs
    against the oracle's one-by-one sums at sampled outputs (first / last element included), and the full-array round
    trip through the distributed inverse."""
    c = si.CONFIGS[name]
    shape, a, b = c["n"], c["a"], c["b"]
    grp = Group(world, shape, a, b, flags=flags)
    try:
        x = si.gaussian(shape, seed=0)
        xs = x_slabs(grp, x)
        torch.cuda.synchronize()
        ys = run_ranks(world, lambda g: grp.plans[g].forward(xs[g], stream=grp.streams[g]))
        y = gather_y(ys)
        idx = si.sample_indices(shape, 24, seed=3)
        ref = oracle.forward_at(x, a, b, idx)
        assert relerr(y[tuple(idx.T)], ref) <= TOL
        zs = run_ranks(world, lambda g: grp.plans[g].inverse(ys[g], stream=grp.streams[g]))
        assert relerr(gather_x(zs), x) <= TOL
    finally:
        grp.close()
