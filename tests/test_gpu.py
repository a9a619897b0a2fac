"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north star): relative l2 error <= 1e-10 against the oracle on the same seeded inputs
(fp64), and forward->inverse round trip <= 1e-10.  The method's own error at eps = 1e-12 is ~1e-12.
Full-size configs are checked on sampled outputs computed one by one by the oracle plus the round trip.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1901_07275_b200 as jt

TOL = 1e-10


def relerr(x, ref):
    return float(np.linalg.norm(np.ravel(x) - np.ravel(ref)) / np.linalg.norm(np.ravel(ref)))


def gpu_forward(plan, x_np, inverse=False, inplace=False, stream=None):
    x = torch.from_numpy(x_np).cuda()
    if inplace:
        out = x
    else:
        out = torch.empty_like(x)
    (jt.jt_inverse if inverse else jt.jt_forward)(plan.handle, x, out, stream)
    torch.cuda.synchronize()
    return out.cpu().numpy()


# ragged and edge shapes: n <= k0 (dense-only), n = k0 + 1, non powers of two (FFT length N > n),
# line counts that are not multiples of the CTA's line tile
CASES_1D = [(2, 0.1, -0.2), (16, 0.3, 0.3), (27, -0.5, 0.5), (28, 0.25, -0.3), (64, 0.45, -0.45),
            (100, -0.75, 0.2), (256, 0.1, -0.4), (333, 0.9, -0.9), (512, 0.25, -0.25), (777, 0.0, 0.0),
            (1024, 0.25, -0.3), (2048, -0.3, 0.6), (3000, 0.2, 0.2), (4096, 0.45, -0.45)]


@pytest.mark.parametrize("n,a,b", CASES_1D)
def test_1d_forward_inverse(n, a, b):
    p = jt.Plan(n, a, b, 1e-12)
    x = si.gaussian((n,), seed=n)
    y = gpu_forward(p, x)
    assert relerr(y, oracle.forward(x, a, b)) <= TOL
    z = gpu_forward(p, x, inverse=True)
    assert relerr(z, oracle.inverse(x, a, b)) <= TOL
    assert relerr(gpu_forward(p, y, inverse=True), x) <= TOL


CASES_ND = [((256, 256), (0.1, -0.25), (-0.4, 0.35)),              # BASELINE config 2
            ((100, 300), (0.3, -0.6), (0.2, 0.45)),
            ((33, 7), (0.0, 0.5), (0.0, -0.5)),
            ((4096, 16), (0.45, 0.0), (-0.45, 0.0)),
            ((17, 2048), (-0.2, 0.7), (0.1, 0.3)),
            ((64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
            ((5, 130, 9), (0.25, 0.25, 0.25), (-0.25, -0.25, -0.25)),
            ((128, 128, 128), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1))]


@pytest.mark.parametrize("shape,a,b", CASES_ND)
def test_nd_forward_inverse(shape, a, b):
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=len(shape))
    y = gpu_forward(p, x)
    assert relerr(y, oracle.forward(x, a, b)) <= TOL
    z = gpu_forward(p, x, inverse=True)
    assert relerr(z, oracle.inverse(x, a, b)) <= TOL


def test_config1_1d_1024():
    c = si.CONFIGS["cfg1_1d_1024"]
    p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
    x = si.gaussian(c["n"], seed=0)
    y = gpu_forward(p, x)
    assert relerr(y, oracle.forward(x, c["a"], c["b"])) <= TOL
    assert relerr(gpu_forward(p, y, inverse=True), x) <= TOL


def test_config4_3d_256_full():
    c = si.CONFIGS["cfg4_3d_256"]
    p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
    x = si.gaussian(c["n"], seed=0)
    y = gpu_forward(p, x)
    assert relerr(y, oracle.forward(x, c["a"], c["b"])) <= TOL
    yi = si.gaussian(c["n"], seed=1)
    assert relerr(gpu_forward(p, yi, inverse=True), oracle.inverse(yi, c["a"], c["b"])) <= TOL
    assert relerr(gpu_forward(p, y, inverse=True), x) <= TOL


@pytest.mark.parametrize("name", ["cfg3_2d_4096", "cfg5_3d_512"])
def test_full_size_sampled(name):
    """Full-size configs in the launch configuration bench.py times: sampled outputs vs the oracle's
    one-by-one sums (forward_at / inverse_at), plus the round trip over the whole array."""
    c = si.CONFIGS[name]
    p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
    x = si.gaussian(c["n"], seed=0)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    jt.jt_forward(p.handle, xd, yd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    idx = si.sample_indices(c["n"], 24, seed=3)
    ref = oracle.forward_at(x, c["a"], c["b"], idx)
    got = y[tuple(idx.T)]
    assert np.max(np.abs(got - ref)) <= TOL * np.linalg.norm(ref) / np.sqrt(len(ref)) * 10
    assert relerr(got, ref) <= TOL
    # round trip over the whole array (orthogonality: Phi^T Phi = I)
    zd = torch.empty_like(xd)
    jt.jt_inverse(p.handle, yd, zd)
    torch.cuda.synchronize()
    assert relerr(zd.cpu().numpy(), x) <= TOL
    if c["inverse"]:
        idx2 = si.sample_indices(c["n"], 24, seed=4)
        ref2 = oracle.inverse_at(y, c["a"], c["b"], idx2)
        got2 = zd.cpu().numpy()[tuple(idx2.T)]
        assert relerr(got2, ref2) <= TOL


def test_cfg5_full_forward_and_determinism():
    """The bench workload (512^3) compared over the WHOLE array (a sampled check once missed a race that
    corrupted ~1e-4 of the rows), and bitwise-repeatable forward and inverse (no atomics anywhere)."""
    c = si.CONFIGS["cfg5_3d_512"]
    p = jt.Plan(c["n"], c["a"], c["b"], c["eps"])
    x = si.gaussian(c["n"], seed=0)
    xd = torch.from_numpy(x).cuda()
    y1 = torch.empty_like(xd)
    y2 = torch.empty_like(xd)
    jt.jt_forward(p.handle, xd, y1)
    jt.jt_forward(p.handle, xd, y2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    z1 = torch.empty_like(xd)
    z2 = torch.empty_like(xd)
    jt.jt_inverse(p.handle, y1, z1)
    jt.jt_inverse(p.handle, y1, z2)
    torch.cuda.synchronize()
    assert torch.equal(z1, z2)
    y = y1.cpu().numpy()
    del y1, y2, z2
    ref = oracle.forward(x, c["a"], c["b"])
    assert relerr(y, ref) <= TOL
    assert np.max(np.abs(y - ref)) <= 1e-10 * np.max(np.abs(ref))
    assert relerr(z1.cpu().numpy(), x) <= TOL


def test_inplace_and_stream_and_determinism():
    shape, a, b = (96, 200), (0.3, -0.1), (0.2, 0.4)
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=9)
    y1 = gpu_forward(p, x)
    y2 = gpu_forward(p, x, inplace=True)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        jt.jt_forward(p.handle, xd, yd, s)
    s.synchronize()
    np.testing.assert_array_equal(y1, y2)
    np.testing.assert_array_equal(y1, yd.cpu().numpy())


def test_host_entry_points_match_device():
    shape, a, b = (64, 64, 64), (0.1, 0.2, 0.3), (-0.1, -0.2, -0.3)
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=2)
    # identical up to rounding: a few-line launch may split its rank terms over CTAs (term split) where the
    # host path's chunks do not, summing the same terms in another order
    assert relerr(p.forward_host(x), gpu_forward(p, x)) <= 1e-14
    assert relerr(p.inverse_host(x), gpu_forward(p, x, inverse=True)) <= 1e-14


def test_axis_entry_points_compose():
    shape, a, b = (40, 72, 33), (0.1, -0.6, 0.5), (0.0, 0.3, -0.2)
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=5)
    xd = torch.from_numpy(x).cuda()
    w = xd.clone()
    for ax in (0, 1, 2):  # any axis order (the Kronecker factors commute)
        outer = int(np.prod(shape[:ax]))
        inner = int(np.prod(shape[ax + 1:]))
        jt.jt_forward_axis(p.handle, ax, w, w, outer, inner)
    torch.cuda.synchronize()
    assert relerr(w.cpu().numpy(), oracle.forward(x, a, b)) <= TOL


def test_partial_overlap_rejected():
    p = jt.Plan(64, 0.1, 0.1, 1e-12)
    buf = torch.zeros(128, dtype=torch.float64, device="cuda")
    with pytest.raises(jt.JTError) as ei:
        jt.jt_forward(p.handle, buf[:64], buf[8:72])
    assert ei.value.status == jt.JT_ERR_ARG


class _VirtualDist:
    """get_world_size / get_rank of one virtual rank (no collective is ever called: the test does the
    exchange itself between phases, so no kernel waits on another)."""

    def __init__(self, rank, world):
        self.r, self.w = rank, world

    def get_world_size(self, group=None):
        return self.w

    def get_rank(self, group=None):
        return self.r


@pytest.mark.parametrize("world,shape,a,b", [
    (4, (64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
    (8, (96, 64, 33), (0.25, -0.1, 0.0), (-0.25, 0.6, 0.0)),
    (2, (256, 256), (0.1, -0.25), (-0.4, 0.35)),
    (8, (512, 64, 16), (0.25, 0.25, 0.25), (-0.25, -0.25, -0.25)),
])
def test_chunk_major_layouts_virtual_ranks(world, shape, a, b):
    """The slab schedule (paper_1901_07275_b200/dist.py) on one GPU with `world` virtual ranks run one
    after another: the kernels' chunk-major output (out_split) and input (in_split) layouts plus a
    tensor-copy all-to-all must reproduce the oracle's full transform, block by block."""
    from paper_1901_07275_b200.dist import SlabPlan
    sps = [SlabPlan(shape, a, b, 1e-12, _VirtualDist(g, world)) for g in range(world)]
    x = si.gaussian(shape, seed=11)
    ref = oracle.forward(x, a, b)
    c = sps[0].count // world

    def exchange():
        for g in range(world):
            sps[g]._recv.copy_(torch.cat([sps[q]._send[g * c:(g + 1) * c] for q in range(world)]))

    outs = [sp.forward_local(sp.local_input(x)) for sp in sps]
    exchange()
    ys = [sp.forward_finish(o) for sp, o in zip(sps, outs)]
    y_full = np.concatenate([y.cpu().numpy() for y in ys], axis=1)
    assert relerr(y_full, ref) <= TOL
    # inverse from the y-slabs back to x-slabs
    outs = [sp.inverse_local(y) for sp, y in zip(sps, ys)]
    exchange()
    zs = [sp.inverse_finish(o) for sp, o in zip(sps, outs)]
    z_full = np.concatenate([z.cpu().numpy() for z in zs], axis=0)
    assert relerr(z_full, x) <= TOL
    for sp in sps:
        sp.close()


def test_axis_pass_split_arguments_rejected():
    p = jt.Plan((12, 10), (0.1, 0.2), (0.0, 0.1), 1e-12)
    x = torch.zeros(120, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    for args in [(0, 5, 1), (0, 1, 5), (1, 0, 1)]:  # 5 does not divide 12; split 0
        ax, isp, osp = args
        with pytest.raises(jt.JTError) as ei:
            jt.jt_axis_pass(p.handle, ax, False, x, y, 1, 10 if ax == 0 else 1, isp, osp)
        assert ei.value.status == jt.JT_ERR_ARG
    with pytest.raises(jt.JTError):  # chunk-major in place
        jt.jt_axis_pass(p.handle, 0, False, x, x, 1, 10, 1, 2)


def test_slab_plan_nccl_world1():
    """The NCCL all-to-all path of SlabPlan (world size 1: the collective is a self-copy) against the oracle:
    exercises the same code bench.py runs under torchrun on N GPUs."""
    import socket
    import torch.distributed as dist
    from paper_1901_07275_b200.dist import SlabPlan
    if not dist.is_available() or not dist.is_nccl_available():
        pytest.skip("no NCCL")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        from paper_1901_07275_b200.dist import LibSlabPlan
        for shape, a, b in [((48, 40, 36), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
                            ((64, 80), (0.1, -0.25), (-0.4, 0.35))]:
            x = si.gaussian(shape, seed=13)
            for cls in (SlabPlan, LibSlabPlan):  # torch-collective twin and the library-owned NCCL path
                sp = cls(shape, a, b, 1e-12, dist)
                assert sp.local_box(0) == ((0,) * len(shape), shape)
                y = sp.forward(sp.local_input(x))
                assert relerr(y.cpu().numpy(), oracle.forward(x, a, b)) <= TOL, cls
                if cls is LibSlabPlan:  # the pipelined host-buffer path (row chunks may take the term-split
                    # launches, which sum the rank terms in another order: equal up to rounding)
                    xh = sp.local_input(torch.from_numpy(x)).cpu().pin_memory()
                    yh = [torch.empty(sp.y_shape, dtype=torch.float64).pin_memory() for _ in range(3)]
                    sp.forward_host(xh, yh[0])
                    for k in (1, 2):  # two calls in flight through the staging slots
                        sp.forward_host_async(xh, yh[k])
                    sp.wait_host()
                    for k in range(3):
                        assert relerr(yh[k].numpy(), y.cpu().numpy()) <= 1e-14, k
                z = sp.inverse(y)
                assert relerr(z.cpu().numpy(), x) <= TOL, cls
                sp.close()
    finally:
        dist.destroy_process_group()


def test_host_async_stream_matches_device():
    """jt_forward_host_async / jt_inverse_host_async: several calls in flight over the two staging slots, each
    result equal to the device-pointer path up to rounding (include/jt.h)."""
    shape, a, b = (64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)
    p = jt.Plan(shape, a, b, 1e-12)
    xs = [si.gaussian(shape, seed=30 + k) for k in range(5)]
    ys = [np.empty(shape) for _ in range(5)]
    for k in range(5):
        jt.jt_forward_host_async(p.handle, xs[k], ys[k])
    jt.jt_host_wait(p.handle)
    for k in range(5):
        assert relerr(ys[k], gpu_forward(p, xs[k])) <= 1e-14
    zs = [np.empty(shape) for _ in range(3)]
    for k in range(3):
        jt.jt_inverse_host_async(p.handle, ys[k], zs[k])
    jt.jt_host_wait(p.handle)
    for k in range(3):
        assert relerr(zs[k], gpu_forward(p, ys[k], inverse=True)) <= 1e-14
        assert relerr(zs[k], xs[k]) <= TOL


@pytest.mark.parametrize("shape,a,b", [((16, 512, 48), (0.25, 0.25, -0.1), (-0.25, -0.25, 0.3)),
                                       ((300, 256), (0.1, -0.25), (-0.4, 0.35)),
                                       ((2, 4096), (0.2, 0.45), (0.1, -0.45)),
                                       ((48, 1024), (0.3, 0.25), (0.0, -0.3))])
def test_repeat_determinism(shape, a, b):
    """Repeated launches are bitwise identical (no atomics on the data path; the ring refill election and the
    TMEM state cannot change any arithmetic), forward and inverse, for each kernel family."""
    p = jt.Plan(shape, a, b, 1e-12)
    x = torch.from_numpy(si.gaussian(shape, seed=17)).cuda()
    ys = []
    zs = []
    for _ in range(4):
        y = torch.empty_like(x)
        z = torch.empty_like(x)
        jt.jt_forward(p.handle, x, y)
        jt.jt_inverse(p.handle, x, z)
        ys.append(y)
        zs.append(z)
    torch.cuda.synchronize()
    for k in range(1, 4):
        assert torch.equal(ys[0], ys[k]) and torch.equal(zs[0], zs[k])


@pytest.mark.parametrize("shape,a,b", [((512,), (-0.5,), (-0.5,)),           # r = 2: W V mostly outside the ring
                                       ((1000,), (0.5,), (0.5,)),             # r ~ 9, N > n
                                       ((3, 1024), (0.25, -0.5), (-0.3, -0.5)),
                                       ((7, 256, 5), (0.1, 0.2, 0.3), (0.0, -0.1, 0.2)),
                                       ((4096,), (0.3,), (-0.2,)),       # r ~ 22 over 16 CTAs: group term split
                                       ((2048,), (-0.4,), (0.6,))])
def test_term_split_launches(shape, a, b):
    """Few-line launches take the term-split path (rank terms over several CTAs, reduced in a cluster or by ts_reduce,
    DESIGN.md §6), including plans with r < k0 / 2 whose dense block is applied outside the term loop (split over the
    slices), and one-line batches whose CTAs deal their terms to two groups (Ctx::gsl)."""
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=23)
    assert relerr(gpu_forward(p, x), oracle.forward(x, a, b)) <= TOL
    assert relerr(gpu_forward(p, x, inverse=True), oracle.inverse(x, a, b)) <= TOL


def test_last_launches_counts_kernels():
    """jt_last_launches (bench.py's gpu_launches): one fused pass per axis, plus one reduction per term-split axis."""
    p = jt.Plan((128, 128, 128), 0.2, -0.3, 1e-12)  # 16384 lines per axis: no term split
    x = torch.from_numpy(si.gaussian((128, 128, 128), seed=3)).cuda()
    y = torch.empty_like(x)
    jt.jt_forward(p.handle, x, y)
    assert jt.jt_last_launches(p) == 3
    jt.jt_forward_axis(p.handle, 1, x, y, 128, 128)
    assert jt.jt_last_launches(p) == 1
    p.close()
    q = jt.Plan(1024, 0.25, -0.3, 1e-12)  # one line: term split, reduced in a thread-block cluster (one launch)
    x1 = torch.from_numpy(si.gaussian((1024,), seed=3)).cuda()  # or, where no cluster fits, + ts_reduce
    y1 = torch.empty_like(x1)
    jt.jt_inverse(q.handle, x1, y1)
    assert jt.jt_last_launches(q) in (1, 2)
    torch.cuda.synchronize()
    q.close()


@pytest.mark.parametrize("shape,a,b", [((100, 128, 120), (0.3, -0.2, 0.1), (0.2, 0.45, -0.6)),   # many lines: radix 32
                                       ((128, 96), (0.25, -0.3), (-0.1, 0.4)),                   # term split: radix 16
                                       ((2000, 3), (0.1, 0.2), (0.3, -0.4))])                    # N = 2048, radix 16
def test_radix_per_launch_kind(shape, a, b):
    """FFT lengths whose large launches and term-split launches use different register radixes (N = 128: 32 / 16,
    with the term-split twiddle tables uploaded separately; tuning.h) against the oracle."""
    p = jt.Plan(shape, a, b, 1e-12)
    x = si.gaussian(shape, seed=29)
    assert relerr(gpu_forward(p, x), oracle.forward(x, a, b)) <= TOL
    assert relerr(gpu_forward(p, x, inverse=True), oracle.inverse(x, a, b)) <= TOL
    p.close()


@pytest.mark.parametrize("shape,a,b", [((64, 48, 40), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),   # many-line passes
                                       ((1024,), (0.25,), (-0.3,)),                          # cluster term split
                                       ((256, 256), (0.1, -0.25), (-0.4, 0.35))])
def test_cuda_graph_capture(shape, a, b):
    """jt_forward / jt_inverse are capture-safe after one uncaptured call (include/jt.h streams note): a CUDA graph
    of the call replays to the same bits as a direct call."""
    p = jt.Plan(shape, a, b, 1e-12)
    x = torch.from_numpy(si.gaussian(shape, seed=41)).cuda()
    s = torch.cuda.Stream()
    for fn in (jt.jt_forward, jt.jt_inverse):
        y_ref = torch.empty_like(x)
        y = torch.empty_like(x)
        with torch.cuda.stream(s):
            fn(p.handle, x, y_ref, s)  # sizes any workspace outside the capture
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                fn(p.handle, x, y, s)
            y.zero_()
            g.replay()
            s.synchronize()
        assert torch.equal(y, y_ref)
    p.close()
