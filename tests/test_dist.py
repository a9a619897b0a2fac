"""Slab-distributed schedule on CPU: world size 2 and 4 over
gloo, the axis pass replaced by an oracle-backed stand-in with the SAME layout contract as
include/jt.h jt_axis_pass (chunk-major input / output with c = n / G).  What is tested is the host
logic: which local passes run, with which (outer, inner, split) geometry, and that one all-to-all of
the chunk-major blocks turns x-slabs into y-slabs (and back).  The composed result must equal the
oracle's full transform restricted to this rank's box.

The LIBRARY's own distributed schedule (transform_dist / the distributed host paths: the pipelined row-chunk
launches with ostride > outer, the fused peer-store exchange and the NCCL all-to-all mode, capacity mode) runs at
G = 2, 4, 8 virtual ranks on one GPU in tests/test_gpu_dist.py, against the oracle and bit for bit against this
module's Python twin (dist.SlabPlan); tests/test_gpu.py::test_chunk_major_layouts_virtual_ranks covers the twin's
whole-slab chunk-major launches (ostride == outer).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")


def chunk_index(outer, n, inner, split, ostride=None):
    """Flat positions of element (o, j, i) of an (outer, n, inner) array in the chunk-major layout
    (include/jt.h jt_axis_pass / jt_axis_pass_ex): (j / c) (ostride c inner) + o c inner + (j % c) inner + i,
    c = n / split, ostride = outer unless the launch covers part of the rows."""
    c = n // split
    ostride = outer if ostride is None else ostride
    o = np.arange(outer)[:, None, None]
    j = np.arange(n)[None, :, None]
    i = np.arange(inner)[None, None, :]
    return (j // c) * (ostride * c * inner) + o * c * inner + (j % c) * inner + i


def make_oracle_axis_pass(shape, a, b):
    mats = [oracle.phi(shape[ax], a[ax], b[ax]) for ax in range(len(shape))]

    def axis_pass(axis, inverse, src, dst, outer, inner, in_split, out_split, ostride=None):
        n = shape[axis]
        M = mats[axis].T if inverse else mats[axis]
        s = src.reshape(-1).numpy()
        X = s[chunk_index(outer, n, inner, in_split, ostride if in_split > 1 else None)]   # (outer, n, inner)
        Y = np.einsum("jk,okI->ojI", M, X)
        d = dst.reshape(-1)
        idx = chunk_index(outer, n, inner, out_split, ostride if out_split > 1 else None)
        d[torch.from_numpy(idx.ravel())] = torch.from_numpy(Y.ravel())
    return axis_pass


def _worker(rank, world, port, shape, a, b, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1901_07275_b200.dist import SlabPlan
        sp = SlabPlan(shape, a, b, 1e-12, dist, axis_pass=make_oracle_axis_pass(shape, a, b))
        x = si.gaussian(shape, seed=3)
        xs = sp.local_input(x)
        ys = sp.forward(xs)
        ref = oracle.forward(x, a, b)
        lo, hi = sp.local_box(1)
        e_fwd = float(np.max(np.abs(ys.numpy() - ref[:, lo[1]:hi[1]])))
        zs = sp.inverse(ys)
        lo0, hi0 = sp.local_box(0)
        e_rt = float(np.max(np.abs(zs.numpy() - x[lo0[0]:hi0[0]])))
        # inverse alone from an independent y-slab
        yv = si.gaussian(shape, seed=4)
        ws = sp.inverse(sp.local_output(yv))
        e_inv = float(np.max(np.abs(ws.numpy() - oracle.inverse(yv, a, b)[lo0[0]:hi0[0]])))
        # other pipeline depths (one chunk, a ragged split, one row per chunk) give the same slabs
        R = shape[0] // world
        for k in sorted({1, 3, R}):
            e_fwd = max(e_fwd, float(np.max(np.abs(sp.forward(xs, chunks=k).numpy() - ys.numpy()))))
            e_inv = max(e_inv, float(np.max(np.abs(sp.inverse(sp.local_output(yv), chunks=k).numpy() - ws.numpy()))))
        q.put((rank, e_fwd, e_rt, e_inv, tuple(ys.shape), tuple(ws.shape)))
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,shape,a,b", [
    (2, (8, 12, 10), (0.2, -0.4, 0.35), (-0.2, 0.3, 0.1)),
    (2, (16, 6), (0.1, -0.25), (-0.4, 0.35)),
    (4, (8, 16, 5), (0.25, 0.25, -0.6), (-0.25, -0.25, 0.4)),
    (4, (12, 8), (0.45, 0.0), (-0.45, 0.0)),
])
def test_slab_schedule_gloo(world, shape, a, b):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, a, b, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 6, r
        _, e_fwd, e_rt, e_inv, yshape, wshape = r
        assert e_fwd < 1e-12 and e_rt < 1e-12 and e_inv < 1e-12, r
        assert yshape == (shape[0], shape[1] // world) + tuple(shape[2:])
        assert wshape == (shape[0] // world,) + tuple(shape[1:])


def test_chunk_index_is_plain_for_split_one():
    idx = chunk_index(3, 7, 5, 1)
    np.testing.assert_array_equal(idx.ravel(), np.arange(3 * 7 * 5))


def test_chunk_index_is_a_permutation():
    idx = chunk_index(4, 12, 3, 4)
    assert sorted(idx.ravel().tolist()) == list(range(4 * 12 * 3))
