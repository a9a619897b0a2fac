"""Slab-distributed d-dimensional (d = 2, 3) transform over a torch.distributed process group
(DESIGN.md §7).

Every line of an axis pass is independent (the paper's "n 2D transforms and n^2 1D transforms",
PAPER.md:724; "n 1D transforms" per axis in 2D), so the only exchange of the
axis-factored schedule (eq:TJ PAPER.md:669-674, eq:TJ3 PAPER.md:718-722) is the transpose between
passes.  Rank g of G holds

    forward input  / inverse output: the x-slab  [g n0/G, (g+1) n0/G) x n1 (x n2)      (C-order)
    forward output / inverse input:  the y-slab  n0 x [g n1/G, (g+1) n1/G) (x n2)      (C-order)

Forward: the local axis passes d-1 .. 1, the axis-1 pass writing its output in the CHUNK-MAJOR layout
(`out_split = G`, include/jt.h jt_axis_pass) so that chunk p is the contiguous block for rank p; one
all-to-all (NCCL over NVLink on GPUs); the received buffer is already the C-order y-slab, on which the
axis-0 pass runs.  Inverse: axis d-1 pass, axis-0 pass with `out_split = G`, all-to-all, axis-1 pass
reading the chunk-major layout (`in_split = G`).  There is no pack / unpack kernel and no other
collective.

This module is host-side schedule only: every arithmetic step runs in libjt.so's kernels through
`jt_axis_pass`; the exchange is `torch.distributed.all_to_all_single`.  For CPU tests of the schedule
(gloo, world size > 1) an `axis_pass` callable with the same semantics may be injected.
"""
from __future__ import annotations

import numpy as np


class SlabPlan:
    """Plan + buffers of one rank of a slab-distributed transform.

    shape, a, b, eps: as for `Plan` (d = 2 or 3; shape[0] and shape[1] divisible by the world size).
    dist:      the `torch.distributed` module (initialised); `group` an optional process group.
    axis_pass: optional stand-in `f(axis, inverse, src, dst, outer, inner, in_split, out_split)`; default is
               libjt.so's jt_axis_pass on the current CUDA stream.
    """

    def __init__(self, shape, a, b, eps, dist, group=None, axis_pass=None, device=None, **plan_kw):
        import torch
        self.shape = tuple(int(v) for v in shape)
        self.d = len(self.shape)
        if self.d not in (2, 3):
            raise ValueError("slab decomposition needs d = 2 or 3")
        self.dist = dist
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        n0, n1 = self.shape[0], self.shape[1]
        if n0 % self.G or n1 % self.G:
            raise ValueError(f"n0 = {n0} and n1 = {n1} must be divisible by the world size {self.G}")
        self.rest = int(np.prod(self.shape[2:])) if self.d == 3 else 1
        self.x_shape = (n0 // self.G, n1) + self.shape[2:]
        self.y_shape = (n0, n1 // self.G) + self.shape[2:]
        self.count = int(np.prod(self.x_shape))
        self.plan = None
        if axis_pass is None:
            from . import Plan, jt_axis_pass_ex
            self.plan = Plan(self.shape, a, b, eps, **plan_kw)
            self.ranks = [self.plan.rank(i) for i in range(self.d)]
            handle = self.plan.handle

            def axis_pass(axis, inverse, src, dst, outer, inner, in_split, out_split, ostride=None):
                jt_axis_pass_ex(handle, axis, inverse, src, dst, outer, inner, in_split, out_split,
                                outer if ostride is None else ostride)
            self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        else:
            self.ranks = None
            self.device = torch.device("cpu") if device is None else device
        self._axis = axis_pass
        self._send = torch.empty(self.count, dtype=torch.float64, device=self.device)
        self._recv = torch.empty(self.count, dtype=torch.float64, device=self.device)

    # ---- geometry ----
    def local_box(self, which: int):
        """(lo, hi) index box of this rank's block: which = 0 forward input (x-slab), 1 forward output."""
        lo = [0] * self.d
        hi = list(self.shape)
        ax = 0 if which == 0 else 1
        step = self.shape[ax] // self.G
        lo[ax], hi[ax] = self.rank * step, (self.rank + 1) * step
        return tuple(lo), tuple(hi)

    def local_input(self, full):
        """This rank's x-slab of a full (host) array, as a contiguous tensor on the plan's device."""
        import torch
        lo, hi = self.local_box(0)
        t = torch.as_tensor(full)[lo[0]:hi[0]].contiguous()
        return t.to(self.device)

    def local_output(self, full):
        """This rank's y-slab of a full array (e.g. for the inverse's input)."""
        import torch
        lo, hi = self.local_box(1)
        t = torch.as_tensor(full)[:, lo[1]:hi[1]].contiguous()
        return t.to(self.device)

    # ---- exchange ----
    def _exchange(self):
        self.dist.all_to_all_single(self._recv, self._send, group=self.group)

    # ---- transforms ----
    def forward(self, x, out=None, chunks=None):
        """x-slab coefficients -> y-slab weighted values (the local block of Phi_0 (x) ... (x) Phi_{d-1} alpha).

        The axis-1 pass and the all-to-all are pipelined over `chunks` row chunks of the slab (default
        min(4, rows), the same as the library's transform_dist): chunk k's rows of every chunk-major block are
        exchanged (point-to-point) after its axis-1 pass."""
        import torch
        if tuple(x.shape) != self.x_shape:
            raise ValueError(f"expected the x-slab shape {self.x_shape}")
        out = torch.empty(self.y_shape, dtype=torch.float64, device=self.device) if out is None else out
        G, (n0, n1), r = self.G, self.shape[:2], self.rest
        R, c = n0 // G, n1 // G
        K = chunks if chunks is not None else min(4, R)
        src = x
        if self.d == 3:
            self._axis(2, False, x, out, R * n1, 1, 1, 1)
            src = out
        flat_src = src.reshape(-1)
        for k in range(K):
            r0, r1 = R * k // K, R * (k + 1) // K
            if r1 == r0:
                continue
            self._axis(1, False, flat_src[r0 * n1 * r:r1 * n1 * r], self._send[r0 * c * r:], r1 - r0, r, 1, G,
                       ostride=R)
            self._exchange_rows(r0, r1, c * r)
        return self.forward_finish(out)

    def _exchange_rows(self, r0, r1, rowlen):
        """Rows [r0, r1) of every chunk-major block to / from every rank (point-to-point)."""
        CH = self.count // self.G
        reqs = []
        for g in range(self.G):
            s_view = self._send[g * CH + r0 * rowlen:g * CH + r1 * rowlen]
            r_view = self._recv[g * CH + r0 * rowlen:g * CH + r1 * rowlen]
            if g == self.rank:
                r_view.copy_(s_view)
            else:
                reqs.append(self.dist.isend(s_view, g, group=self.group))
                reqs.append(self.dist.irecv(r_view, g, group=self.group))
        for q in reqs:
            q.wait()

    def forward_local(self, x, out=None):
        """Forward phase 1: the local axis passes d-1 .. 1; leaves the chunk-major send buffer filled."""
        import torch
        if tuple(x.shape) != self.x_shape:
            raise ValueError(f"expected the x-slab shape {self.x_shape}")
        out = torch.empty(self.y_shape, dtype=torch.float64, device=self.device) if out is None else out
        G, (n0, n1), r = self.G, self.shape[:2], self.rest
        if self.d == 3:
            self._axis(2, False, x, out, (n0 // G) * n1, 1, 1, 1)                  # axis 2, tmp in `out`
            self._axis(1, False, out, self._send, n0 // G, r, 1, G)              # axis 1 -> chunk-major
        else:
            self._axis(1, False, x, self._send, n0 // G, 1, 1, G)
        return out

    def forward_finish(self, out):
        """Forward phase 2 (after the all-to-all): the axis-0 pass on the received y-slab."""
        G, (n0, n1), r = self.G, self.shape[:2], self.rest
        self._axis(0, False, self._recv, out, 1, (n1 // G) * r, 1, 1)
        return out

    def inverse(self, y, out=None, chunks=None):
        """y-slab weighted values -> x-slab coefficients (transpose in every axis).

        The all-to-all and the axis-1 pass are pipelined over `chunks` row chunks of the x-slab (default
        min(4, rows), as in the library's transform_dist): rows [r0, r1) of every block are exchanged, then the
        axis-1 pass runs on those rows while the next chunk is in flight."""
        out = self.inverse_local(y, out)
        G, (n0, n1), r = self.G, self.shape[:2], self.rest
        R, c = n0 // G, n1 // G
        K = chunks if chunks is not None else min(4, R)
        flat_out = out.reshape(-1)
        for k in range(K):
            r0, r1 = R * k // K, R * (k + 1) // K
            if r1 == r0:
                continue
            self._exchange_rows(r0, r1, c * r)
            self._axis(1, True, self._recv[r0 * c * r:], flat_out[r0 * n1 * r:r1 * n1 * r], r1 - r0, r, G, 1,
                       ostride=R)
        return out

    def inverse_local(self, y, out=None):
        """Inverse phase 1: axis d-1 pass, axis-0 pass into the chunk-major send buffer."""
        import torch
        if tuple(y.shape) != self.y_shape:
            raise ValueError(f"expected the y-slab shape {self.y_shape}")
        out = torch.empty(self.x_shape, dtype=torch.float64, device=self.device) if out is None else out
        G, (n0, n1), r = self.G, self.shape[:2], self.rest
        if self.d == 3:
            self._axis(2, True, y, out, n0 * (n1 // G), 1, 1, 1)                  # axis 2, tmp in `out`
            self._axis(0, True, out, self._send, 1, (n1 // G) * r, 1, G)         # axis 0 -> chunk-major
        else:
            self._axis(0, True, y, self._send, 1, n1 // G, 1, G)
        return out

    def inverse_finish(self, out):
        """Inverse phase 2 (after the all-to-all): the axis-1 pass reading the chunk-major receive buffer."""
        G, (n0, n1), r = self.G, self.shape[:2], self.rest
        self._axis(1, True, self._recv, out, n0 // G, r, G, 1)
        return out

    def forward_host(self, x_host, y_host, x_dev, y_dev):
        """End-to-end forward of this rank's x-slab: pinned host x-slab -> device -> transform -> host y-slab."""
        x_dev.copy_(x_host, non_blocking=True)
        self.forward(x_dev, y_dev)
        y_host.copy_(y_dev, non_blocking=True)
        return y_host

    def make_forward_step(self, x):
        """Closure running one forward transform of the resident x-slab into a preallocated y-slab."""
        import torch
        out = torch.empty(self.y_shape, dtype=torch.float64, device=self.device)

        def step():
            self.forward(x, out)
            return out
        step.out = out
        return step

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None


class LibSlabPlan:
    """The same slab-distributed transform with the schedule AND the all-to-all inside libjt.so
    (jt_plan_dist: a library-owned NCCL communicator, grouped ncclSend/ncclRecv on the caller's stream).
    torch.distributed is only used to broadcast the 128-byte NCCL unique id from rank 0.  This is the path
    bench.py times; `SlabPlan` above is its host-side twin used by the gloo CPU tests."""

    def __init__(self, shape, a, b, eps, dist=None, group=None, flags: int = 0, vgroup=None, rank=None,
                 **plan_kw):
        """dist/group: the torch.distributed module and process group (NCCL communicator created inside the
        library).  Test mode (include/jt_debug.h): vgroup = a jt_debug_vgroup_create handle and rank = this
        virtual rank, no torch.distributed (the library's in-process exchange instead of NCCL).
        flags: JT_DIST_LOWMEM (capacity mode: the input slab is the workspace and is destroyed)."""
        import torch
        from . import (jt_debug_plan_virtual, jt_destroy, jt_dist_unique_id, jt_local_box, jt_plan_dist,
                       jt_plan_info, jt_plan_rank)
        self.shape = tuple(int(v) for v in shape)
        self.d = len(self.shape)
        self.flags = flags
        if vgroup is not None:
            self.rank = int(rank)
            self.handle = jt_debug_plan_virtual(self.shape, a, b, eps, vgroup, self.rank, flags=flags, **plan_kw)
        else:
            self.G = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if self.rank == 0:
                uid.copy_(torch.frombuffer(bytearray(jt_dist_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, src=0, group=group)
            self.handle = jt_plan_dist(self.shape, a, b, eps, bytes(uid.cpu().numpy().tobytes()), self.rank, self.G,
                                       flags=flags, **plan_kw)
        self._destroy = jt_destroy
        self.ranks = [jt_plan_rank(self.handle, i) for i in range(self.d)]
        self.infos = [jt_plan_info(self.handle, i) for i in range(self.d)]
        lo0, hi0 = jt_local_box(self.handle, 0, self.d)
        lo1, hi1 = jt_local_box(self.handle, 1, self.d)
        self.box = {0: (lo0, hi0), 1: (lo1, hi1)}
        self.x_shape = tuple(h - l for l, h in zip(lo0, hi0))
        self.y_shape = tuple(h - l for l, h in zip(lo1, hi1))
        self.G = self.shape[0] // self.x_shape[0]
        self.device = torch.device("cuda", torch.cuda.current_device())

    def local_box(self, which: int):
        return self.box[which]

    def local_input(self, full):
        import torch
        lo, hi = self.box[0]
        return torch.as_tensor(full)[lo[0]:hi[0]].contiguous().to(self.device)

    def local_output(self, full):
        import torch
        lo, hi = self.box[1]
        return torch.as_tensor(full)[:, lo[1]:hi[1]].contiguous().to(self.device)

    def forward(self, x, out=None, stream=None):
        """x-slab -> y-slab (with JT_DIST_LOWMEM the x-slab is overwritten: it is the workspace)."""
        import torch
        from . import jt_forward
        out = torch.empty(self.y_shape, dtype=torch.float64, device=self.device) if out is None else out
        jt_forward(self.handle, x, out, stream)
        return out

    def inverse(self, y, out=None, stream=None):
        """y-slab -> x-slab (with JT_DIST_LOWMEM the y-slab is overwritten)."""
        import torch
        from . import jt_inverse
        out = torch.empty(self.x_shape, dtype=torch.float64, device=self.device) if out is None else out
        jt_inverse(self.handle, y, out, stream)
        return out

    def forward_host(self, x_host, y_host, x_dev=None, y_dev=None, stream=None):
        """End-to-end forward of this rank's slab from / to (pinned) host memory (C: jt_forward_host)."""
        from . import jt_forward_host
        jt_forward_host(self.handle, x_host.numpy(), y_host.numpy(), stream)
        return y_host

    def inverse_host(self, y_host, x_host, stream=None):
        """End-to-end inverse of this rank's y-slab (C: jt_inverse_host)."""
        from . import jt_inverse_host
        jt_inverse_host(self.handle, y_host.numpy(), x_host.numpy(), stream)
        return x_host

    def inverse_host_async(self, y_host, x_host, stream=None):
        """Enqueue an end-to-end inverse of this rank's y-slab (C: jt_inverse_host_async); valid after wait_host()."""
        from . import jt_inverse_host_async
        jt_inverse_host_async(self.handle, y_host.numpy(), x_host.numpy(), stream)
        return x_host

    def forward_host_async(self, x_host, y_host, stream=None):
        """Enqueue an end-to-end forward of this rank's slab (C: jt_forward_host_async; consecutive calls overlap
        through the plan's two staging slots); results are valid after wait_host()."""
        from . import jt_forward_host_async
        jt_forward_host_async(self.handle, x_host.numpy(), y_host.numpy(), stream)
        return y_host

    def wait_host(self):
        from . import jt_host_wait
        jt_host_wait(self.handle)

    def make_forward_step(self, x):
        import torch
        out = torch.empty(self.y_shape, dtype=torch.float64, device=self.device)

        def step():
            self.forward(x, out)
            return out
        step.out = out
        return step

    def close(self):
        if getattr(self, "handle", None):
            self._destroy(self.handle)
            self.handle = None
