"""B200-native fast multi-dimensional Jacobi polynomial transform (arXiv 1901.07275).

Thin ctypes binding over the C ABI of `libjt.so` (include/jt.h): argument marshalling only; every
step of the transform runs in the library's sm_100a kernels, every step of the plan in its host C++.
PyTorch supplies device memory and streams (tensors are passed by `data_ptr()`).

There is no CPU fallback: importing this package fails loudly if `libjt.so` has not been built
(`python -m paper_1901_07275_b200.build`), and device calls fail with a JTError if no GPU is present.

Names follow the C ABI: jt_plan / jt_forward / jt_inverse / jt_destroy (+ introspection), plus a
convenience `Plan` class.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# JT_LIB: path of an alternative in-tree build (kernel A/B experiments, tools/); default libjt.so
LIB_PATH = os.environ.get("JT_LIB") or os.path.join(_HERE, "libjt.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1901_07275_b200.build` "
                      "(there is deliberately no fallback path)")
_lib = ctypes.CDLL(LIB_PATH)

JT_OK, JT_ERR_ARG, JT_ERR_DOMAIN, JT_ERR_NUMERIC, JT_ERR_ALLOC, JT_ERR_CUDA, JT_ERR_NCCL = range(7)
JT_KIND_P, JT_KIND_Q = 0, 1
_STATUS = {0: "JT_OK", 1: "JT_ERR_ARG", 2: "JT_ERR_DOMAIN", 3: "JT_ERR_NUMERIC", 4: "JT_ERR_ALLOC",
           5: "JT_ERR_CUDA", 6: "JT_ERR_NCCL"}

# Every symbol declared in include/jt.h and include/jt_debug.h (checked by tests/test_abi.py).
EXPORTED = ["jt_default_opts", "jt_plan", "jt_plan_ex", "jt_adjoint", "jt_plan_kind", "jt_dist_unique_id",
            "jt_plan_dist", "jt_local_box", "jt_forward_host_async", "jt_inverse_host_async", "jt_host_wait",
            "jt_forward", "jt_inverse", "jt_forward_host", "jt_inverse_host",
            "jt_forward_axis", "jt_inverse_axis", "jt_axis_pass", "jt_axis_pass_ex", "jt_destroy", "jt_plan_rank", "jt_plan_info",
            "jt_plan_nodes", "jt_plan_factors", "jt_plan_sigma", "jt_last_launches", "jt_last_error", "jt_version",
            "jt_plan_dist_ex", "jt_sync", "jt_profile", "jt_last_profile", "jt_dist_mode",
            "jt_debug_modified_pq", "jt_debug_checks", "jt_debug_vgroup_create", "jt_debug_vgroup_destroy",
            "jt_debug_plan_virtual", "jt_debug_axis_pass_lim", "jt_debug_pair_factors"]

JT_DIST_LOWMEM = 1
JT_DIST_NCCL_A2A = 2  # the NCCL all-to-all instead of the fused (peer-store) exchange


class JTError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.jt_last_error().decode()
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class jt_opts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("k0", ctypes.c_int), ("rmax_init", ctypes.c_int),
                ("q", ctypes.c_int), ("sweeps", ctypes.c_int), ("device", ctypes.c_int)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_lib.jt_default_opts.argtypes = [ctypes.POINTER(jt_opts)]
_lib.jt_plan.argtypes = [ctypes.POINTER(_P), ctypes.c_int, _I64, _D, _D, ctypes.c_double, ctypes.POINTER(jt_opts)]
_lib.jt_plan_ex.argtypes = [ctypes.POINTER(_P), ctypes.c_int, _I64, _D, _D, ctypes.c_void_p, ctypes.c_int,
                            ctypes.c_double, ctypes.POINTER(jt_opts)]
_lib.jt_dist_unique_id.argtypes = [ctypes.c_void_p]
_lib.jt_plan_dist.argtypes = [ctypes.POINTER(_P), ctypes.c_int, _I64, _D, _D, ctypes.c_double, ctypes.POINTER(jt_opts),
                              ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
_lib.jt_plan_dist_ex.argtypes = [ctypes.POINTER(_P), ctypes.c_int, _I64, _D, _D, ctypes.c_double,
                                 ctypes.POINTER(jt_opts), ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
_lib.jt_sync.argtypes = [_P, ctypes.c_void_p]
_lib.jt_dist_mode.argtypes = [_P, ctypes.POINTER(ctypes.c_int)]
_lib.jt_profile.argtypes = [_P, ctypes.c_int]
_lib.jt_last_profile.argtypes = [_P, _D]
_lib.jt_debug_checks.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_ulonglong),
                                 ctypes.POINTER(ctypes.c_int)]
_lib.jt_debug_vgroup_create.argtypes = [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int]
_lib.jt_debug_vgroup_destroy.argtypes = [_P]
_lib.jt_debug_plan_virtual.argtypes = [ctypes.POINTER(_P), ctypes.c_int, _I64, _D, _D, ctypes.c_double,
                                       ctypes.POINTER(jt_opts), _P, ctypes.c_int, ctypes.c_int]
_lib.jt_debug_axis_pass_lim.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_void_p]
_lib.jt_local_box.argtypes = [_P, ctypes.c_int, _I64, _I64]
_lib.jt_plan_kind.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
_lib.jt_host_wait.argtypes = [_P]
for _f in ("jt_forward", "jt_inverse", "jt_adjoint", "jt_forward_host", "jt_inverse_host", "jt_forward_host_async",
           "jt_inverse_host_async"):
    getattr(_lib, _f).argtypes = [_P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
for _f in ("jt_forward_axis", "jt_inverse_axis"):
    getattr(_lib, _f).argtypes = [_P, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_int64, ctypes.c_void_p]
_lib.jt_axis_pass.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                              ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
_lib.jt_axis_pass_ex.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]
_lib.jt_destroy.argtypes = [_P]
_lib.jt_plan_rank.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
_lib.jt_plan_info.argtypes = [_P, ctypes.c_int, _I64, _I64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
_lib.jt_plan_nodes.argtypes = [_P, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
_lib.jt_plan_factors.argtypes = [_P, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.jt_plan_sigma.argtypes = [_P, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                               ctypes.POINTER(ctypes.c_int)]
_lib.jt_last_launches.argtypes = [_P, ctypes.POINTER(ctypes.c_int)]
_lib.jt_last_error.restype = ctypes.c_char_p
_lib.jt_version.restype = ctypes.c_char_p
_lib.jt_debug_modified_pq.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
for _f in EXPORTED:
    if _f not in ("jt_last_error", "jt_version"):
        getattr(_lib, _f).restype = ctypes.c_int


def _check(status: int, where: str):
    if status != JT_OK:
        raise JTError(status, where)


def _ptr(x) -> int:
    """Device or host address of a torch tensor / numpy array (C-contiguous float64 required)."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags.c_contiguous:
            raise ValueError("numpy arrays must be C-contiguous float64")
        return x.ctypes.data
    if x.dtype.__repr__() != "torch.float64" or not x.is_contiguous():
        raise ValueError("tensors must be contiguous torch.float64")
    return x.data_ptr()


def _local_elems(plan: int, which: int) -> int:
    """Elements of the plan's local array: which = 0 the forward input (x-slab), 1 the forward output (y-slab);
    the whole array for non-distributed plans (C: jt_local_box)."""
    lo = (ctypes.c_int64 * 3)(0, 0, 0)
    hi = (ctypes.c_int64 * 3)(1, 1, 1)
    _check(_lib.jt_local_box(plan, which, lo, hi), "jt_local_box")
    return int(np.prod([h - l for l, h in zip(lo, hi)]))


def _host_ptr(x, plan: int, which: int) -> int:
    """Address of a host buffer of a *_host call after checking it: a C-contiguous float64 numpy array with exactly
    the plan's local element count (the C side reads / writes that many doubles)."""
    if not isinstance(x, np.ndarray):
        raise TypeError("host buffers must be numpy arrays (e.g. tensor.numpy() of a pinned CPU tensor)")
    if x.dtype != np.float64 or not x.flags.c_contiguous:
        raise ValueError("host buffers must be C-contiguous float64")
    want = _local_elems(plan, which)
    if x.size != want:
        raise ValueError(f"host buffer has {x.size} elements, the plan's local array has {want}")
    if not x.flags.writeable and which == 1:
        raise ValueError("output host buffer is read-only")
    return x.ctypes.data


# Host buffers of *_host_async calls in flight, per plan handle: kept alive until jt_host_wait (the copies read /
# write them asynchronously).
_INFLIGHT: dict = {}


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def jt_last_launches(plan) -> int:
    """Kernels the most recent transform call on `plan` (a Plan or a raw handle) enqueued."""
    c = ctypes.c_int(0)
    _check(_lib.jt_last_launches(getattr(plan, "handle", plan), ctypes.byref(c)), "jt_last_launches")
    return c.value


def jt_version() -> str:
    return _lib.jt_version().decode()


def jt_default_opts() -> jt_opts:
    o = jt_opts()
    _check(_lib.jt_default_opts(ctypes.byref(o)), "jt_default_opts")
    return o


def jt_plan(n, a, b, eps: float = 1e-12, seed: int = 0, k0: int = -1, rmax_init: int = 0, q: int = 3,
            sweeps: int = 2, device: int = -1, points=None, kind: int = JT_KIND_P) -> int:
    """Build a plan (C: jt_plan, or jt_plan_ex when `points` / `kind` are given).

    device=-1: current CUDA device; device=-2: host-only plan.  points: None (uniform) or a sequence of d
    entries, each None (uniform axis) or n[i] nonuniform points in (0, pi), non-decreasing.  kind: JT_KIND_P
    (P~ expansions) or JT_KIND_Q (Q~ expansions)."""
    n = [int(v) for v in np.atleast_1d(n)]
    d = len(n)
    a = np.broadcast_to(np.asarray(a, dtype=np.float64), (d,)).copy()
    b = np.broadcast_to(np.asarray(b, dtype=np.float64), (d,)).copy()
    o = jt_default_opts()
    o.seed, o.k0, o.rmax_init, o.q, o.sweeps, o.device = seed, k0, rmax_init, q, sweeps, device
    h = _P()
    if points is None and kind == JT_KIND_P:
        _check(_lib.jt_plan(ctypes.byref(h), d, (ctypes.c_int64 * d)(*n), a.ctypes.data_as(_D),
                            b.ctypes.data_as(_D), float(eps), ctypes.byref(o)), "jt_plan")
        return h.value
    keep = []
    ptrs = (ctypes.c_void_p * d)()
    if points is not None:
        if len(points) != d:
            raise ValueError("points needs one entry per axis")
        for i, pts in enumerate(points):
            if pts is None:
                continue
            arr = np.ascontiguousarray(pts, dtype=np.float64)
            if arr.shape != (n[i],):
                raise ValueError(f"axis {i}: expected {n[i]} points")
            keep.append(arr)
            ptrs[i] = arr.ctypes.data
    _check(_lib.jt_plan_ex(ctypes.byref(h), d, (ctypes.c_int64 * d)(*n), a.ctypes.data_as(_D),
                           b.ctypes.data_as(_D), ctypes.cast(ptrs, ctypes.c_void_p) if points is not None else None,
                           int(kind), float(eps), ctypes.byref(o)), "jt_plan_ex")
    return h.value


def jt_forward(plan: int, coeffs, values, stream=None):
    _check(_lib.jt_forward(plan, _ptr(coeffs), _ptr(values), _stream_handle(stream)), "jt_forward")


def jt_inverse(plan: int, values, coeffs, stream=None):
    _check(_lib.jt_inverse(plan, _ptr(values), _ptr(coeffs), _stream_handle(stream)), "jt_inverse")


def jt_dist_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.jt_dist_unique_id(buf), "jt_dist_unique_id")
    return buf.raw


def jt_plan_dist(n, a, b, eps: float, uid: bytes, rank: int, nranks: int, seed: int = 0, k0: int = -1,
                 device: int = -1, flags: int = 0) -> int:
    """Slab-distributed plan with a library-owned NCCL communicator (C: jt_plan_dist_ex; flags JT_DIST_LOWMEM)."""
    n = [int(v) for v in np.atleast_1d(n)]
    d = len(n)
    a = np.broadcast_to(np.asarray(a, dtype=np.float64), (d,)).copy()
    b = np.broadcast_to(np.asarray(b, dtype=np.float64), (d,)).copy()
    o = jt_default_opts()
    o.seed, o.k0, o.device = seed, k0, device
    if len(uid) != 128:
        raise ValueError("uid must be the 128-byte NCCL unique id")
    h = _P()
    idbuf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(_lib.jt_plan_dist_ex(ctypes.byref(h), d, (ctypes.c_int64 * d)(*n), a.ctypes.data_as(_D),
                                b.ctypes.data_as(_D), float(eps), ctypes.byref(o), idbuf, rank, nranks, flags),
           "jt_plan_dist_ex")
    return h.value


def jt_local_box(plan: int, which: int, d: int):
    lo, hi = (ctypes.c_int64 * d)(), (ctypes.c_int64 * d)()
    _check(_lib.jt_local_box(plan, which, lo, hi), "jt_local_box")
    return tuple(lo), tuple(hi)


def jt_adjoint(plan: int, values, coeffs, stream=None):
    _check(_lib.jt_adjoint(plan, _ptr(values), _ptr(coeffs), _stream_handle(stream)), "jt_adjoint")


def jt_plan_kind(plan: int, axis: int):
    """(uniform: bool, kind: int) of axis `axis`."""
    u, k = ctypes.c_int(), ctypes.c_int()
    _check(_lib.jt_plan_kind(plan, axis, ctypes.byref(u), ctypes.byref(k)), "jt_plan_kind")
    return bool(u.value), k.value


def jt_forward_host(plan: int, coeffs_host: np.ndarray, values_host: np.ndarray, stream=None):
    _check(_lib.jt_forward_host(plan, _host_ptr(coeffs_host, plan, 0), _host_ptr(values_host, plan, 1),
                                _stream_handle(stream)), "jt_forward_host")


def jt_inverse_host(plan: int, values_host: np.ndarray, coeffs_host: np.ndarray, stream=None):
    _check(_lib.jt_inverse_host(plan, _host_ptr(values_host, plan, 1), _host_ptr(coeffs_host, plan, 0),
                                _stream_handle(stream)), "jt_inverse_host")


def jt_forward_host_async(plan: int, coeffs_host: np.ndarray, values_host: np.ndarray, stream=None):
    a, b = _host_ptr(coeffs_host, plan, 0), _host_ptr(values_host, plan, 1)
    _check(_lib.jt_forward_host_async(plan, a, b, _stream_handle(stream)), "jt_forward_host_async")
    _INFLIGHT.setdefault(plan, []).append((coeffs_host, values_host))


def jt_inverse_host_async(plan: int, values_host: np.ndarray, coeffs_host: np.ndarray, stream=None):
    a, b = _host_ptr(values_host, plan, 1), _host_ptr(coeffs_host, plan, 0)
    _check(_lib.jt_inverse_host_async(plan, a, b, _stream_handle(stream)), "jt_inverse_host_async")
    _INFLIGHT.setdefault(plan, []).append((values_host, coeffs_host))


def jt_host_wait(plan: int):
    try:
        _check(_lib.jt_host_wait(plan), "jt_host_wait")
    finally:
        _INFLIGHT.pop(plan, None)


DIST_MODES = {0: "single", 1: "fused", 2: "nccl_all_to_all", 3: "lowmem"}


def jt_dist_mode(plan: int) -> str:
    """'single', 'fused' (peer-store exchange), 'nccl_all_to_all' or 'lowmem' (C: jt_dist_mode)."""
    m = ctypes.c_int()
    _check(_lib.jt_dist_mode(plan, ctypes.byref(m)), "jt_dist_mode")
    return DIST_MODES[m.value]


def jt_sync(plan: int, stream=None):
    """Wait for `stream`, polling a distributed plan's communicator (JT_ERR_NCCL instead of a hang)."""
    _check(_lib.jt_sync(plan, _stream_handle(stream)), "jt_sync")


def jt_profile(plan: int, enable: bool = True):
    _check(_lib.jt_profile(plan, int(bool(enable))), "jt_profile")


def jt_last_profile(plan: int) -> dict:
    """Phase times (ms) of the most recent profiled transform: axis passes 0/1/2, the all-to-all, the whole call."""
    ms = (ctypes.c_double * 5)()
    _check(_lib.jt_last_profile(plan, ms), "jt_last_profile")
    return {"axis_ms": [ms[0], ms[1], ms[2]], "exchange_ms": ms[3], "total_ms": ms[4]}


def jt_debug_checks():
    """(enabled, violations since the last call, source line of the first) of the bounds-checked build."""
    e, c, ln = ctypes.c_int(), ctypes.c_ulonglong(), ctypes.c_int()
    _check(_lib.jt_debug_checks(ctypes.byref(e), ctypes.byref(c), ctypes.byref(ln)), "jt_debug_checks")
    return bool(e.value), int(c.value), int(ln.value)


def jt_debug_axis_pass_lim(plan: int, axis: int, inverse: bool, x_in, x_out, outer: int, inner: int, in_lim: int,
                           out_lim: int, stream=None):
    """Axis pass with caller-declared buffer extents (include/jt_debug.h): the checks build's negative control."""
    _check(_lib.jt_debug_axis_pass_lim(plan, axis, int(bool(inverse)), _ptr(x_in), _ptr(x_out), outer, inner, in_lim,
                                       out_lim, _stream_handle(stream)), "jt_debug_axis_pass_lim")


def jt_debug_vgroup_create(nranks: int, timeout_ms: int = 120000) -> int:
    g = _P()
    _check(_lib.jt_debug_vgroup_create(ctypes.byref(g), nranks, timeout_ms), "jt_debug_vgroup_create")
    return g.value


def jt_debug_vgroup_destroy(group: int):
    _check(_lib.jt_debug_vgroup_destroy(group), "jt_debug_vgroup_destroy")


def jt_debug_plan_virtual(n, a, b, eps: float, group: int, rank: int, flags: int = 0, seed: int = 0,
                          k0: int = -1, device: int = -1) -> int:
    """Rank `rank`'s distributed plan in a virtual group (include/jt_debug.h): the library's slab schedule with an
    in-process exchange instead of NCCL (tests on one GPU)."""
    n = [int(v) for v in np.atleast_1d(n)]
    d = len(n)
    a = np.broadcast_to(np.asarray(a, dtype=np.float64), (d,)).copy()
    b = np.broadcast_to(np.asarray(b, dtype=np.float64), (d,)).copy()
    o = jt_default_opts()
    o.seed, o.k0, o.device = seed, k0, device
    h = _P()
    _check(_lib.jt_debug_plan_virtual(ctypes.byref(h), d, (ctypes.c_int64 * d)(*n), a.ctypes.data_as(_D),
                                      b.ctypes.data_as(_D), float(eps), ctypes.byref(o), group, rank, flags),
           "jt_debug_plan_virtual")
    return h.value


def jt_forward_axis(plan: int, axis: int, x_in, x_out, outer: int, inner: int, stream=None):
    _check(_lib.jt_forward_axis(plan, axis, _ptr(x_in), _ptr(x_out), outer, inner, _stream_handle(stream)),
           "jt_forward_axis")


def jt_inverse_axis(plan: int, axis: int, x_in, x_out, outer: int, inner: int, stream=None):
    _check(_lib.jt_inverse_axis(plan, axis, _ptr(x_in), _ptr(x_out), outer, inner, _stream_handle(stream)),
           "jt_inverse_axis")


def jt_axis_pass(plan: int, axis: int, inverse: bool, x_in, x_out, outer: int, inner: int, in_split: int = 1,
                 out_split: int = 1, stream=None):
    """One axis pass with optional chunk-major (all-to-all) input / output layouts (include/jt.h)."""
    _check(_lib.jt_axis_pass(plan, axis, int(bool(inverse)), _ptr(x_in), _ptr(x_out), outer, inner, in_split,
                             out_split, _stream_handle(stream)), "jt_axis_pass")


def jt_axis_pass_ex(plan: int, axis: int, inverse: bool, x_in, x_out, outer: int, inner: int, in_split: int,
                    out_split: int, ostride: int, stream=None):
    """jt_axis_pass over part of the rows of a chunk-major array (include/jt.h)."""
    _check(_lib.jt_axis_pass_ex(plan, axis, int(bool(inverse)), _ptr(x_in), _ptr(x_out), outer, inner, in_split,
                                out_split, ostride, _stream_handle(stream)), "jt_axis_pass_ex")


def jt_destroy(plan: int):
    try:
        _check(_lib.jt_destroy(plan), "jt_destroy")
    finally:
        _INFLIGHT.pop(plan, None)


def jt_plan_rank(plan: int, axis: int) -> int:
    r = ctypes.c_int()
    _check(_lib.jt_plan_rank(plan, axis, ctypes.byref(r)), "jt_plan_rank")
    return r.value


def jt_plan_info(plan: int, axis: int) -> dict:
    n, N, k0, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
    _check(_lib.jt_plan_info(plan, axis, ctypes.byref(n), ctypes.byref(N), ctypes.byref(k0), ctypes.byref(r)),
           "jt_plan_info")
    return {"n": n.value, "N": N.value, "k0": k0.value, "r": r.value}


def jt_plan_nodes(plan: int, axis: int):
    n = jt_plan_info(plan, axis)["n"]
    t = np.empty(n)
    w = np.empty(n)
    _check(_lib.jt_plan_nodes(plan, axis, t.ctypes.data, w.ctypes.data), "jt_plan_nodes")
    return t, w


def jt_plan_factors(plan: int, axis: int):
    """(u (n x r complex), v (r x N complex), phiv (n x k0), bins (n int32)) — see include/jt.h."""
    info = jt_plan_info(plan, axis)
    n, N, k0, r = info["n"], info["N"], info["k0"], info["r"]
    u = np.zeros((n, r), dtype=np.complex128)
    v = np.zeros((r, N), dtype=np.complex128)
    phiv = np.zeros((n, k0), dtype=np.float64)
    bins = np.zeros(n, dtype=np.int32)
    _check(_lib.jt_plan_factors(plan, axis, u.ctypes.data, v.ctypes.data, phiv.ctypes.data, bins.ctypes.data),
           "jt_plan_factors")
    return u, v, phiv, bins


def jt_plan_sigma(plan: int, axis: int):
    cnt, rmax = ctypes.c_int(), ctypes.c_int()
    _check(_lib.jt_plan_sigma(plan, axis, None, ctypes.byref(cnt), ctypes.byref(rmax)), "jt_plan_sigma")
    s = np.zeros(cnt.value)
    _check(_lib.jt_plan_sigma(plan, axis, s.ctypes.data, ctypes.byref(cnt), ctypes.byref(rmax)), "jt_plan_sigma")
    return s, rmax.value


def jt_debug_pair_factors(plan: int, axis: int):
    """The paired-real-term factor set of the forward passes (include/jt_debug.h): None if the axis has none, else
    (u (n x 2r complex: P, conj(Q) per pair), v (r x N complex), phiv (n x k0), bins (n int32), rreal)."""
    r, rr = ctypes.c_int(), ctypes.c_int()
    _lib.jt_debug_pair_factors.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    _check(_lib.jt_debug_pair_factors(plan, axis, ctypes.byref(r), ctypes.byref(rr), None, None, None, None),
           "jt_debug_pair_factors")
    if r.value == 0:
        return None
    info = jt_plan_info(plan, axis)
    n, N, k0 = info["n"], info["N"], info["k0"]
    u = np.zeros((n, 2 * r.value), dtype=np.complex128)
    v = np.zeros((r.value, N), dtype=np.complex128)
    phiv = np.zeros((n, k0), dtype=np.float64)
    bins = np.zeros(n, dtype=np.int32)
    _check(_lib.jt_debug_pair_factors(plan, axis, ctypes.byref(r), ctypes.byref(rr), u.ctypes.data, v.ctypes.data,
                                      phiv.ctypes.data, bins.ctypes.data), "jt_debug_pair_factors")
    return u, v, phiv, bins, rr.value


def jt_debug_modified_pq(a: float, b: float, t, kmax: int):
    """P~_k(t), Q~_k(t) for k = 0..kmax by the plan's route (include/jt_debug.h)."""
    t = np.ascontiguousarray(np.atleast_1d(t), dtype=np.float64)
    P = np.zeros((t.size, kmax + 1))
    Q = np.zeros((t.size, kmax + 1))
    _check(_lib.jt_debug_modified_pq(a, b, t.size, t.ctypes.data, kmax, P.ctypes.data, Q.ctypes.data),
           "jt_debug_modified_pq")
    return P, Q


class Plan:
    """Owning wrapper: Plan(n, a, b, eps) -> .forward(x) / .inverse(y) on CUDA float64 tensors."""

    def __init__(self, n, a, b, eps: float = 1e-12, **kw):
        self.shape = tuple(int(v) for v in np.atleast_1d(n))
        self.d = len(self.shape)
        self.handle = jt_plan(self.shape, a, b, eps, **kw)

    def _out(self, x, out):
        if out is None:
            import torch
            out = torch.empty(self.shape, dtype=torch.float64, device=x.device)
        if tuple(x.shape) != self.shape or tuple(out.shape) != self.shape:
            raise ValueError(f"expected shape {self.shape}")
        return out

    def forward(self, coeffs, out=None, stream=None):
        out = self._out(coeffs, out)
        jt_forward(self.handle, coeffs, out, stream)
        return out

    def inverse(self, values, out=None, stream=None):
        out = self._out(values, out)
        jt_inverse(self.handle, values, out, stream)
        return out

    def adjoint(self, values, out=None, stream=None):
        out = self._out(values, out)
        jt_adjoint(self.handle, values, out, stream)
        return out

    def kind(self, axis: int = 0):
        return jt_plan_kind(self.handle, axis)

    def forward_host(self, coeffs: np.ndarray, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(self.shape)
        out = np.empty(self.shape) if out is None else out
        jt_forward_host(self.handle, coeffs, out, stream)
        return out

    def inverse_host(self, values: np.ndarray, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        values = np.ascontiguousarray(values, dtype=np.float64).reshape(self.shape)
        out = np.empty(self.shape) if out is None else out
        jt_inverse_host(self.handle, values, out, stream)
        return out

    def forward_host_async(self, coeffs: np.ndarray, out: np.ndarray, stream=None):
        """Enqueue a host-buffer forward transform (results valid after wait_host()); see include/jt.h."""
        jt_forward_host_async(self.handle, coeffs, out, stream)
        return out

    def wait_host(self):
        jt_host_wait(self.handle)

    def rank(self, axis: int = 0) -> int:
        return jt_plan_rank(self.handle, axis)

    def info(self, axis: int = 0) -> dict:
        return jt_plan_info(self.handle, axis)

    def nodes(self, axis: int = 0):
        return jt_plan_nodes(self.handle, axis)

    def factors(self, axis: int = 0):
        return jt_plan_factors(self.handle, axis)

    def sigma(self, axis: int = 0):
        return jt_plan_sigma(self.handle, axis)

    def close(self):
        if getattr(self, "handle", None):
            jt_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
