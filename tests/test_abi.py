"""CPU checks of the C-ABI boundary (no compute calls need a GPU): the library loads, exports every
symbol declared in include/*.h, and reports argument / domain errors as documented in include/jt.h."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1901_07275_b200 as jt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("jt.h", "jt_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(jt_[a-z_0-9]+)\s*\(", src))
    return names


def test_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 16
    lib = ctypes.CDLL(jt.LIB_PATH)
    for name in sorted(names):
        assert hasattr(lib, name), f"libjt.so does not export {name}"
    assert names <= set(jt.EXPORTED), names - set(jt.EXPORTED)


def test_version_and_defaults():
    assert "sm_100a" in jt.jt_version()
    o = jt.jt_default_opts()
    assert (o.seed, o.k0, o.rmax_init, o.q, o.sweeps, o.device) == (0, -1, 0, 3, 2, -1)  # k0 -1 = auto


@pytest.mark.parametrize("kw,code", [
    (dict(n=[64], a=[1.0], b=[0.0]), jt.JT_ERR_DOMAIN),
    (dict(n=[64], a=[0.0], b=[-1.0]), jt.JT_ERR_DOMAIN),
    (dict(n=[1], a=[0.0], b=[0.0]), jt.JT_ERR_ARG),
    (dict(n=[8192], a=[0.0], b=[0.0]), jt.JT_ERR_ARG),
    (dict(n=[8, 8, 8, 8], a=[0.0] * 4, b=[0.0] * 4), jt.JT_ERR_ARG),
    (dict(n=[64], a=[0.0], b=[0.0], eps=1e-20), jt.JT_ERR_ARG),
    (dict(n=[64], a=[0.0], b=[0.0], k0=33), jt.JT_ERR_ARG),
    (dict(n=[64], a=[0.0], b=[0.0], k0=-2), jt.JT_ERR_ARG),
])
def test_plan_argument_errors(kw, code):
    with pytest.raises(jt.JTError) as ei:
        jt.jt_plan(device=-2, **kw)
    assert ei.value.status == code
    assert len(jt._lib.jt_last_error()) > 0


def test_host_only_plan_refuses_device_calls():
    p = jt.Plan(64, 0.1, -0.2, device=-2)
    x = np.zeros(64)
    with pytest.raises(jt.JTError) as ei:
        jt.jt_forward(p.handle, x, x, stream=0)
    assert ei.value.status == jt.JT_ERR_ARG
    info = p.info()
    assert info["n"] == 64 and info["N"] == 64 and info["k0"] in (27, 32) and info["r"] == p.rank()
    p.close()


def test_destroy_null_ok():
    assert jt._lib.jt_destroy(None) == jt.JT_OK


def test_last_launches_arguments():
    assert jt._lib.jt_last_launches(None, None) == jt.JT_ERR_ARG
    p = jt.Plan(64, 0.1, -0.2, device=-2)
    assert jt.jt_last_launches(p) == 0  # no transform yet
    p.close()


def test_debug_hook_errors():
    with pytest.raises(jt.JTError):
        jt.jt_debug_modified_pq(1.5, 0.0, [1.0], 3)


def test_rank_growth_cap_is_numeric_error():
    """SURVEY.md §8(b) / SPEC S:210 growth cap (reading R25): the adaptive rank may grow beyond its start
    value only up to min(n, n - k0) / 4.  n = 64 (k0 = 27: 37 columns, cap 9) started at rmax 4 needs rank ~10."""
    with pytest.raises(jt.JTError) as ei:
        jt.jt_plan(64, 0.45, -0.45, 1e-12, rmax_init=4, device=-2)
    assert ei.value.status == jt.JT_ERR_NUMERIC
    assert "growth cap" in str(ei.value)
    p = jt.Plan(64, 0.45, -0.45, 1e-12, device=-2)  # the default start (32) factors B without growing
    assert 1 <= p.rank() <= 32
    p.close()
    q = jt.Plan(1024, 0.25, -0.3, 1e-12, rmax_init=4, device=-2)  # 4 -> 8 -> 16 -> 32, cap 249: converges
    assert q.rank() == jt.Plan(1024, 0.25, -0.3, 1e-12, device=-2).rank()
    q.close()


def test_host_buffers_checked_before_the_call():
    """*_host calls check their numpy buffers against the plan's local element count (the C side reads and writes
    exactly that many doubles) before any pointer crosses the ABI."""
    p = jt.Plan((8, 12), (0.1, 0.2), (0.0, 0.1), device=-2)
    good = np.zeros((8, 12))
    for bad in (np.zeros((8, 11)), np.zeros((8, 12), dtype=np.float32), np.zeros((12, 8)).T):
        with pytest.raises((ValueError, TypeError)):
            jt.jt_forward_host(p.handle, bad, good)
        with pytest.raises((ValueError, TypeError)):
            jt.jt_forward_host_async(p.handle, good, bad)
    with pytest.raises(TypeError):
        jt.jt_inverse_host(p.handle, [0.0] * 96, good)
    assert p.handle not in jt._INFLIGHT
    p.close()


def test_dist_and_debug_argument_errors():
    n = (ctypes.c_int64 * 2)(8, 8)
    a = (ctypes.c_double * 2)(0.1, 0.1)
    h = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    o = jt.jt_default_opts()
    o.device = -2
    assert jt._lib.jt_plan_dist_ex(ctypes.byref(h), 2, n, a, a, 1e-12, ctypes.byref(o), uid, 0, 2, 0) == jt.JT_ERR_ARG
    o.device = -1
    assert jt._lib.jt_plan_dist_ex(ctypes.byref(h), 2, n, a, a, 1e-12, ctypes.byref(o), uid, 0, 2, 4) == jt.JT_ERR_ARG
    assert jt._lib.jt_plan_dist_ex(ctypes.byref(h), 2, n, a, a, 1e-12, ctypes.byref(o), uid, 0, 33, 0) == jt.JT_ERR_ARG
    assert jt._lib.jt_plan_dist_ex(ctypes.byref(h), 2, n, a, a, 1e-12, ctypes.byref(o), None, 0, 2, 0) == jt.JT_ERR_ARG
    with pytest.raises(jt.JTError):
        jt.jt_debug_vgroup_create(0)
    g = jt.jt_debug_vgroup_create(2, 1000)
    with pytest.raises(jt.JTError):  # a virtual rank outside the group
        jt.jt_debug_plan_virtual((8, 8), 0.1, 0.1, 1e-12, g, 2)
    jt.jt_debug_vgroup_destroy(g)
    p = jt.Plan(16, 0.1, -0.2, device=-2)
    jt.jt_profile(p.handle, True)
    with pytest.raises(jt.JTError) as ei:  # no profiled call yet
        jt.jt_last_profile(p.handle)
    assert ei.value.status == jt.JT_ERR_ARG
    with pytest.raises(jt.JTError):
        jt.jt_sync(p.handle, 0)  # host-only plan
    p.close()
