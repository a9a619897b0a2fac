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
