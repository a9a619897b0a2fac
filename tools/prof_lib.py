"""One forward + one inverse of a BASELINE config through a given libjt build (raw ctypes; ncu captures)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import seeded_inputs as si  # noqa: E402

lib, name = sys.argv[1], sys.argv[2]
what = sys.argv[3] if len(sys.argv) > 3 else "fi"
L = ctypes.CDLL(lib)
P = ctypes.c_void_p
L.jt_plan.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_double, ctypes.c_void_p]
for f in ("jt_forward", "jt_inverse"):
    getattr(L, f).argtypes = [P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
c = si.CONFIGS[name]
d = len(c["n"])
h = P()
assert L.jt_plan(ctypes.byref(h), d, (ctypes.c_int64 * d)(*c["n"]), (ctypes.c_double * d)(*c["a"]),
                 (ctypes.c_double * d)(*c["b"]), c["eps"], None) == 0
x = torch.from_numpy(si.gaussian(c["n"], 0)).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
if "f" in what:
    L.jt_forward(h, x.data_ptr(), y.data_ptr(), s)
if "i" in what:
    L.jt_inverse(h, y.data_ptr(), x.data_ptr(), s)
torch.cuda.synchronize()
print("ok", lib, name)
