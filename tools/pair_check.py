"""Dev tool: the paired-real-term forward (Cfg::PAIR, JT_PAIR) against the oracle and against the unpaired forward,
with timings.  Run on a GPU box:  python tools/pair_check.py"""
import os
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import oracle
    import paper_1901_07275_b200 as jt
    import seeded_inputs as si
    out = {}
    cases = [((512,), (0.25,), (-0.25,)), ((512, 24), (0.1, 0.2), (-0.4, 0.3)), ((40, 512), (0.2, 0.0), (0.3, 0.0)),
             ((512, 512), (0.25, -0.3), (-0.25, 0.2)), ((8, 512, 512), (0.1, 0.25, -0.45), (0.2, -0.25, 0.45)),
             ((256,), (0.2,), (-0.2,)), ((256, 40), (-0.4, 0.1), (0.3, 0.2)), ((24, 256, 256), (0.0, 0.35, 0.1), (0.0, 0.1, -0.4)),
             ((4096,), (0.45,), (-0.45,)), ((3, 4096), (0.1, 0.0), (0.1, 0.0)), ((4096, 5), (-0.3, 0.0), (0.3, 0.0))]
    for shape, a, b in cases:
        p = jt.Plan(shape, a, b, 1e-12)
        x = si.gaussian(shape, seed=1)
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        jt.jt_forward(p.handle, xd, yd)
        torch.cuda.synchronize()
        ref = oracle.forward(x, a, b)
        e = float(np.linalg.norm(yd.cpu().numpy() - ref) / np.linalg.norm(ref))
        zd = torch.empty_like(xd)
        jt.jt_inverse(p.handle, yd, zd)
        torch.cuda.synchronize()
        ert = float(np.linalg.norm(zd.cpu().numpy() - x) / np.linalg.norm(x))
        out["x".join(map(str, shape))] = {"fwd_err": e, "roundtrip": ert, "ranks": [p.rank(i) for i in range(len(shape))],
                                           "pairs": [(jt.jt_debug_pair_factors(p.handle, i) or [None, np.zeros((0, 0))])[1].shape[0]
                                                     for i in range(len(shape))]}
        p.close()
    # timing: the BASELINE configs' forwards, sampled oracle check of the full-size outputs
    for name in ("cfg2_2d_256", "cfg4_3d_256", "cfg3_2d_4096", "cfg5_3d_512", "grid_2048x2048", "grid_2048x2048x8"):
        c = si.CONFIGS[name] if name in si.CONFIGS else {
            "n": tuple(int(v) for v in name[5:].split("x")), "eps": 1e-12,
            "a": (0.25, -0.3, 0.1)[:len(name[5:].split("x"))], "b": (-0.25, 0.2, 0.3)[:len(name[5:].split("x"))]}
        shape = tuple(c["n"])
        p = jt.Plan(shape, c["a"], c["b"], c["eps"])
        x = si.gaussian(shape, seed=0)
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        for _ in range(3):
            jt.jt_forward(p.handle, xd, yd)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            jt.jt_forward(p.handle, xd, yd)
        e1.record()
        torch.cuda.synchronize()
        idx = np.stack([np.random.default_rng(3).integers(0, shape[i], 32) for i in range(len(shape))], axis=1)
        ref = oracle.forward_at(x, c["a"], c["b"], idx)
        got = yd.cpu().numpy()[tuple(idx[:, i] for i in range(len(shape)))]
        zd = torch.empty_like(xd)
        for _ in range(3):
            jt.jt_inverse(p.handle, yd, zd)
        torch.cuda.synchronize()
        rt = float(np.linalg.norm(zd.cpu().numpy() - x) / np.linalg.norm(x))
        i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        i0.record()
        for _ in range(20):
            jt.jt_inverse(p.handle, yd, zd)
        i1.record()
        torch.cuda.synchronize()
        jt.jt_inverse(p.handle, xd, zd)  # the inverse of independent values against the oracle's inverse, sampled
        torch.cuda.synchronize()
        iref = oracle.inverse_at(x, c["a"], c["b"], idx)
        igot = zd.cpu().numpy()[tuple(idx[:, i] for i in range(len(shape)))]
        out[name] = {"fwd_ms": e0.elapsed_time(e1) / 20, "inv_ms": i0.elapsed_time(i1) / 20, "roundtrip": rt,
                     "inv_sampled_err": float(np.linalg.norm(igot - iref) / np.linalg.norm(iref)),
                     "sampled_err": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                     "ranks": [p.rank(i) for i in range(len(shape))],
                     "pairs": [(jt.jt_debug_pair_factors(p.handle, i) or [None, np.zeros((0, 0))])[1].shape[0] for i in range(len(shape))]}
        p.close()
    shape = (512, 512, 512)
    p = jt.Plan(shape, (0.25,) * 3, (-0.25,) * 3, 1e-12)
    xd = torch.from_numpy(si.gaussian(shape, seed=0)).cuda()
    yd = torch.empty_like(xd)
    jt.jt_forward(p.handle, xd, yd)
    torch.cuda.synchronize()
    # sampled oracle check of the full-size output
    idx = np.stack([np.random.default_rng(3).integers(0, 512, 64) for _ in range(3)], axis=1)
    x = si.gaussian(shape, seed=0)
    ref = oracle.forward_at(x, (0.25,) * 3, (-0.25,) * 3, idx)
    got = yd.cpu().numpy()[idx[:, 0], idx[:, 1], idx[:, 2]]
    out["512^3_sampled_err"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    print("RESULT " + json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for pair in ("1", "0"):
            env = dict(os.environ, JT_PAIR=pair)
            r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=900)
            print("JT_PAIR=" + pair, r.returncode)
            print(r.stdout[-3000:])
            print(r.stderr[-3000:])
