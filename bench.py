"""Benchmark: fp64 uniform Jacobi transform (arXiv 1901.07275 hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]
    torchrun --nproc-per-node N bench.py --gpus N ...          (slab-distributed, NCCL all-to-all)

Workload (BASELINE.json configs[4], the largest grid, the one the metric's 1/2/4/8-GPU scaling is
quoted on): 3D uniform forward transform, 512 x 512 x 512 (134M fp64 coefficients), (a,b) =
(0.25,-0.25) on every axis, eps = 1e-12, coefficients iid N(0,1) from seed 0.  A step = one whole
forward transform (all three fused axis passes; with N > 1 also the all-to-all).  Inputs (1.07 GB) are
larger than L2 (126 MB), so no extra flush is needed between steps.

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the only reference that
exists for this paper: BASELINE.json published = {}) on host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# NCCL's log (NCCL_DEBUG=VERSION is the GPU image's default; INFO shows the communicators' ranks) goes to stderr,
# so stdout carries only the one JSON line and the driver can still read NCCL's banner and init lines
if os.environ.get("NCCL_DEBUG") and not os.environ.get("NCCL_DEBUG_FILE"):
    os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
sys.path.insert(0, ROOT)

import seeded_inputs as si  # noqa: E402

METRIC = "Jacobi-transform coefficients/sec (fp64, 2D/3D) and % of HBM roofline at 1/2/4/8 GPUs"
FP64_PEAK_TFLOPS = 37.0   # measured DFMA peak (profiles/fp64_peak_r01.json); derived 148*64*2*1.965 GHz = 37.2
K0 = 27


def algorithmic_flops_per_point(N: int, r: int, k0: int = K0) -> float:
    """per axis pass per point r (5 log2 N + 6) + 2 k0 (conventional FFT count; N = the
    axis's FFT length, k0 = its dense-block width as the plan chose it)."""
    return r * (5 * np.log2(N) + 6) + 2 * k0


def executed_flops_per_point(N: int, ffts: int, k0: int = K0) -> float:
    """The same count for the schedule a paired axis executes (DESIGN.md §6 "Two real rank terms per FFT"): per FFT
    5 log2 N + 2 (column scale, complex x real) + 8 (two factor rows per node: P Z[m] and conj(Q) Z[N-1-m])."""
    return ffts * (5 * np.log2(N) + 10) + 2 * k0


def ffts_per_line(handle, axis: int, rank: int, nlines: int) -> int:
    """Complex FFTs per line of a forward pass of this axis: the paired factor set's pair count where the plan has
    one and the launch has enough lines for it (csrc/tuning.h JT_PAIR_MIN_LINES), else the rank."""
    import paper_1901_07275_b200 as jt
    got = jt.jt_debug_pair_factors(handle, axis)
    return int(got[1].shape[0]) if (got is not None and nlines >= 2400) else int(rank)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        mhz, maxmhz, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                mhz.append(float(f[1]))
                maxmhz.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": max(maxmhz) if maxmhz else None,
                "reasons": sorted(reasons), "samples": len(mhz), "power_w_max": max(power) if power else None}


def cpu_oracle_rate(cfg, max_seconds: float = 30.0):
    """The oracle (oracle/jacobi.py) as it stands, on this host's cores: full forward of the config if it
    fits the time bound, else a slab of it.  Returns (coefficients/s, sample description, threads)."""
    import oracle
    shape, a, b = cfg["n"], cfg["a"], cfg["b"]
    pts, kind = si.config_points(cfg), cfg.get("kind", 0)
    for ax in range(len(shape)):  # Phi construction is the oracle's "fac"; not part of the apply rate
        oracle.axis_matrix(shape[ax], a[ax], b[ax], None if pts is None else pts[ax], kind)
    x = si.gaussian(shape, seed=0)
    t0 = time.perf_counter()
    oracle.forward_ex(x, a, b, pts, kind)
    dt = time.perf_counter() - t0
    threads = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        threads = max(int(i.get("num_threads", 1)) for i in threadpool_info()) or threads
    except Exception:
        pass
    desc = f"full {'x'.join(map(str, shape))} forward (dense separable mode products, fp64 BLAS), 1 run, {dt:.1f} s"
    return float(np.prod(shape)) / dt, desc, threads


def cpu_oracle_rate_one_core(cfg):
    """The oracle on ONE core (the paper's single-processor setting), on a bounded
    sample: axes d-1..1 on an x-slab of n0/32 planes (the whole 1D transform for d = 1).  Returns
    (coefficients/s of the whole transform at that per-point cost, sample description) or None."""
    import oracle
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        return None
    shape, a, b = cfg["n"], cfg["a"], cfg["b"]
    pts, kind = si.config_points(cfg), cfg.get("kind", 0)
    x = si.gaussian(shape, seed=0)
    d = len(shape)
    for ax in range(d):  # the matrices (the oracle's "fac") are built outside the timed region
        oracle.axis_matrix(shape[ax], a[ax], b[ax], None if pts is None else pts[ax], kind)
    with threadpool_limits(limits=1):
        if d == 1:
            t0 = time.perf_counter()
            oracle.forward_ex(x, a, b, pts, kind)
            dt = time.perf_counter() - t0
            return float(x.size) / dt, f"full 1D forward on one core, {dt * 1e3:.2f} ms"
        slab = max(1, shape[0] // 32)
        xs = np.ascontiguousarray(x[:slab])
        t0 = time.perf_counter()
        oracle.forward_axes(xs, a, b, axes=list(range(d - 1, 0, -1)), points=pts, kind=kind)
        dt = time.perf_counter() - t0
    return (xs.size * (d - 1) / dt / d,
            f"one core: axes {d - 1}..1 on an x-slab of {slab} planes ({xs.size * (d - 1)} axis-pass points, "
            f"{dt:.2f} s); value = axis-pass points/s / d")


def run_reference(args, cfg, rank: int):
    """--impl reference: the CPU oracle timed on the host (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    shape, a, b = cfg["n"], cfg["a"], cfg["b"]
    pts, kind = si.config_points(cfg), cfg.get("kind", 0)
    for ax in range(len(shape)):
        oracle.axis_matrix(shape[ax], a[ax], b[ax], None if pts is None else pts[ax], kind)
    # Bounded sample per step (1/8 of the transform's work): the last d-1 axis passes on an x-slab of
    # n0/8 planes, and the axis-0 pass on the full-height block of the first n1/8 columns.  Both have the
    # exact per-point cost of the full transform's passes.
    x = si.gaussian(shape, seed=0)
    slab = max(1, shape[0] // 8)
    xs = np.ascontiguousarray(x[:slab])

    def step():
        y = oracle.forward_axes(xs, a, b, axes=list(range(len(shape) - 1, 0, -1)), points=pts, kind=kind)
        # axis 0 on the full-height columns of the first slab/8 columns of axis 1 (bounded work)
        cols = np.ascontiguousarray(x[:, : max(1, shape[1] // 8)])
        oracle.forward_axes(cols, a, b, axes=[0], points=pts, kind=kind)
        return y

    pts_step = xs.size + (x[:, : max(1, shape[1] // 8)].size if len(shape) > 1 else 0)
    pass_pts = xs.size * (len(shape) - 1) + (x[:, : max(1, shape[1] // 8)].size if len(shape) > 1 else 0)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    # rate in coefficients/s of the whole transform: (axis-pass points per second) / d
    value = pass_pts / dt / len(shape)
    threads = os.cpu_count()
    sample = (f"per step 1/8 of the transform's work: axes {len(shape)-1}..1 on an x-slab of {slab} planes + "
              f"axis 0 on the first n1/8 columns ({pass_pts} axis-pass points); value = axis-pass points/s / d")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "coefficients/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1), seed 0",
            "config": config_block(args, cfg, None),
            "cpu_baseline": {"value": value, "unit": "coefficients/s", "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "coefficients/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(args, cfg, ranks, k0s=None):
    kindtxt = ("nonuniform (random points)" if cfg.get("points") else "uniform") + (
        " second-kind Q~" if cfg.get("kind", 0) == 1 else "")
    return {"workload": f"{args.config}: {'x'.join(map(str, cfg['n']))} {kindtxt} forward, (a,b)="
                        f"{list(zip(cfg['a'], cfg['b']))}, eps={cfg['eps']}",
            "model": "none (transform)", "global_batch": 1, "seq_len": int(np.prod(cfg["n"])),
            "ranks_per_axis": ranks, "k0_per_axis": k0s, "parallelism": f"slab{args.gpus}" if (args.gpus > 1 or args.slab) else "single",
            "l2_policy": "inputs (8 B x prod(n)) larger than the 126 MB L2; no extra flush"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5_3d_512", choices=list(si.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--slab", action="store_true",
                    help="run the slab-distributed path (NCCL all-to-all) even at world size 1 (path check)")
    args = ap.parse_args()
    cfg = si.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    args.warmup = max(args.warmup, 3)
    slab = world > 1 or args.slab

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import paper_1901_07275_b200 as jt
    torch.cuda.set_device(local_rank)
    dist = None
    if slab:
        import torch.distributed as dist
        if "RANK" not in os.environ:  # `--slab` without torchrun: a world of one over NCCL
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        from paper_1901_07275_b200.dist import LibSlabPlan
    shape, a, b, eps = cfg["n"], cfg["a"], cfg["b"], cfg["eps"]
    d = len(shape)
    stream = torch.cuda.current_stream()

    if not slab:
        t_fac = time.perf_counter()
        plan = jt.Plan(shape, a, b, eps, points=si.config_points(cfg), kind=cfg.get("kind", 0))
        fac_s = time.perf_counter() - t_fac  # the paper's "fac": host plan + upload, untimed
        ranks = [plan.rank(i) for i in range(d)]
        infos = [plan.info(i) for i in range(d)]
        k0s = [inf["k0"] for inf in infos]
        x = torch.from_numpy(si.gaussian(shape, seed=0)).cuda()
        y = torch.empty_like(x)
        strides = []
        for ax in range(d - 1, -1, -1):
            strides.append((ax, int(np.prod(shape[:ax])), int(np.prod(shape[ax + 1:]))))

        def step(evs=None, count=None):
            src = x
            for i, (ax, outer, inner) in enumerate(strides):
                if evs is not None:
                    evs[i].record(stream)
                jt.jt_forward_axis(plan.handle, ax, src, y, outer, inner, stream)
                if count is not None:  # kernels this axis call enqueued (the pass, + a reduction if term-split)
                    count[0] += jt.jt_last_launches(plan.handle)
                src = y
            if evs is not None:
                evs[-1].record(stream)
        cnt = [0]
        step(count=cnt)  # (an extra warm-up step) counts the library's kernel launches per step
        launches_per_step = cnt[0]
        local_points = int(np.prod(shape))
    else:
        t_fac = time.perf_counter()
        plan = LibSlabPlan(shape, a, b, eps, dist)
        fac_s = time.perf_counter() - t_fac
        ranks = plan.ranks
        k0s = [inf["k0"] for inf in plan.infos]
        x = plan.local_input(torch.from_numpy(si.gaussian(shape, seed=0)))
        step = plan.make_forward_step(x)
        step()  # (an extra warm-up step) counts the library's kernel launches per step
        launches_per_step = jt.jt_last_launches(plan.handle)
        local_points = x.numel()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    time.sleep(0.3)
    nev = (d + 1) if not slab else 2
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        if not slab:
            step(evs[k])
        else:
            step()
    end.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    ms_total = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    total_points = float(np.prod(shape))
    value = total_points / (ms_step * 1e-3)

    roofline = None
    per_axis_ms = None
    step_stats = None
    slab_phases = None
    if slab:
        # phase split of the distributed step (jt_profile / jt_last_profile: CUDA events inside the library's
        # schedule), taken on extra profiled steps AFTER the timed region so the timed steps carry no host syncs
        jt.jt_profile(plan.handle, True)
        prof = []
        for _ in range(max(3, min(args.steps, 10))):
            step()
            prof.append(jt.jt_last_profile(plan.handle))
        jt.jt_profile(plan.handle, False)
        med = lambda v: float(np.median(v))  # noqa: E731
        axis_ms = [med([p["axis_ms"][i] for p in prof]) for i in range(3)][:d]
        slab_phases = {"axis_ms": [round(v, 4) for v in axis_ms], "exchange_ms": round(med([p["exchange_ms"] for p in prof]), 4),
                       "call_ms": round(med([p["total_ms"] for p in prof]), 4),
                       "exchange_mode": jt.jt_dist_mode(plan.handle),
                       "note": "rank-local CUDA events (library jt_profile), median of extra profiled steps after the "
                               "timed region; fused mode: the axis-1 pass stores each block into its owner's receive "
                               "buffer (NVLink peer stores) and exchange_ms is the closing barrier; nccl_all_to_all "
                               "mode: axis 1 runs in row chunks overlapped with the all-to-all"}
        if dist is not None:
            t = torch.tensor([slab_phases["call_ms"], slab_phases["exchange_ms"]] + axis_ms, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            slab_phases["max_over_ranks"] = [round(float(v), 4) for v in t.cpu()]
        # dominant kernel: the axis-0 pass (one whole launch on the received y-slab, n0 x (n1/G)(n2) points)
        flops = algorithmic_flops_per_point(plan.infos[0]["N"], ranks[0], k0s[0]) * local_points
        achieved = flops / (axis_ms[0] * 1e-3) / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                    "kernel": f"fwd_axis_kernel<N={shape[0]}> (axis 0, on this rank's y-slab)",
                    "flops_per_launch": flops,
                    "peak_source": "FP64 DFMA measured 37.0 TF/s burst = sustained (profiles/fp64_peak_r01.json)"}
    if not slab:
        per_axis = np.array([[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(d)] for k in range(args.steps)])
        per_axis_ms = per_axis.mean(axis=0)  # in launch order (axis d-1 first)
        step_ms = per_axis.sum(axis=1)       # each timed step (CUDA events on the launching stream)
        step_stats = {"median": round(float(np.median(step_ms)), 4), "min": round(float(step_ms.min()), 4),
                      "max": round(float(step_ms.max()), 4)}
        # dominant kernel: the fused forward axis pass (all d launches are this kernel; take the slowest axis)
        i_dom = int(np.argmax(per_axis_ms))
        ax_dom = strides[i_dom][0]
        flops = algorithmic_flops_per_point(infos[ax_dom]["N"], ranks[ax_dom], k0s[ax_dom]) * total_points
        achieved = flops / (per_axis_ms[i_dom] * 1e-3) / 1e12
        # what the launch executes: paired axes run ~half as many FFTs as the rank (two real terms per complex FFT)
        nfft = [ffts_per_line(plan.handle, ax, ranks[ax], total_points // shape[ax]) for ax in range(d)]
        flops_x = executed_flops_per_point(infos[ax_dom]["N"], nfft[ax_dom], k0s[ax_dom]) * total_points \
            if nfft[ax_dom] != ranks[ax_dom] else flops
        achieved_x = flops_x / (per_axis_ms[i_dom] * 1e-3) / 1e12
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
                prof = json.load(f)
            traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        hbm_bytes = 16.0 * total_points
        roofline = {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                    "kernel": f"fwd_axis_kernel<N={shape[ax_dom]}> (axis {ax_dom})",
                    "flops_per_launch": flops,
                    # `achieved` / `frac` count the algorithmic work of SURVEY.md §8(d) (the paper's schedule: one
                    # complex FFT per rank term, r = the plan's rank); `executed` counts the FFTs the launch really
                    # runs
                    "executed": {"ffts_per_line_per_axis": nfft, "flops_per_launch": flops_x, "achieved": achieved_x,
                                 "frac": achieved_x / FP64_PEAK_TFLOPS},
                    "per_axis_ms_launch_order": [round(float(v), 4) for v in per_axis_ms],
                    "hbm_algorithmic_GBps": hbm_bytes / (per_axis_ms[i_dom] * 1e-3) / 1e9,
                    # ncu-measured DRAM bytes of one launch (profiles/ncu_summary.json) over the live launch time
                    "hbm_measured_frac": (traffic / (per_axis_ms[i_dom] * 1e-3) / 1e9 / load_peaks()["hbm_gbs"]
                                          if traffic else None),
                    "hbm_frac_of_measured": hbm_bytes / (per_axis_ms[i_dom] * 1e-3) / 1e9 / load_peaks()["hbm_gbs"],
                    # SURVEY.md §8(d) "north-star model": the HBM traffic an unfused one-rank-term-per-pass schedule
                    # would move (24 B per point per term: read input, read + write the accumulator) over the
                    # measured step time, as a fraction of the measured HBM bandwidth (a fusion gain; may exceed 1)
                    "north_star_hbm_model_frac": 24.0 * total_points * sum(ranks) / (ms_step * 1e-3) / 1e9
                                                 / load_peaks()["hbm_gbs"],
                    "peak_source": "FP64 DFMA measured 37.0 TF/s burst = sustained (profiles/fp64_peak_r01.json); "
                                   "148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz = 37.2 derived"}

    e2e = None
    if not slab and not args.no_e2e:
        xh = torch.from_numpy(si.gaussian(shape, seed=0)).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        xn, yn = xh.numpy(), yh.numpy()
        # a stream of end-to-end transforms through the public async host API: each step copies its input from
        # pinned host memory and its result back; consecutive steps overlap the two PCIe directions
        xs_h = [xn, torch.from_numpy(si.gaussian(shape, seed=1)).pin_memory().numpy()]
        ys_h = [yn, torch.empty_like(xh).pin_memory().numpy()]
        for k in range(2):  # warm both staging slots
            plan.forward_host_async(xs_h[k], ys_h[k], stream)
        plan.wait_host()
        e2e_steps = max(4, min(args.steps, 8))
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        for k in range(e2e_steps):
            plan.forward_host_async(xs_h[k % 2], ys_h[k % 2], stream)
        plan.wait_host()
        torch.cuda.synchronize()
        ms_e2e = (time.perf_counter() - t_start) * 1e3 / e2e_steps
        e2e = {"value": total_points / (ms_e2e * 1e-3), "unit": "coefficients/s",
               "h2d_bytes_per_step": int(8 * total_points), "d2h_bytes_per_step": int(8 * total_points),
               "ms_per_step": ms_e2e,
               "api": "jt_forward_host_async x steps + jt_host_wait, host wall clock (pinned host buffers; each "
                      "step: chunked H2D overlapped with the axis-2/1 passes, axis-0 column blocks overlapped with "
                      "the D2H, and consecutive steps overlapping the two PCIe directions)"}
    elif slab and not args.no_e2e:
        # a stream of end-to-end transforms of this rank's slab through the async host API (two staging slots:
        # consecutive steps overlap the two PCIe directions), host wall clock, max over ranks
        xs_h = [plan.local_input(torch.from_numpy(si.gaussian(shape, seed=sd))).cpu().pin_memory() for sd in (0, 1)]
        ys_h = [torch.empty(plan.y_shape, dtype=torch.float64).pin_memory() for _ in range(2)]
        for k in range(2):  # warm both staging slots
            plan.forward_host_async(xs_h[k], ys_h[k], stream)
        plan.wait_host()
        e2e_steps = max(3, args.steps)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            plan.forward_host_async(xs_h[k % 2], ys_h[k % 2], stream)
        plan.wait_host()
        t = torch.tensor([(time.perf_counter() - t0) * 1e3 / e2e_steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
        e2e = {"value": total_points / (ms_e2e * 1e-3), "unit": "coefficients/s",
               "h2d_bytes_per_step": int(8 * total_points), "d2h_bytes_per_step": int(8 * total_points),
               "ms_per_step": ms_e2e, "api": "jt_forward_host_async x steps + jt_host_wait on the distributed plan per rank (pinned "
                                             "slabs; H2D + passes + slab exchange + D2H), host wall clock, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, desc, threads = cpu_oracle_rate(cfg)
        cpu = {"value": v, "unit": "coefficients/s", "cores": threads, "kind": "oracle", "sample": desc}
        one = cpu_oracle_rate_one_core(cfg)
        if one is not None:
            cpu["one_core"] = {"value": one[0], "unit": "coefficients/s", "cores": 1, "sample": one[1]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "coefficients/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1) fp64, numpy PCG64 seed 0",
                "config": config_block(args, cfg, ranks, k0s), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
                "ms_per_step_stats": step_stats, "fac_s": round(fac_s, 3)}
        if slab_phases is not None:
            line["slab_phases"] = slab_phases
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
