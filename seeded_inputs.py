"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds none of the method's arithmetic: it only draws random arrays.
Both `oracle/` (via tests and bench's cpu_baseline leg) and the product path
(via tests and bench.py) take their inputs from here, so the two sides see the
same bytes.

Recipe (SURVEY.md §8(c) reading 15): the paper measures on
"random vectors" (§4.1 eq:stability) and BASELINE.json's configs
say "coefficients iid N(0,1) fp64 from seed".  We use numpy's PCG64
`default_rng(seed).standard_normal(shape)` in float64, C-order.
"""
from __future__ import annotations

import numpy as np

# BASELINE.json "configs" (index 0..4) as concrete shapes and per-axis (a, b).
CONFIGS = {
    "cfg1_1d_1024": dict(n=(1024,), a=(0.25,), b=(-0.3,), eps=1e-12, inverse=True),
    "cfg2_2d_256": dict(n=(256, 256), a=(0.1, -0.25), b=(-0.4, 0.35), eps=1e-12, inverse=True),
    "cfg3_2d_4096": dict(n=(4096, 4096), a=(0.45, 0.0), b=(-0.45, 0.0), eps=1e-12, inverse=True),
    "cfg4_3d_256": dict(n=(256, 256, 256), a=(0.2, -0.4, 0.35), b=(-0.2, 0.3, 0.1), eps=1e-12,
                        inverse=True),
    "cfg5_3d_512": dict(n=(512, 512, 512), a=(0.25, 0.25, 0.25), b=(-0.25, -0.25, -0.25),
                        eps=1e-12, inverse=False),
    # SURVEY.md §8(f) NEXT rows (not BASELINE configs): the paper's 3D nonuniform experiment setting
    # (a = b = 0.4 on every axis, random points) and a second-kind (Q~) uniform transform
    "nu_3d_256": dict(n=(256, 256, 256), a=(0.4, 0.4, 0.4), b=(0.4, 0.4, 0.4), eps=1e-12, inverse=False,
                      points="random"),
    "q_3d_256": dict(n=(256, 256, 256), a=(0.2, -0.4, 0.35), b=(-0.2, 0.3, 0.1), eps=1e-12, inverse=False,
                     kind=1),
}


def points(n: int, seed: int) -> np.ndarray:
    """n sorted random angles, uniform in (0, pi) (nonuniform-transform locations; no method arithmetic)."""
    rng = np.random.default_rng(seed)
    return np.pi * np.sort(rng.uniform(0, 1, int(n))) * (1 - 2e-6) + 1e-6


def config_points(cfg):
    """Per-axis point arrays of a config (None = uniform Gauss-Jacobi nodes), seeds 100 + axis."""
    if cfg.get("points") != "random":
        return None
    return [points(n, 100 + i) for i, n in enumerate(cfg["n"])]


def gaussian(shape, seed: int = 0) -> np.ndarray:
    """iid N(0,1) float64 array of `shape`, C-order, from numpy PCG64 `seed`."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.standard_normal(tuple(int(s) for s in shape)), dtype=np.float64)


def sample_indices(shape, count: int, seed: int = 12345) -> np.ndarray:
    """`count` distinct-ish random multi-indices into an array of `shape` (for sampled parity).

    Always includes the first and last element (corner cases) so ragged ends are covered.
    """
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, s, size=count) for s in shape], axis=1)
    idx[0] = 0
    idx[-1] = np.array(shape) - 1
    return idx
