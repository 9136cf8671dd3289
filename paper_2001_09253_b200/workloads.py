"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module only draws random numbers; it holds none of the method's arithmetic
(no tridiagonal rows, no locate, no interpolation), so it may serve both the CUDA
path and the CPU oracle (the one thing they share).  The recipes follow
SURVEY.md §8(d) and the readings c10/c11 listed in DESIGN.md; they stand in for
the paper's own inputs (the hand curve P:1142-1143, the randomised curves of
P:1724-1727 and the evenly spaced sweeps of P:1736-1738).  No public dataset is
involved.

Every array is numpy, C-contiguous, curve-major: x, y are (B, n), q is (B, m),
yp1/ypn are (B,) (or None for natural ends).  Generation uses numpy PCG64
(``default_rng``) in a fixed draw order; config k uses seed k-1, and shard r of
a multi-GPU weak-scaling job uses ``default_rng([seed, r])``.
"""
from __future__ import annotations

import dataclasses
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BC_NATURAL, BC_CLAMP_START, BC_CLAMP_END, BC_CLAMPED = 0, 1, 2, 3
FLAG_Q_SORTED, FLAG_X_UNIFORM = 1, 2


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    cid: int
    name: str
    batch: int
    n: int
    m: int
    dtype: str  # "f32" | "f64"
    bc: int
    flags: int
    seed: int


CONFIGS = {
    1: ConfigSpec(1, "cfg1: 1 curve x n=16, fp64, natural, 1000 unsorted queries", 1, 16, 1000, "f64",
                  BC_NATURAL, 0, 0),
    2: ConfigSpec(2, "cfg2: 65536 curves x n=64, fp32, clamped, 256 unsorted queries/curve", 65536, 64, 256,
                  "f32", BC_CLAMPED, 0, 1),
    3: ConfigSpec(3, "cfg3: 1048576 curves x n=8 (uniform grid), fp32, natural, 32 queries/curve", 1 << 20, 8,
                  32, "f32", BC_NATURAL, FLAG_X_UNIFORM, 2),
    4: ConfigSpec(4, "cfg4: 4096 curves x n=4096, fp64, clamped (analytic), 16 sorted queries/knot", 4096, 4096,
                  65536, "f64", BC_CLAMPED, FLAG_Q_SORTED, 3),
    5: ConfigSpec(5, "cfg5: 1 curve x n=2^26 (jittered grid), fp64, natural, 2^28 unsorted queries", 1, 1 << 26,
                  1 << 28, "f64", BC_NATURAL, 0, 4),
}


@dataclasses.dataclass
class Workload:
    spec: ConfigSpec
    x: np.ndarray
    y: np.ndarray
    q: np.ndarray
    yp1: np.ndarray | None
    ypn: np.ndarray | None
    bc: int
    flags: int

    @property
    def batch(self) -> int:
        return self.y.shape[0]

    @property
    def n(self) -> int:
        return self.y.shape[1]

    @property
    def m(self) -> int:
        return self.q.shape[1]

    @property
    def np_dtype(self):
        return np.float32 if self.spec.dtype == "f32" else np.float64


def slice_batch(wl: "Workload", b0: int, b1: int) -> "Workload":
    """Curves [b0, b1) of a workload (strong scaling: rank r owns [r B / G, (r+1) B / G) of the
    config's batch), as contiguous copies."""
    sl = lambda a: None if a is None else np.ascontiguousarray(a[b0:b1])
    x = wl.x if wl.x.ndim == 1 else sl(wl.x)  # shared knots stay one row
    return Workload(wl.spec, x, sl(wl.y), sl(wl.q), sl(wl.yp1), sl(wl.ypn), wl.bc, wl.flags)


def _rng(seed: int, shard: int) -> np.random.Generator:
    return np.random.default_rng(seed if shard == 0 else [seed, shard])


def _fix_f32_increasing(x32: np.ndarray) -> np.ndarray:
    """Reading c11: after rounding to fp32, force strict increase by nextafter."""
    x32 = x32.copy()
    for j in range(1, x32.shape[1]):
        bad = x32[:, j] <= x32[:, j - 1]
        if bad.any():
            x32[bad, j] = np.nextafter(x32[bad, j - 1], np.float32(np.inf))
    return x32


def _queries(rng, x: np.ndarray, m: int, dt, lo=None, hi=None) -> np.ndarray:
    """m Uniform queries per curve in [x_0, x_{n-1}], drawn in fp64, rounded to dt, clamped."""
    B = x.shape[0]
    a = x[:, :1].astype(np.float64) if lo is None else np.full((B, 1), lo)
    b = x[:, -1:].astype(np.float64) if hi is None else np.full((B, 1), hi)
    u = rng.random((B, m))
    q = (a + u * (b - a)).astype(dt)
    return np.clip(q, a.astype(dt), b.astype(dt))


def _sort_rows(a: np.ndarray) -> np.ndarray:
    if a.shape[0] < 64:
        a.sort(axis=1)
        return a
    chunks = np.array_split(np.arange(a.shape[0]), 16)
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(lambda ix: a[ix[0]:ix[-1] + 1].sort(axis=1), chunks))
    return a


def generate(cid: int, batch: int | None = None, n: int | None = None, m: int | None = None,
             seed: int | None = None, shard: int = 0) -> Workload:
    """Draw config ``cid`` (1..5), optionally with overridden sizes (parity cases)."""
    spec = CONFIGS[cid]
    B = spec.batch if batch is None else batch
    n = spec.n if n is None else n
    m = spec.m if m is None else m
    rng = _rng(spec.seed if seed is None else seed, shard)
    yp1 = ypn = None

    if cid == 1:
        # gaps U(0.5, 1.5) normalised to [0, 1]; y = sin(2 pi x) + N(0, 0.01) (variance; c10)
        g = rng.uniform(0.5, 1.5, (B, n - 1))
        x = np.concatenate([np.zeros((B, 1)), np.cumsum(g, axis=1)], axis=1) / g.sum(axis=1, keepdims=True)
        x[:, 0] = 0.0
        x[:, -1] = 1.0
        y = np.sin(2 * np.pi * x) + rng.normal(0.0, 0.1, (B, n))
        q = _queries(rng, x, m, np.float64)
    elif cid == 2:
        # x = cumsum Exp(1) gaps from 0; y = random walk of N(0,1) steps; clamped N(0,1) slopes
        gaps = rng.exponential(1.0, (B, n - 1))
        steps = rng.standard_normal((B, n))
        yp1 = rng.standard_normal(B).astype(np.float32)
        ypn = rng.standard_normal(B).astype(np.float32)
        x = np.concatenate([np.zeros((B, 1)), np.cumsum(gaps, axis=1)], axis=1)
        x = _fix_f32_increasing(x.astype(np.float32))
        y = np.cumsum(steps, axis=1).astype(np.float32)
        q = _queries(rng, x, m, np.float32)
    elif cid == 3:
        # evenly spaced grid x_j = j/(n-1), stored per curve (c10); y ~ U(-1, 1); q ~ U[0, 1)
        grid = (np.arange(n, dtype=np.float64) / (n - 1)).astype(np.float32)
        x = np.ascontiguousarray(np.broadcast_to(grid, (B, n)))
        y = rng.uniform(-1.0, 1.0, (B, n)).astype(np.float32)
        q = _queries(rng, x, m, np.float32)
    elif cid == 4:
        # x = cumsum Exp(1); y = sum of 3 sinusoids (f ~ U(1,50) cycles over the range,
        # phase U(0, 2pi), amplitude U(0.5, 2)) + N(0, 1e-3); analytic clamped slopes; sorted q
        gaps = rng.exponential(1.0, (B, n - 1))
        f = rng.uniform(1.0, 50.0, (B, 3))
        ph = rng.uniform(0.0, 2 * np.pi, (B, 3))
        A = rng.uniform(0.5, 2.0, (B, 3))
        noise = rng.normal(0.0, np.sqrt(1e-3), (B, n))
        x = np.concatenate([np.zeros((B, 1)), np.cumsum(gaps, axis=1)], axis=1)
        L = x[:, -1:] - x[:, :1]
        w = 2 * np.pi * f / L  # (B, 3) angular frequency per unit x
        y = np.zeros((B, n))
        for k in range(3):
            y += A[:, k:k + 1] * np.sin(w[:, k:k + 1] * (x - x[:, :1]) + ph[:, k:k + 1])
        y += noise
        yp1 = (A * w * np.cos(ph)).sum(axis=1)
        ypn = (A * w * np.cos(w * L + ph)).sum(axis=1)
        q = _sort_rows(_queries(rng, x, m, np.float64))
    elif cid == 5:
        # x_j = (j + U(-0.1, 0.1))/(n-1), ends pinned to 0 and 1; Brownian y, N(0, 1/n) steps
        jit = rng.uniform(-0.1, 0.1, (B, n))
        steps = rng.normal(0.0, np.sqrt(1.0 / n), (B, n))
        x = (np.arange(n, dtype=np.float64)[None, :] + jit) / (n - 1)
        x[:, 0] = 0.0
        x[:, -1] = 1.0
        steps[:, 0] = 0.0
        y = np.cumsum(steps, axis=1)
        q = _queries(rng, x, m, np.float64, lo=0.0, hi=1.0)
    else:
        raise ValueError(f"unknown config {cid}")

    dt = np.float32 if spec.dtype == "f32" else np.float64
    x = np.ascontiguousarray(x, dtype=dt)
    y = np.ascontiguousarray(y, dtype=dt)
    if yp1 is not None:
        yp1 = np.ascontiguousarray(yp1, dtype=dt)
        ypn = np.ascontiguousarray(ypn, dtype=dt)
    return Workload(spec, x, y, np.ascontiguousarray(q, dtype=dt), yp1, ypn, spec.bc, spec.flags)


# The hand-generated curve of the paper's quality checks.
HAND_KNOTS = [0, 0.5, 1, 1.01, 1.25, 1.5, 1.58, 1.79, 2.12, 2.30, 2.402, 2.451, 2.5]
HAND_VALUES = [1, 1.2, 2, 0.25, 0.25, 0.25, 0.63, 0.96, 1.17, 1.23, 1.245, 1.249, 1.25]


def sweep_curves(n: int, batch: int, seed: int = 0, dtype=np.float64):
    """The paper's randomised timing curves: y_i = eps, x_i = x_{i-1} + eps with
    eps ~ U(0, 1) (eps == 0 -> 1e-4), and n uniformly spaced query points from x_0 to x_{n-1}
    per curve (sorted).  Returns (x, y, q) as (batch, n) arrays; natural ends are implied."""
    rng = np.random.default_rng([seed, n])
    eps = rng.random((batch, n))
    eps[eps == 0] = 1e-4
    x = np.cumsum(eps, axis=1)
    y = rng.random((batch, n))
    y[y == 0] = 1e-4
    t = np.linspace(0.0, 1.0, n)
    q = x[:, :1] + t[None, :] * (x[:, -1:] - x[:, :1])
    q = np.minimum(np.maximum(q, x[:, :1]), x[:, -1:])
    return x.astype(dtype), y.astype(dtype), q.astype(dtype)


def sweep_schedule(points: int, n_min: int = 4, n_max: int = 1 << 20):
    """The paper's list of control-point counts: (r (sqrt(n_max) - sqrt(n_min))
    + sqrt(n_min))^2 at `points` evenly spaced r in [0, 1] (biased towards short curves)."""
    r = np.linspace(0.0, 1.0, points)
    return [int(round((v * (np.sqrt(n_max) - np.sqrt(n_min)) + np.sqrt(n_min)) ** 2)) for v in r]
