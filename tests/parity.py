"""Parity helpers: GPU path vs CPU oracle on the same seeded inputs (test infrastructure).

Tolerances (north star; normalisation = DESIGN.md reading c2):
  y2  : per curve, max|y2 - y2_ref| / max|y2_ref|                      <= 1e-12 (f64) / 2e-5 (f32)
  out : per curve, max|out - out_ref| / max(max|y|, max|out_ref|)       <= 1e-12 (f64) / 2e-5 (f32)
  idx : bit-exact (the largest j in [0, n-2] with x_j <= q; -1 outside / NaN).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle

TOL = {np.float32: 2e-5, np.float64: 1e-12}


def tol_for(dt) -> float:
    return TOL[np.dtype(dt).type]


def y2_rel_err(y2, ref, x=None, y=None) -> np.ndarray:
    """Per-curve relative y2 error (reading c2; scale 0 falls back to 6 max|dd| / min h)."""
    y2 = np.asarray(y2, dtype=np.float64).reshape(ref.shape)
    err = np.max(np.abs(y2 - ref), axis=-1)
    scale = np.max(np.abs(ref), axis=-1)
    if x is not None and np.any(scale == 0):
        h = np.diff(np.asarray(x, np.float64), axis=-1)
        dd = np.diff(np.asarray(y, np.float64), axis=-1) / h
        fb = 6 * np.max(np.abs(dd), axis=-1) / np.min(h, axis=-1)
        scale = np.where(scale == 0, fb, scale)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(err == 0, 0.0, err / scale)
    return r


def out_rel_err(out, ref, y) -> np.ndarray:
    out = np.asarray(out, dtype=np.float64).reshape(ref.shape)
    both_nan = np.isnan(out) & np.isnan(ref)
    d = np.where(both_nan, 0.0, np.abs(out - ref))
    d = np.where(np.isnan(d), np.inf, d)
    err = np.max(d, axis=-1)
    scale = np.maximum(np.max(np.abs(np.asarray(y, np.float64)), axis=-1),
                       np.max(np.where(np.isnan(ref), 0, np.abs(ref)), axis=-1))
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(err == 0, 0.0, err / scale)


def out_rel_err_literal(out, ref, y) -> np.ndarray:
    """BASELINE.json's literal normalisation, reported beside reading c2: per curve
    max|out - out_ref| / max|y| (max|y| alone, without the overshoot of the spline itself)."""
    out = np.asarray(out, dtype=np.float64).reshape(ref.shape)
    both_nan = np.isnan(out) & np.isnan(ref)
    d = np.where(both_nan, 0.0, np.abs(out - ref))
    d = np.where(np.isnan(d), np.inf, d)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.max(d, axis=-1) / np.max(np.abs(np.asarray(y, np.float64)), axis=-1)


def to_dev(a, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def gpu_build(api, wl, dev="cuda"):
    x, y = to_dev(wl.x, dev), to_dev(wl.y, dev)
    yp1 = to_dev(wl.yp1, dev) if wl.yp1 is not None else None
    ypn = to_dev(wl.ypn, dev) if wl.ypn is not None else None
    return x, y, api.build(x, y, wl.bc, yp1, ypn)


def oracle_build(wl, nthreads=8):
    y2, nbad = oracle.build_y2(wl.x, wl.y, wl.bc, wl.yp1, wl.ypn, nthreads=nthreads)
    return y2


def check_case(api, wl, flags=None, nthreads=8, check_e2e=True, y2_only=False):
    """Full parity of one workload: build (y2), isolated eval (GPU eval on y2_ref rounded to T,
    reading c12), and end to end (GPU build -> GPU eval)."""
    dt = wl.np_dtype
    tol = tol_for(dt)
    flags = wl.flags if flags is None else flags
    x, y, y2 = gpu_build(api, wl)
    y2_ref = oracle_build(wl, nthreads)
    e = y2_rel_err(y2.cpu().numpy(), y2_ref, wl.x, wl.y)
    assert np.all(e <= tol), f"y2 max rel err {e.max():.3e} > {tol}"
    if y2_only:
        return
    q = to_dev(wl.q)
    out_ref, idx_ref, _ = oracle.evaluate(wl.x, wl.y, y2_ref, wl.q, nthreads=nthreads)
    out, idx = api.evaluate(x, y, to_dev(y2_ref.astype(dt)), q, flags)
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    eo = out_rel_err(out.cpu().numpy(), out_ref, wl.y)
    assert np.all(eo <= tol), f"out (isolated) max rel err {eo.max():.3e} > {tol}"
    if check_e2e:
        out2, idx2 = api.evaluate(x, y, y2, q, flags)
        np.testing.assert_array_equal(idx2.cpu().numpy(), idx_ref)
        eo2 = out_rel_err(out2.cpu().numpy(), out_ref, wl.y)
        assert np.all(eo2 <= tol), f"out (end to end) max rel err {eo2.max():.3e} > {tol}"
    lit = out_rel_err_literal(out.cpu().numpy(), out_ref, wl.y)
    return dict(y2=float(e.max()), out=float(eo.max()), out_literal=float(lit.max()))
