"""CPU oracle for the cubic-spline hot path of arXiv 2001.09253 (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2001_09253_b200`` never imports it, and the two share no code.

The arithmetic lives in ``oracle.c`` (plain C, fp64, ``-O2 -ffp-contract=off``);
this module only compiles it (``build()``) and marshals numpy arrays into it.

Parity status of each function (pins are in ``tests/test_oracle_pins.py``):
  build   -- pinned: Table nat1, exact rational solve, dense solve,
             closed forms (linear -> 0, cubic reproduction), natural ends == 0.
  locate  -- pinned: brute-force linear scan, knot ties, out-of-range.
  interp  -- pinned: hand-computed segments, knot interpolation,
             exact rational evaluation, cubic reproduction, E7 sweep MSE.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

BC_NATURAL = 0
BC_CLAMP_START = 1
BC_CLAMP_END = 2
BC_CLAMPED = 3

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
               "-shared", "-pthread", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.oracle_build.argtypes = [vp, vp, i64, i32, d, d, vp]
        lib.oracle_build.restype = i32
        lib.oracle_locate.argtypes = [vp, i64, d]
        lib.oracle_locate.restype = i64
        lib.oracle_interp.argtypes = [d, vp, vp, vp, i64]
        lib.oracle_interp.restype = d
        lib.oracle_build_batch.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp, i32]
        lib.oracle_build_batch.restype = i32
        lib.oracle_eval_batch.argtypes = [vp, vp, vp, i64, i64, vp, i64, vp, vp, i32]
        lib.oracle_eval_batch.restype = i32
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def build_y2(x, y, bc: int = BC_NATURAL, yp1=None, ypn=None, nthreads: int = 1):
    """Second derivatives for a batch of curves, ``x``/``y`` of shape (B, n) or (n,).

    ``yp1``/``ypn`` are per-curve clamped slopes (ignored for natural ends).
    Returns (y2 float64 with the input's shape, number of bad curves).
    """
    lib = _load()
    x = _f64(x)
    y = _f64(y)
    shape = x.shape
    if x.ndim == 1:
        x = x[None]
        y = y[None]
    B, n = x.shape
    if n < 3:
        raise ValueError("n must be >= 3 (P:1047)")
    s = _f64(np.broadcast_to(0.0 if yp1 is None else np.asarray(yp1, dtype=np.float64), (B,)))
    e = _f64(np.broadcast_to(0.0 if ypn is None else np.asarray(ypn, dtype=np.float64), (B,)))
    y2 = np.empty((B, n), dtype=np.float64)
    nbad = lib.oracle_build_batch(_ptr(x), _ptr(y), n, B, bc, _ptr(s), _ptr(e), _ptr(y2), nthreads)
    return y2.reshape(shape), nbad


def locate(x, q) -> int:
    lib = _load()
    x = _f64(x)
    return int(lib.oracle_locate(_ptr(x), x.shape[-1], float(q)))


def interp(q, x, y, y2, j) -> float:
    lib = _load()
    x, y, y2 = _f64(x), _f64(y), _f64(y2)
    return float(lib.oracle_interp(float(q), _ptr(x), _ptr(y), _ptr(y2), int(j)))


def evaluate(x, y, y2, q, nthreads: int = 1):
    """Locate + Eq. nr_formula for queries ``q`` of shape (B, m) against curves (B, n).

    Returns (out float64 (B, m), idx int64 (B, m), number of out-of-range queries).
    """
    lib = _load()
    x, y, y2, q = _f64(x), _f64(y), _f64(y2), _f64(q)
    qshape = q.shape
    if x.ndim == 1:
        x, y, y2 = x[None], y[None], y2[None]
        q = q.reshape(1, -1)
    B, n = x.shape
    m = q.shape[-1]
    out = np.empty((B, m), dtype=np.float64)
    idx = np.empty((B, m), dtype=np.int64)
    nbad = lib.oracle_eval_batch(_ptr(x), _ptr(y), _ptr(y2), n, B, _ptr(q), m, _ptr(out), _ptr(idx), nthreads)
    return out.reshape(qshape), idx.reshape(qshape), nbad
