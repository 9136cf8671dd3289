"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage or closed form it follows.  A plausible mistake in the
oracle (a dropped term, a wrong sign or index, a transposed end row, a wrong
tie-break) fails at least one of them:
  * transposed clamped end row (P:1033-1035 vs P:1018)  -> exact/dense solve, cubic reproduction
  * wrong sign / index in d_j                            -> Table nat1, exact solve, linear data
  * natural ends not exactly 0                           -> natural-ends invariant
  * wrong A/B/C/D in eval                                -> segment examples, exact eval, cubic reproduction
  * tie-break / off-by-one in locate                      -> brute-force scan with knot ties
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import refmath
from paper_2001_09253_b200 import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_tsv(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([float(v) for v in line.split()])
    return np.array(rows)


def _random_curve(rng, n, spread=1.0):
    gaps = rng.exponential(spread, n - 1) + 1e-3
    x = np.concatenate([[rng.normal()], rng.normal() + np.cumsum(gaps)])
    x = np.sort(x)
    y = rng.normal(size=n)
    return x, y


# ------------------------------------------------------------------ build pins

def test_table_nat1_hand_curve():
    """Table tbl:test_compare_nat1: natural y'' of the hand curve, 6 decimals."""
    t = _read_tsv("nat1_hand_curve.tsv")
    np.testing.assert_array_equal(t[:, 0], np.array(workloads.HAND_KNOTS, dtype=float))
    np.testing.assert_array_equal(t[:, 1], np.array(workloads.HAND_VALUES, dtype=float))
    y2, nbad = oracle.build_y2(workloads.HAND_KNOTS, workloads.HAND_VALUES, oracle.BC_NATURAL)
    assert nbad == 0
    assert np.max(np.abs(y2 - t[:, 2])) <= 5e-7


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [3, 4, 5, 8, 12])
def test_exact_rational_solve(bc, n):
    """Brute force on tiny inputs: exact rational elimination of the row definitions."""
    rng = np.random.default_rng(100 * n + bc)
    for _ in range(3):
        x, y = _random_curve(rng, n)
        yp1, ypn = rng.normal(size=2)
        y2, _ = oracle.build_y2(x, y, bc, [yp1], [ypn])
        ex = refmath.exact_solve(x, y, bc, yp1, ypn)
        scale = max(abs(float(v)) for v in ex)
        err = max(abs(Fraction(float(a)) - b) for a, b in zip(y2, ex))
        assert float(err) <= 1e-14 * scale


def test_hand_curve_exact_all_bcs():
    """The three quality-check cases of P:1145-1160: natural, y'=0 both ends, (-1, 1)."""
    for bc, s, e in [(0, 0.0, 0.0), (3, 0.0, 0.0), (3, -1.0, 1.0)]:
        y2, _ = oracle.build_y2(workloads.HAND_KNOTS, workloads.HAND_VALUES, bc, [s], [e])
        ex = refmath.exact_solve(workloads.HAND_KNOTS, workloads.HAND_VALUES, bc, s, e)
        # Tables nat/flat/twist report per-knot deltas vs 30 digits of at most 6.8e-13
        err = max(abs(float(Fraction(float(a)) - b)) for a, b in zip(y2, ex))
        assert err <= 1e-12


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_dense_gaussian_elimination(bc):
    """Textbook dense solve (partial pivoting) of the same rows, n <= 64."""
    rng = np.random.default_rng(7 + bc)
    for n in [3, 6, 17, 33, 64]:
        x, y = _random_curve(rng, n)
        yp1, ypn = rng.normal(size=2)
        y2, _ = oracle.build_y2(x, y, bc, [yp1], [ypn])
        ref = refmath.dense_solve_numpy(x, y, bc, yp1, ypn)
        assert np.max(np.abs(y2 - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_natural_ends_exactly_zero():
    rng = np.random.default_rng(3)
    x, y = _random_curve(rng, 50)
    for bc in [0, 1, 2]:
        y2, _ = oracle.build_y2(x, y, bc, [0.7], [-0.3])
        if not bc & 1:
            assert y2[0] == 0.0
        if not bc & 2:
            assert y2[-1] == 0.0


def test_linear_data_zero_curvature():
    """Linear data: y2 == 0 for natural ends and for clamped ends with the exact slope (V3)."""
    x = np.array([0.0, 0.5, 1.25, 2.0, 3.0, 3.5, 4.0])
    y = 2.0 * x - 1.0
    for bc in [0, 1, 2, 3]:
        y2, _ = oracle.build_y2(x, y, bc, [2.0], [2.0])
        assert np.all(y2 == 0.0)


def test_simple_ends_are_clamped_zero_not_zero_curvature():
    """Reading c5: the collapse ends equal clamped y'=0; on y=2x they are NOT zero (V3)."""
    x = np.array([0.0, 1.0, 2.0, 3.0])
    y2, _ = oracle.build_y2(x, 2 * x, 3, [0.0], [0.0])
    np.testing.assert_allclose(y2, [7.2, -2.4, 2.4, -7.2], rtol=1e-14)


@pytest.mark.parametrize("deg", [2, 3])
def test_cubic_reproduction(deg):
    """A cubic (or quadratic) with exact clamped slopes is reproduced: y2 = f'' at the knots
    and the spline equals f everywhere (V4).  Catches a transposed clamped end row."""
    rng = np.random.default_rng(11 + deg)
    c = rng.normal(size=4)
    if deg == 2:
        c[3] = 0.0
    f = lambda t: c[0] + c[1] * t + c[2] * t ** 2 + c[3] * t ** 3
    fp = lambda t: c[1] + 2 * c[2] * t + 3 * c[3] * t ** 2
    fpp = lambda t: 2 * c[2] + 6 * c[3] * t
    x = np.sort(rng.uniform(-2, 2, 40))
    y = f(x)
    y2, _ = oracle.build_y2(x, y, 3, [fp(x[0])], [fp(x[-1])])
    assert np.max(np.abs(y2 - fpp(x))) <= 1e-10 * np.max(np.abs(fpp(x)))
    q = rng.uniform(x[0], x[-1], 500)
    out, idx, nbad = oracle.evaluate(x, y, y2, q)
    assert nbad == 0
    assert np.max(np.abs(out - f(q))) <= 1e-10 * np.max(np.abs(f(x)))


def test_c1_continuity_and_clamped_slopes():
    """Analytic slope from Eq. nr_formula: continuous at interior knots; equals yp1/ypn
    at the clamped ends.  Residual bound 16 eps x sum of |terms|."""
    rng = np.random.default_rng(5)
    eps = np.finfo(np.float64).eps
    for bc in [0, 3]:
        x, y = _random_curve(rng, 30)
        yp1, ypn = 0.8, -1.7
        y2, _ = oracle.build_y2(x, y, bc, [yp1], [ypn])
        scale = np.max(np.abs(y2)) * np.max(np.diff(x)) + np.max(np.abs(np.diff(y) / np.diff(x)))
        for j in range(1, 29):
            left = refmath.slope(x[j], x, y, y2, j - 1)
            right = refmath.slope(x[j], x, y, y2, j)
            assert abs(left - right) <= 64 * eps * scale
        if bc == 3:
            assert abs(refmath.slope(x[0], x, y, y2, 0) - yp1) <= 64 * eps * scale
            assert abs(refmath.slope(x[-1], x, y, y2, 28) - ypn) <= 64 * eps * scale


def test_power_of_two_scaling_is_bitwise():
    """x -> 8x, slopes / 8 gives y2 / 64 bitwise: every operation commutes with 2^k scaling."""
    rng = np.random.default_rng(9)
    x, y = _random_curve(rng, 40)
    a, _ = oracle.build_y2(x, y, 3, [0.3], [-0.2])
    b, _ = oracle.build_y2(8 * x, y, 3, [0.3 / 8], [-0.2 / 8])
    np.testing.assert_array_equal(a / 64, b)


def test_reversal_symmetry():
    """x -> -x reversed, y reversed, ends swapped with slopes negated: y2 reversed."""
    rng = np.random.default_rng(10)
    x, y = _random_curve(rng, 40)
    a, _ = oracle.build_y2(x, y, 3, [0.3], [-0.2])
    b, _ = oracle.build_y2(-x[::-1], y[::-1], 3, [0.2], [-0.3])
    np.testing.assert_allclose(a, b[::-1], rtol=1e-13, atol=1e-13 * np.max(np.abs(a)))


def test_bad_knots_and_n_lt_3():
    y2, nbad = oracle.build_y2([[0, 1, 1, 2], [0, 1, 2, 3]], [[0, 1, 2, 3], [0, 1, 0, 1]], 0)
    assert nbad == 1
    assert np.all(np.isnan(y2[0])) and np.all(np.isfinite(y2[1]))
    y2, nbad = oracle.build_y2([0, 1, 2, np.nan], [0, 1, 2, 3], 0)
    assert nbad == 1
    y2, nbad = oracle.build_y2([0, 1, 2], [0, 1, 2], 1, [np.inf], [0.0])
    assert nbad == 1
    with pytest.raises(ValueError):
        oracle.build_y2([0, 1], [0, 1], 0)


# ------------------------------------------------------------------- locate pins

def test_locate_brute_force_with_ties():
    rng = np.random.default_rng(12)
    for n in [3, 4, 7, 16, 65]:
        x, _ = _random_curve(rng, n)
        qs = list(rng.uniform(x[0] - 0.5, x[-1] + 0.5, 300)) + list(x) + [x[0], x[-1], np.nan,
                                                                          np.nextafter(x[0], -np.inf),
                                                                          np.nextafter(x[-1], np.inf)]
        for q in qs:
            assert oracle.locate(x, q) == refmath.brute_locate(x, q), (n, q)
    x = np.arange(5.0)
    assert oracle.locate(x, 0.0) == 0
    assert oracle.locate(x, 2.0) == 2      # interior tie: the knot is the LEFT end (reading c1)
    assert oracle.locate(x, 4.0) == 3      # q = x_{n-1} -> n-2
    assert oracle.locate(x, 4.5) == -1


# --------------------------------------------------------------------- eval pins

def test_segment_examples():
    t = _read_tsv("segment_examples.tsv")
    for q, a, b, u, v, up, vp, expect in t:
        got = oracle.interp(q, [a, b], [u, v], [up, vp], 0)
        assert got == pytest.approx(expect, rel=0, abs=2 * np.finfo(float).eps * max(1.0, abs(expect)))


def test_knot_interpolation_bitwise():
    rng = np.random.default_rng(13)
    x, y = _random_curve(rng, 33)
    y2, _ = oracle.build_y2(x, y, 0)
    out, idx, _ = oracle.evaluate(x, y, y2, x)
    np.testing.assert_array_equal(out, y)   # A=1 (or B=1 at x_{n-1}) and C=D=0 exactly


def test_eval_exact_rational():
    rng = np.random.default_rng(14)
    x, y = _random_curve(rng, 9)
    y2, _ = oracle.build_y2(x, y, 3, [0.5], [-0.5])
    q = rng.uniform(x[0], x[-1], 50)
    out, idx, _ = oracle.evaluate(x, y, y2, q)
    for k in range(50):
        ex = refmath.exact_eval(q[k], x, y, [Fraction(float(v)) for v in y2], idx[k])
        assert abs(float(Fraction(float(out[k])) - ex)) <= 8 * np.finfo(float).eps * (
            np.max(np.abs(y)) + np.max(np.abs(y2)) * np.max(np.diff(x)) ** 2)


def test_e7_sweep_mse_order_of_magnitude():
    """E7: clamped (-1, 1) hand curve, 2048-point sweep vs a 'true' (here exact
    rational) reference; the paper prints MSE 1.57e-30.  Order-of-magnitude pin."""
    x, y = workloads.HAND_KNOTS, workloads.HAND_VALUES
    y2, _ = oracle.build_y2(x, y, 3, [-1.0], [1.0])
    ex_y2 = refmath.exact_solve(x, y, 3, -1.0, 1.0)
    q = np.linspace(min(x), max(x), 2048)
    out, idx, nbad = oracle.evaluate(x, y, y2, q)
    assert nbad == 0
    errs = [float(Fraction(float(out[k])) - refmath.exact_eval(q[k], x, y, ex_y2, idx[k]))
            for k in range(0, 2048, 4)]
    mse = float(np.mean(np.square(errs)))
    assert mse < 1e-26


def test_out_of_range_and_nan_queries():
    x = np.array([0.0, 1.0, 2.0, 3.0])
    y2, _ = oracle.build_y2(x, x * x, 0)
    out, idx, nbad = oracle.evaluate(x, x * x, y2, [-1.0, 3.5, np.nan, 1.5])
    assert list(idx) == [-1, -1, -1, 1]
    assert np.isnan(out[:3]).all() and np.isfinite(out[3])
    assert nbad == 3


# ------------------------------------------------------------- batch-driver pins
# oracle_build_batch / oracle_eval_batch (oracle.c) pick each curve's slopes and offsets; these
# pins check every curve of a batch against its OWN exact solution, so a driver that reads curve
# 0's slope (yp1[c] -> yp1[0]) or drops a per-curve offset (x + c*n -> x) fails.

def _distinct_batch(rng, B, n):
    xs, ys = [], []
    for c in range(B):
        x, y = _random_curve(rng, n, spread=0.5 + c)   # every curve its own range and spacing
        xs.append(x + 3.0 * c)
        ys.append(y * (1 + c))
    return np.array(xs), np.array(ys)


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
@pytest.mark.parametrize("nthreads", [1, 3])
def test_batch_build_each_curve_exact(bc, nthreads):
    """Every row of a batched build equals the exact rational solve of THAT curve with THAT
    curve's clamped slopes (rows Eq. init_val)."""
    rng = np.random.default_rng(40 + bc)
    B, n = 5, 7
    x, y = _distinct_batch(rng, B, n)
    yp1 = rng.normal(size=B) * 3 + np.arange(B)       # distinct per curve
    ypn = rng.normal(size=B) * 3 - np.arange(B)
    y2, nbad = oracle.build_y2(x, y, bc, yp1, ypn, nthreads=nthreads)
    assert nbad == 0
    for c in range(B):
        ex = refmath.exact_solve(x[c], y[c], bc, yp1[c], ypn[c])
        scale = max(abs(float(v)) for v in ex)
        err = max(abs(Fraction(float(a)) - b) for a, b in zip(y2[c], ex))
        assert float(err) <= 1e-14 * scale, (bc, c)


def test_batch_build_bad_curve_isolated():
    """A bad curve in the middle of a batch NaN-fills only its own row."""
    rng = np.random.default_rng(44)
    x, y = _distinct_batch(rng, 4, 6)
    x[2, 3] = x[2, 2]                                   # curve 2: repeated knot
    y2, nbad = oracle.build_y2(x, y, 3, np.arange(4.0), -np.arange(4.0), nthreads=2)
    assert nbad == 1
    assert np.isnan(y2[2]).all()
    for c in (0, 1, 3):
        ex = refmath.exact_solve(x[c], y[c], 3, float(c), -float(c))
        assert np.max(np.abs(y2[c] - np.array([float(v) for v in ex]))) <= 1e-13 * max(abs(float(v)) for v in ex)


@pytest.mark.parametrize("nthreads", [1, 4])
def test_batch_eval_each_curve_exact(nthreads):
    """Every (curve, query) of a batched eval: idx = the brute-force scan over THAT curve's knots
    (reading c1) and out = Eq. nr_formula in exact rationals on THAT curve.  The
    curves occupy disjoint x ranges, so a query routed to another curve is out of its range."""
    rng = np.random.default_rng(45)
    B, n, m = 4, 6, 9
    x, y = _distinct_batch(rng, B, n)
    y2 = rng.normal(size=(B, n)) * np.arange(1, B + 1)[:, None]  # any y2: eval is defined for it
    q = np.array([rng.uniform(x[c, 0], x[c, -1], m) for c in range(B)])
    q[1, 0] = x[1, 2]                                   # a knot tie
    q[2, 1] = x[2, -1]                                  # the last knot
    q[3, 2] = x[0, 1]                                   # inside curve 0's range, outside curve 3's
    out, idx, nbad = oracle.evaluate(x, y, y2, q, nthreads=nthreads)
    assert nbad == 1
    for c in range(B):
        for k in range(m):
            j = refmath.brute_locate(x[c], q[c, k])
            assert idx[c, k] == j, (c, k)
            if j < 0:
                assert np.isnan(out[c, k])
                continue
            ex = refmath.exact_eval(q[c, k], x[c], y[c], [Fraction(float(v)) for v in y2[c]], j)
            tol = 8 * np.finfo(float).eps * (np.max(np.abs(y[c])) + np.max(np.abs(y2[c])) * np.max(np.diff(x[c])) ** 2)
            assert abs(float(Fraction(float(out[c, k])) - ex)) <= tol, (c, k)


def test_batch_threads_identical():
    wl = workloads.generate(2, batch=64, m=32)
    a, _ = oracle.build_y2(wl.x, wl.y, wl.bc, wl.yp1, wl.ypn, nthreads=1)
    b, _ = oracle.build_y2(wl.x, wl.y, wl.bc, wl.yp1, wl.ypn, nthreads=4)
    np.testing.assert_array_equal(a, b)
    o1, i1, _ = oracle.evaluate(wl.x, wl.y, a, wl.q, nthreads=1)
    o2, i2, _ = oracle.evaluate(wl.x, wl.y, a, wl.q, nthreads=3)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(i1, i2)
