"""Independent mathematics used to PIN the oracle (test infrastructure only).

None of this is the oracle's algorithm: the oracle is the paper's Thomas sweep
(P:1041-1125); here the same system is written as a dense matrix straight from
its row definitions and solved by other means (numpy Gaussian elimination, and
exact rational elimination with ``fractions.Fraction``), and the spline's
derivative is written out analytically from Eq. nr_formula.

Rows (0-based, h_j = x_{j+1}-x_j, dd_j = (y_{j+1}-y_j)/h_j):
  interior j=1..n-2   h_{j-1} y2_{j-1} + 2(h_{j-1}+h_j) y2_j + h_j y2_{j+1} = 6(dd_j - dd_{j-1})
                      (Eq. init_val)
  natural start/end   y2_0 = 0 / y2_{n-1} = 0
  clamped start       2 h_0 y2_0 + h_0 y2_1 = 6(dd_0 - yp1)
  clamped end         h_{n-2} y2_{n-2} + 2 h_{n-2} y2_{n-1} = 6(ypn - dd_{n-2})
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def dense_system(x, y, bc, yp1=0.0, ypn=0.0, num=float):
    n = len(x)
    x = [num(v) for v in x]
    y = [num(v) for v in y]
    h = [x[j + 1] - x[j] for j in range(n - 1)]
    dd = [(y[j + 1] - y[j]) / h[j] for j in range(n - 1)]
    M = [[num(0)] * n for _ in range(n)]
    d = [num(0)] * n
    for j in range(1, n - 1):
        M[j][j - 1] = h[j - 1]
        M[j][j] = 2 * (h[j - 1] + h[j])
        M[j][j + 1] = h[j]
        d[j] = 6 * (dd[j] - dd[j - 1])
    if bc & 1:
        M[0][0] = 2 * h[0]
        M[0][1] = h[0]
        d[0] = 6 * (dd[0] - num(yp1))
    else:
        M[0][0] = num(1)
    if bc & 2:
        M[n - 1][n - 2] = h[n - 2]
        M[n - 1][n - 1] = 2 * h[n - 2]
        d[n - 1] = 6 * (num(ypn) - dd[n - 2])
    else:
        M[n - 1][n - 1] = num(1)
    return M, d


def dense_solve_numpy(x, y, bc, yp1=0.0, ypn=0.0):
    M, d = dense_system(x, y, bc, yp1, ypn)
    return np.linalg.solve(np.array(M, dtype=np.float64), np.array(d, dtype=np.float64))


def exact_solve(x, y, bc, yp1=0.0, ypn=0.0):
    """Exact rational Gaussian elimination on the exact binary values of the inputs."""
    M, d = dense_system([Fraction(float(v)) for v in x], [Fraction(float(v)) for v in y], bc,
                        Fraction(float(yp1)), Fraction(float(ypn)), num=Fraction)
    n = len(d)
    for k in range(n):
        p = max(range(k, n), key=lambda r: abs(M[r][k]))
        M[k], M[p] = M[p], M[k]
        d[k], d[p] = d[p], d[k]
        for r in range(k + 1, n):
            if M[r][k] != 0:
                f = M[r][k] / M[k][k]
                for c in range(k, n):
                    M[r][c] -= f * M[k][c]
                d[r] -= f * d[k]
    sol = [Fraction(0)] * n
    for k in range(n - 1, -1, -1):
        s = d[k] - sum(M[k][c] * sol[c] for c in range(k + 1, n))
        sol[k] = s / M[k][k]
    return sol


def exact_eval(q, x, y, y2, j):
    """Eq. nr_formula in exact rationals."""
    q, a, b = Fraction(float(q)), Fraction(float(x[j])), Fraction(float(x[j + 1]))
    h = b - a
    A = (b - q) / h
    B = (q - a) / h
    return (A * Fraction(float(y[j])) + B * Fraction(float(y[j + 1]))
            + (A ** 3 - A) * h * h / 6 * Fraction(y2[j]) + (B ** 3 - B) * h * h / 6 * Fraction(y2[j + 1]))


def slope(q, x, y, y2, j):
    """Analytic y'(q) on segment j, differentiated from Eq. nr_formula:
    y' = dd_j - (3A^2-1) h y2_j / 6 + (3B^2-1) h y2_{j+1} / 6."""
    h = x[j + 1] - x[j]
    A = (x[j + 1] - q) / h
    B = (q - x[j]) / h
    dd = (y[j + 1] - y[j]) / h
    return dd - (3 * A * A - 1) * h * y2[j] / 6 + (3 * B * B - 1) * h * y2[j + 1] / 6


def brute_locate(x, q):
    """Linear scan: the largest j in [0, n-2] with x_j <= q, -1 if q outside [x_0, x_{n-1}]."""
    n = len(x)
    if not (x[0] <= q <= x[n - 1]):
        return -1
    j = 0
    for k in range(n - 1):
        if x[k] <= q:
            j = k
    return j
