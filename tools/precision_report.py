"""extended-precision accuracy report of the GPU path, in the form of the
paper's Quality Checks: the hand curve, natural / flat
(y' = 0) / twist (y'_1 = -1, y'_n = 1) second derivatives against the "true" values, their mean
square errors (Tables mse_nat, mse_flat, mse_twist), and the 2048-point sweep of the twist spline
(Table mse_full).  "True" = exact rational arithmetic on the DECIMAL inputs (the paper used
mpmath at 30 digits on the decimal strings; exact rationals are the limit of that).
The GPU runs in fp64 (the paper's precision) and, for reference, fp32.

    python tools/precision_report.py [OUT.json]      (needs a GPU; prints a table + one JSON line)
"""
import json
import os
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import refmath  # noqa: E402  (exact rational elimination of the row definitions)
from paper_2001_09253_b200 import api  # noqa: E402

KNOTS = ["0", "0.5", "1", "1.01", "1.25", "1.5", "1.58", "1.79", "2.12", "2.30", "2.402", "2.451", "2.5"]
VALUES = ["1", "1.2", "2", "0.25", "0.25", "0.25", "0.63", "0.96", "1.17", "1.23", "1.245", "1.249", "1.25"]
CASES = {"nat": (0, 0, 0), "flat": (3, 0, 0), "twist": (3, -1, 1)}
PAPER_MSE = {"nat": 4.30368e-26, "flat": 3.36714e-28, "twist": 2.36125e-26, "sweep": 1.5724e-30}  # "our" column


def exact_y2(bc, yp1, ypn):
    xs = [Fraction(v) for v in KNOTS]
    ys = [Fraction(v) for v in VALUES]
    M, d = refmath.dense_system(xs, ys, bc, Fraction(yp1), Fraction(ypn), num=Fraction)
    n = len(d)
    for k in range(n):
        for r in range(k + 1, n):
            if M[r][k] != 0:
                f = M[r][k] / M[k][k]
                for c in range(k, n):
                    M[r][c] -= f * M[k][c]
                d[r] -= f * d[k]
    sol = [Fraction(0)] * n
    for k in range(n - 1, -1, -1):
        sol[k] = (d[k] - sum(M[k][c] * sol[c] for c in range(k + 1, n))) / M[k][k]
    return sol


def exact_interp(q, j, y2):
    a, b = Fraction(KNOTS[j]), Fraction(KNOTS[j + 1])
    h = b - a
    A, B = (b - q) / h, (q - a) / h
    return (A * Fraction(VALUES[j]) + B * Fraction(VALUES[j + 1]) + (A ** 3 - A) * h * h / 6 * y2[j]
            + (B ** 3 - B) * h * h / 6 * y2[j + 1])


def run(dtype):
    dev = torch.device("cuda")
    x = torch.tensor([float(v) for v in KNOTS], dtype=dtype, device=dev)
    y = torch.tensor([float(v) for v in VALUES], dtype=dtype, device=dev)
    res = {}
    api.status()  # clear bits left by earlier work on this device
    for name, (bc, yp1, ypn) in CASES.items():
        true = exact_y2(bc, yp1, ypn)
        kw = {} if bc == 0 else dict(yp1=float(yp1), ypn=float(ypn))
        y2 = api.build(x, y, bc, **kw).cpu().double().numpy()
        delta = [float(Fraction(float(g)) - t) for g, t in zip(y2, true)]
        res[name] = {"delta": delta, "mse": float(np.mean(np.square(delta)))}
        if name == "twist":
            qs = np.linspace(0.0, 2.5, 2048)
            q = torch.tensor(qs, dtype=dtype, device=dev)
            out, idx = api.evaluate(x, y, api.build(x, y, bc, **kw), q, api.Q_SORTED)
            out, idx = out.cpu().double().numpy(), idx.cpu().numpy()
            qd = q.cpu().double().numpy()
            errs = []
            for k in range(len(qs)):
                qf = Fraction(float(qd[k]))
                # the true value on the true (decimal-knot) interval
                j = max(i for i in range(len(KNOTS) - 1) if Fraction(KNOTS[i]) <= qf)
                errs.append(float(Fraction(float(out[k])) - exact_interp(qf, j, true)))
            res["sweep"] = {"mse": float(np.mean(np.square(errs))), "max_abs": float(np.max(np.abs(errs))),
                            "points": len(qs)}
    assert api.status() == 0
    return res


def main():
    if not torch.cuda.is_available():
        raise SystemExit("needs a CUDA device")
    rep = {"mode": "precision", "reference": "exact rationals on the decimal inputs (paper: mpmath, 30 digits)",
           "paper_mse_our": PAPER_MSE, "f64": run(torch.float64), "f32": run(torch.float32),
           "knots": KNOTS, "values": VALUES}
    print(f"{'case':8s} {'GPU f64 MSE':>14s} {'paper (CPU f64)':>16s} {'GPU f32 MSE':>14s}")
    for c in ["nat", "flat", "twist", "sweep"]:
        print(f"{c:8s} {rep['f64'][c]['mse']:14.4e} {PAPER_MSE[c]:16.4e} {rep['f32'][c]['mse']:14.4e}")
    line = json.dumps(rep)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(line + "\n")
    print(line)


if __name__ == "__main__":
    main()
