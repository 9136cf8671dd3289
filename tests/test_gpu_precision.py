"""The paper's Quality Checks on the GPU path, fp64: second derivatives of the
hand curve against exact rationals on the decimal inputs, and the 2048-point
sweep of the twist spline.  Bounds: the paper's own "our" MSEs are 4.3e-26 (natural), 3.4e-28
(flat), 2.4e-26 (twist) and 1.6e-30 (sweep); differences of that kind are chaotic rounding
(P:1287-1296), so the pins allow two orders of magnitude: 1e-23 / 1e-23 / 1e-23 / 1e-27."""
import os
import sys

import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


def test_quality_checks_fp64():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import precision_report
    r = precision_report.run(torch.float64)
    assert r["nat"]["mse"] < 1e-23 and r["flat"]["mse"] < 1e-23 and r["twist"]["mse"] < 1e-23
    assert r["sweep"]["mse"] < 1e-27
    assert r["nat"]["delta"][0] == 0.0 and r["nat"]["delta"][-1] == 0.0  # natural ends exact
