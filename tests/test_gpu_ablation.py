"""GPU parity of spline_eval_ablation: the paper's interpolation variants on the
sorted-run eval kernel.  idx is bit-exact for every form; out meets the north-star tolerance
(reading c2) against the CPU oracle; the product form is bitwise spline_eval; the
no-op form returns y_idx."""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2001_09253_b200 import _lib, workloads



@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_09253_b200 import api as a
    a.status()
    return a


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n,batch,shuffle", [(1000, 8, False), (37, 100, True), (5000, 3, False)])
def test_forms_vs_oracle(api, dt, n, batch, shuffle):
    x, y, q = workloads.sweep_curves(n, batch, seed=7, dtype=dt)
    if dt == np.float32:  # keep fp32 knots strictly increasing after rounding (reading c11)
        for j in range(1, n):
            x[:, j] = np.where(x[:, j] <= x[:, j - 1], np.nextafter(x[:, j - 1], np.float32(np.inf)), x[:, j])
        q = np.clip(q, x[:, :1], x[:, -1:])
    if shuffle:
        q = np.random.default_rng(1).permutation(q, axis=1)
    y2_ref, _ = oracle.build_y2(x, y, 0, None, None, nthreads=8)
    out_ref, idx_ref, _ = oracle.evaluate(x, y, y2_ref, q, nthreads=8)
    X, Y, Z, Q = (parity.to_dev(a) for a in (x, y, y2_ref.astype(dt), q))
    base, base_idx = api.evaluate(X, Y, Z, Q, 0)
    for form in _lib.FORMS:
        out, idx = api.evaluate_ablation(X, Y, Z, Q, form)
        np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref, err_msg=form)
        o = out.cpu().numpy()
        if form == "noop":
            assert np.array_equal(o, np.take_along_axis(y, idx_ref, axis=1))
            continue
        e = parity.out_rel_err(o, out_ref, y)
        assert np.all(e <= parity.tol_for(dt)), f"{form}: {e.max():.3e}"
        if form == "record":
            assert torch.equal(out.view(torch.int8), base.view(torch.int8))
    assert api.status() == 0


def test_sweep_schedule_matches_paper():
    s = workloads.sweep_schedule(5)
    assert s[0] == 4 and s[-1] == 1 << 20
    assert all(a < b for a, b in zip(s, s[1:]))
