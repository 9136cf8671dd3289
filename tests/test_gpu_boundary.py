"""GPU tests of the boundary's contract (include/spline.h): per-stream status words, stream
ordering of programmatic launches, and the binding's buffer checks."""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2001_09253_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_09253_b200 import api as a
    a.status()
    return a


def test_status_is_per_stream(api):
    """Bits raised on one stream are read (and cleared) by spline_status on that stream only."""
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    x = torch.tensor([[0.0, 1.0, 2.0, 3.0]], dtype=torch.float64, device="cuda")
    y = x * x
    bad = torch.tensor([[0.0, 1.0, 1.0, 3.0]], dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s1):
        api.build(bad, y)                                  # BAD_KNOTS on s1
    with torch.cuda.stream(s2):
        y2 = api.build(x, y)
        api.evaluate(x, y, y2, torch.tensor([[5.0]], dtype=torch.float64, device="cuda"))  # OUT_OF_RANGE on s2
    assert api.status(stream=s2) == api.STATUS_Q_OUT_OF_RANGE
    assert api.status(stream=s1) == api.STATUS_BAD_KNOTS
    assert api.status(stream=s1) == 0 and api.status(stream=s2) == 0
    assert api.status() == 0                               # the default stream saw nothing


@pytest.mark.parametrize("n,m", [(8, 32), (16, 64), (64, 256)])
def test_build_then_build_eval_ordering(api, n, m):
    """a build (whose kernels trigger dependent launch early) immediately followed,
    on the same stream, by a build_eval whose y IS the build's y2 output: the second call must
    see the finished y2 (compare with the oracle run on the same chain)."""
    wl = workloads.generate(3 if n == 8 else 2, batch=5000, n=n, m=m)
    x, y = parity.to_dev(wl.x), parity.to_dev(wl.y)
    q = parity.to_dev(wl.q)
    yp1 = parity.to_dev(wl.yp1) if wl.yp1 is not None else None
    ypn = parity.to_dev(wl.ypn) if wl.ypn is not None else None
    for _ in range(3):
        z = api.build(x, y, wl.bc, yp1, ypn)
        z2, out, idx = api.build_eval(x, z, q, wl.bc, yp1, ypn, wl.flags)
    torch.cuda.synchronize()
    assert api.status() == 0
    ref1, _ = oracle.build_y2(wl.x, wl.y, wl.bc, wl.yp1, wl.ypn, nthreads=8)
    zz = z.cpu().numpy()                                   # the GPU y2 is the second call's y
    ref2, _ = oracle.build_y2(wl.x, zz, wl.bc, wl.yp1, wl.ypn, nthreads=8)
    oref, iref, _ = oracle.evaluate(wl.x, zz, ref2, wl.q, nthreads=8)
    tol = parity.tol_for(wl.np_dtype)
    assert parity.y2_rel_err(zz, ref1).max() <= tol
    assert parity.y2_rel_err(z2.cpu().numpy(), ref2).max() <= tol
    assert np.array_equal(idx.cpu().numpy(), iref)
    assert parity.out_rel_err(out.cpu().numpy(), oref, zz).max() <= tol


def test_binding_checks_buffers(api):
    """every caller-supplied buffer is checked for shape, dtype, device, contiguity."""
    wl = workloads.generate(2, batch=64)
    x, y, q = parity.to_dev(wl.x), parity.to_dev(wl.y), parity.to_dev(wl.q)
    yp1, ypn = parity.to_dev(wl.yp1), parity.to_dev(wl.ypn)
    y2 = api.build(x, y, wl.bc, yp1, ypn)
    with pytest.raises(ValueError):
        api.build(x, y, wl.bc, yp1[:10], ypn)                     # short slope array
    with pytest.raises(ValueError):
        api.build(x, y, wl.bc, yp1, ypn, out=torch.empty(64, 63, device="cuda"))
    with pytest.raises(ValueError):
        api.evaluate(x, y, y2, q, out=torch.empty(64, 255, device="cuda"))
    with pytest.raises(ValueError):
        api.evaluate(x, y, y2, q, idx=torch.empty(64, 256, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        api.evaluate(x, y, y2, q, out=torch.empty(256, 64, device="cuda").t())  # not contiguous
    with pytest.raises(ValueError):
        api.build_eval(x, y, q, wl.bc, yp1, ypn, y2=torch.empty(64, 64, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        api.build_eval_host(x.cpu(), y.cpu(), q.cpu(), wl.bc, yp1.cpu(), ypn.cpu(), out=torch.empty(64, 2))
    with pytest.raises(ValueError):
        api.build_eval_host(x.cpu(), y.cpu(), q.cpu(), wl.bc, yp1, ypn.cpu())   # slope on the device
    with pytest.raises(ValueError):
        api.evaluate_ablation(x, y, y2, q, "record", out=torch.empty(3, device="cuda"))
