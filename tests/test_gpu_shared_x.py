"""Shared-knot mode (SPLINE_X_SHARED): one knot vector x (n,) for a whole
batch y (B, n).  Bar: bitwise the same call with the row repeated per curve (native kernels for
n <= 8, the broadcast fallback elsewhere), and the oracle's answer."""
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


def _bits(t):
    return t.contiguous().view(torch.int8)


def _shared_case(cid, dt=None, **kw):
    wl = workloads.generate(cid, **kw)
    x1 = wl.x[0].copy()
    if dt is not None:
        x1 = x1.astype(dt)
        wl = workloads.Workload(wl.spec, np.tile(x1, (wl.batch, 1)), wl.y.astype(dt), wl.q.astype(dt),
                                None if wl.yp1 is None else wl.yp1.astype(dt),
                                None if wl.ypn is None else wl.ypn.astype(dt), wl.bc, wl.flags)
    else:
        wl.x[:] = x1                                # every curve on the first curve's knots
        lo, hi = x1[0], x1[-1]
        wl.q[:] = np.clip(wl.q, lo, hi)
    return wl, x1


@pytest.mark.parametrize("cid,kw,dt", [(3, dict(batch=20000), None), (3, dict(batch=1001, n=5, m=12), None),
                                       (2, dict(batch=700), None), (4, dict(batch=3, n=1000, m=4000), None),
                                       (1, dict(batch=9), None), (3, dict(batch=500, n=7, m=20), np.float64)])
def test_shared_knots_bitwise_and_oracle(api, cid, kw, dt):
    wl, x1 = _shared_case(cid, dt, **kw)
    t = parity.to_dev
    X, Y, Q = t(wl.x), t(wl.y), t(wl.q)
    x1d = t(x1)
    yp1 = t(wl.yp1) if wl.yp1 is not None else None
    ypn = t(wl.ypn) if wl.ypn is not None else None
    api.status()
    # build
    z_rep = api.build(X, Y, wl.bc, yp1, ypn)
    z_sh = api.build(x1d, Y, wl.bc, yp1, ypn)
    assert torch.equal(_bits(z_rep), _bits(z_sh))
    # eval on the same y2
    o_rep, i_rep = api.evaluate(X, Y, z_rep, Q, wl.flags)
    o_sh, i_sh = api.evaluate(x1d, Y, z_rep, Q, wl.flags)
    assert torch.equal(i_rep, i_sh) and torch.equal(_bits(o_rep), _bits(o_sh))
    # build + eval in one call
    zb, ob, ib = api.build_eval(X, Y, Q, wl.bc, yp1, ypn, wl.flags)
    zs, os_, is_ = api.build_eval(x1d, Y, Q, wl.bc, yp1, ypn, wl.flags)
    assert torch.equal(_bits(zb), _bits(zs)) and torch.equal(ib, is_) and torch.equal(_bits(ob), _bits(os_))
    none, o2, _ = api.build_eval(x1d, Y, Q, wl.bc, yp1, ypn, wl.flags, want_y2=False)
    assert none is None and torch.equal(_bits(o2), _bits(ob))
    torch.cuda.synchronize()
    assert api.status() == 0
    # the oracle
    y2_ref = parity.oracle_build(wl)
    out_ref, idx_ref, _ = oracle.evaluate(wl.x, wl.y, y2_ref, wl.q, nthreads=8)
    tol = parity.tol_for(wl.np_dtype)
    assert parity.y2_rel_err(zs.cpu().numpy(), y2_ref, wl.x, wl.y).max() <= tol
    np.testing.assert_array_equal(is_.cpu().numpy(), idx_ref)
    assert parity.out_rel_err(os_.cpu().numpy(), out_ref, wl.y).max() <= tol


def test_shared_knots_host_path(api):
    wl, x1 = _shared_case(3, batch=50000)
    hx = torch.from_numpy(x1).pin_memory()
    hy, hq = torch.from_numpy(wl.y).pin_memory(), torch.from_numpy(wl.q).pin_memory()
    z, o, i = api.build_eval_host(hx, hy, hq, wl.bc, None, None, wl.flags)
    zd, od, id_ = api.build_eval(parity.to_dev(wl.x), parity.to_dev(wl.y), parity.to_dev(wl.q), wl.bc, None, None,
                                 wl.flags)
    assert torch.equal(_bits(z), _bits(zd.cpu())) and torch.equal(i, id_.cpu()) and torch.equal(_bits(o), _bits(od.cpu()))
