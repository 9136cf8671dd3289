"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

cfg2/cfg3 are compared element by element in full; cfg4/cfg5 compare y2 in full and
eval on sampled queries the oracle computes one by one (bisection + Eq. nr_formula).
"""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2001_09253_b200 import workloads

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_09253_b200 import api as a
    return a


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_full_size_elementwise(api, cid):
    r = parity.check_case(api, workloads.generate(cid), nthreads=16)
    print(f"cfg{cid} full: max rel err y2 {r['y2']:.3e} out {r['out']:.3e}")


@pytest.mark.parametrize("cid,curves,qs", [(4, 24, None), (5, 1, 1 << 20)])
def test_full_size_sampled(api, cid, curves, qs):
    wl = workloads.generate(cid)
    dt = wl.np_dtype
    tol = parity.tol_for(dt)
    x, y, y2 = parity.gpu_build(api, wl)
    q = parity.to_dev(wl.q)
    out, idx = api.evaluate(x, y, y2, q, wl.flags)
    torch.cuda.synchronize()
    assert api.status() == 0
    rng = np.random.default_rng(123)
    if cid == 4:
        y2_ref = parity.oracle_build(wl, nthreads=16)
        e = parity.y2_rel_err(y2.cpu().numpy(), y2_ref)
        assert np.all(e <= tol), e.max()
        sel = np.sort(rng.choice(wl.batch, curves, replace=False))
        out_ref, idx_ref, _ = oracle.evaluate(wl.x[sel], wl.y[sel], y2_ref[sel], wl.q[sel], nthreads=16)
        np.testing.assert_array_equal(idx.cpu().numpy()[sel], idx_ref)
        eo = parity.out_rel_err(out.cpu().numpy()[sel], out_ref, wl.y[sel])
        assert np.all(eo <= tol), eo.max()
    else:
        y2_ref = parity.oracle_build(wl, nthreads=1)
        e = parity.y2_rel_err(y2.cpu().numpy(), y2_ref)
        assert np.all(e <= tol), e.max()
        ks = np.sort(rng.choice(wl.m, qs, replace=False))
        qsamp = wl.q[0, ks][None]
        out_ref, idx_ref, _ = oracle.evaluate(wl.x, wl.y, y2_ref, qsamp, nthreads=16)
        kt = torch.from_numpy(ks).cuda()
        np.testing.assert_array_equal(idx[0, kt].cpu().numpy(), idx_ref[0])
        eo = parity.out_rel_err(out[0, kt].cpu().numpy()[None], out_ref, wl.y)
        assert np.all(eo <= tol), eo.max()
    print(f"cfg{cid} full: y2 {e.max():.3e} out(sampled) {eo.max():.3e}")


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_full_size_fused_equals_split(api, cid):
    """The fused kernel at full size (many items per persistent CTA: the hand-off protocol
    runs its whole phase cycle many times) gives bitwise the split path's y2, out and idx."""
    wl = workloads.generate(cid)
    t = parity.to_dev
    x, y, q = t(wl.x), t(wl.y), t(wl.q)
    yp1 = t(wl.yp1) if wl.yp1 is not None else None
    ypn = t(wl.ypn) if wl.ypn is not None else None
    api.status()
    y2f, outf, idxf = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_FUSED)
    y2s, outs, idxs = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_SPLIT)
    torch.cuda.synchronize()
    assert api.status() == 0
    assert torch.equal(y2f.view(torch.int8), y2s.view(torch.int8))
    assert torch.equal(idxf, idxs)
    assert torch.equal(outf.view(torch.int8), outs.view(torch.int8))
