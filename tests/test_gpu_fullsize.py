"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Every config is compared element by element in full: y2 and every query's idx (bit for bit) and out
(north-star tolerance), the oracle running on the host cores.
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
    wl = workloads.generate(cid)
    r = parity.check_case(api, wl, nthreads=16)
    print(f"cfg{cid} full: max rel err y2 {r['y2']:.3e} out {r['out']:.3e} (literal max|y| metric "
          f"{r['out_literal']:.3e})")


@pytest.mark.parametrize("cid", [4, 5])
def test_full_size_every_query(api, cid):
    """cfg4 (4,096 x 4,096 fp64, 268M sorted queries) and cfg5 (one 2^26-knot curve, 2^28 unsorted
    queries) in the launch configuration bench.py times (one spline_build_eval call): y2 and EVERY
    query's idx and out against the oracle run end to end on the host cores."""
    wl = workloads.generate(cid)
    tol = parity.tol_for(wl.np_dtype)
    t = parity.to_dev
    x, y, q = t(wl.x), t(wl.y), t(wl.q)
    yp1 = t(wl.yp1) if wl.yp1 is not None else None
    ypn = t(wl.ypn) if wl.ypn is not None else None
    api.status()
    y2, out, idx = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags)
    torch.cuda.synchronize()
    assert api.status() == 0
    y2_ref = parity.oracle_build(wl, nthreads=16)
    e = parity.y2_rel_err(y2.cpu().numpy(), y2_ref)
    assert np.all(e <= tol), e.max()
    del y2
    out_ref, idx_ref, nbad = oracle.evaluate(wl.x, wl.y, y2_ref, wl.q, nthreads=32)
    assert nbad == 0
    gi = idx.cpu().numpy()
    del idx
    assert np.array_equal(gi, idx_ref), int(np.count_nonzero(gi != idx_ref))
    del gi, idx_ref
    go = out.cpu().numpy()
    eo = parity.out_rel_err(go, out_ref, wl.y)
    assert np.all(eo <= tol), eo.max()
    lit = parity.out_rel_err_literal(go, out_ref, wl.y)  # BASELINE's literal max|y| normalisation (reported)
    print(f"cfg{cid} full, every query: y2 {e.max():.3e} out {eo.max():.3e} (literal max|y| metric {lit.max():.3e})")


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
