"""GPU parity of spline_build_eval (build and evaluate in one call).

Two bars: (1) the oracle, element by element (bit-exact idx; y2 and out within the north-star
tolerances, reading c2) and (2) bitwise identity with spline_build followed by
spline_eval on the same inputs -- the fused kernel runs the same arithmetic on chip.
Cases span several work items and CTAs, ragged last items, chunked single curves, both solver
kinds (registers for n <= 8, two-ended sweep otherwise), both search modes, the fallback for
shapes the fused kernel does not take, bad knots and out-of-range / NaN queries.
"""
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


def _dev(wl):
    t = parity.to_dev
    return (t(wl.x), t(wl.y), t(wl.q), t(wl.yp1) if wl.yp1 is not None else None,
            t(wl.ypn) if wl.ypn is not None else None)


def check_fused(api, wl, flags=None, nthreads=8):
    flags = wl.flags if flags is None else flags
    dt = wl.np_dtype
    tol = parity.tol_for(dt)
    x, y, q, yp1, ypn = _dev(wl)
    api.status()
    y2, out, idx = api.build_eval(x, y, q, wl.bc, yp1, ypn, flags | api.PATH_FUSED)
    bits = api.status()
    # (1) the oracle
    y2_ref = parity.oracle_build(wl, nthreads)
    out_ref, idx_ref, nbad = oracle.evaluate(wl.x, wl.y, y2_ref, wl.q, nthreads=nthreads)
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    e2 = parity.y2_rel_err(y2.cpu().numpy(), y2_ref, wl.x, wl.y)
    eo = parity.out_rel_err(out.cpu().numpy(), out_ref, wl.y)
    assert np.all(e2 <= tol), f"y2 max rel err {e2.max():.3e}"
    assert np.all(eo <= tol), f"out max rel err {eo.max():.3e}"
    assert (bits & api.STATUS_Q_OUT_OF_RANGE) == (api.STATUS_Q_OUT_OF_RANGE if nbad else 0)
    # (2) bitwise the separate path
    y2s = api.build(x, y, wl.bc, yp1, ypn)
    outs, idxs = api.evaluate(x, y, y2s, q, flags)
    assert torch.equal(y2.view(torch.int8), y2s.view(torch.int8)), "y2 differs from spline_build"
    assert torch.equal(idx, idxs)
    assert torch.equal(out.view(torch.int8), outs.view(torch.int8)), "out differs from build -> eval"
    # (3) without y2 / without idx: same out
    F = flags | api.PATH_FUSED
    none, out2, idx2 = api.build_eval(x, y, q, wl.bc, yp1, ypn, F, want_y2=False)
    assert none is None and torch.equal(out2.view(torch.int8), out.view(torch.int8)) and torch.equal(idx2, idx)
    _, out3, none3 = api.build_eval(x, y, q, wl.bc, yp1, ypn, F, want_idx=False)
    assert none3 is None and torch.equal(out3.view(torch.int8), out.view(torch.int8))
    # (4) the other path choices give the same bits
    for pf in (0, api.PATH_SPLIT):
        y2b, outb, idxb = api.build_eval(x, y, q, wl.bc, yp1, ypn, flags | pf)
        assert torch.equal(y2b.view(torch.int8), y2.view(torch.int8)) and torch.equal(idxb, idx)
        assert torch.equal(outb.view(torch.int8), out.view(torch.int8))
    return float(e2.max()), float(eo.max())


@pytest.mark.parametrize("kw", [dict(), dict(batch=3), dict(m=4000), dict(m=100000)])
def test_fused_cfg1_babe_f64(api, kw):
    check_fused(api, workloads.generate(1, **kw))


@pytest.mark.parametrize("kw", [dict(batch=4096), dict(batch=1001, m=252), dict(batch=77, n=64, m=4),
                                dict(batch=33, n=128, m=64), dict(batch=5, n=24, m=2048),
                                dict(batch=1, n=64, m=10000)])
def test_fused_cfg2_babe_f32(api, kw):
    check_fused(api, workloads.generate(2, **kw))


@pytest.mark.parametrize("kw", [dict(batch=20000), dict(batch=4099, m=36), dict(batch=50, n=4, m=8),
                                dict(batch=129, n=8, m=4096)])
def test_fused_cfg3_regs_f32(api, kw):
    wl = workloads.generate(3, **kw)
    check_fused(api, wl)
    check_fused(api, wl, flags=0)  # bisection instead of the uniform-grid index: same answer


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
@pytest.mark.parametrize("dt,n", [(np.float32, 8), (np.float32, 12), (np.float64, 6), (np.float64, 10),
                                  (np.float64, 128), (np.float32, 100)])
def test_fused_bc_dtype_grid(api, bc, dt, n):
    rng = np.random.default_rng(1000 * n + bc)
    B, m = 300, 40
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.05, axis=1).astype(dt)
    y = np.cumsum(rng.normal(size=(B, n)), axis=1).astype(dt)
    q = rng.uniform(x[:, :1], x[:, -1:], (B, m)).astype(dt)
    q[:, :5] = x[:, [0, n - 1, n // 2, 1, n - 2]]  # exact knots: ties, both ends
    yp1 = rng.normal(size=B).astype(dt)
    ypn = rng.normal(size=B).astype(dt)
    spec = workloads.ConfigSpec(0, "t", B, n, m, "f32" if dt == np.float32 else "f64", bc, 0, 0)
    check_fused(api, workloads.Workload(spec, x, y, q, yp1, ypn, bc, 0))


@pytest.mark.parametrize("kw", [dict(n=63, m=255), dict(n=200, m=64), dict(n=5, m=33)])
def test_fused_fallback_shapes(api, kw):
    """Shapes the fused kernel does not take still give the oracle's answer (two kernels)."""
    check_fused(api, workloads.generate(2, batch=300, **kw))


def test_fused_unaligned_views(api):
    wl = workloads.generate(2, batch=200)
    x, y, q, yp1, ypn = _dev(wl)
    # offset by one element: not 16-byte aligned -> the separate kernels
    xs = torch.empty(x.numel() + 1, dtype=x.dtype, device=x.device)[1:].view_as(x).copy_(x)
    y2, out, idx = api.build_eval(xs, y, q, wl.bc, yp1, ypn, api.PATH_FUSED)
    y2r, outr, idxr = api.build_eval(x, y, q, wl.bc, yp1, ypn, api.PATH_FUSED)
    assert torch.equal(idx, idxr) and torch.equal(out.view(torch.int8), outr.view(torch.int8))
    assert torch.equal(y2.view(torch.int8), y2r.view(torch.int8))


def test_fused_bad_knots_and_out_of_range(api):
    wl = workloads.generate(2, batch=64)
    wl.x[5, 10] = wl.x[5, 9]          # repeated knot
    wl.y[9, 3] = np.nan                # non-finite value
    wl.q[2, 7] = wl.x[2, 0] - 1.0      # below the range
    wl.q[3, 8] = np.nan
    x, y, q, yp1, ypn = _dev(wl)
    api.status()
    y2, out, idx = api.build_eval(x, y, q, wl.bc, yp1, ypn, api.PATH_FUSED)
    bits = api.status()
    assert bits == api.STATUS_BAD_KNOTS | api.STATUS_Q_OUT_OF_RANGE
    z = y2.cpu().numpy()
    assert np.all(np.isnan(z[5])) and np.all(np.isnan(z[9]))
    ok = [c for c in range(64) if c not in (5, 9)]
    assert np.all(np.isfinite(z[ok]))
    i = idx.cpu().numpy()
    assert i[2, 7] == -1 and i[3, 8] == -1 and np.isnan(out[2, 7].item()) and np.isnan(out[3, 8].item())
    y2s = api.build(x, y, wl.bc, yp1, ypn)
    outs, idxs = api.evaluate(x, y, y2s, q, 0)
    api.status()
    assert torch.equal(idx, idxs)
    assert torch.equal(out.view(torch.int8), outs.view(torch.int8))


def test_fused_build_only_and_empty(api):
    wl = workloads.generate(2, batch=10, m=4)
    x, y, q, yp1, ypn = _dev(wl)
    q0 = q[:, :0].contiguous()
    y2, out, idx = api.build_eval(x, y, q0, wl.bc, yp1, ypn)
    assert out.shape == (10, 0)
    assert torch.equal(y2.view(torch.int8), api.build(x, y, wl.bc, yp1, ypn).view(torch.int8))
    assert api.status() == 0


# ---- k_tile_eval: mid-length curves with sorted queries solved and evaluated in one kernel ----

@pytest.mark.parametrize("kw", [dict(batch=6, n=4096, m=16384), dict(batch=5, n=1000, m=3001),
                                dict(batch=3, n=129, m=2048), dict(batch=2, n=3000, m=100),
                                dict(batch=2, n=4096, m=65536), dict(batch=40, n=257, m=9000)])
def test_tile_eval_cfg4_f64(api, kw):
    """cfg4-shaped (fp64, clamped, sorted): one launch per call (k_tile_eval) -- dense runs (record
    window), sparse runs, odd m (scalar query I/O), one leaf row per thread (n <= 256), several
    query chunks per curve (few curves), against the oracle and bitwise the split path."""
    check_fused(api, workloads.generate(4, **kw))


@pytest.mark.parametrize("bc", [0, 3])
@pytest.mark.parametrize("dt,n,m", [(np.float32, 8000, 40000), (np.float32, 700, 6000), (np.float64, 2500, 777)])
def test_tile_eval_dtypes_sorted(api, bc, dt, n, m):
    rng = np.random.default_rng(7 * n + bc)
    B = 7
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.05, axis=1).astype(dt)
    y = np.cumsum(rng.normal(size=(B, n)), axis=1).astype(dt)
    q = np.sort(rng.uniform(x[:, :1], x[:, -1:], (B, m)).astype(dt), axis=1)
    q[:, 0] = x[:, 0]
    q[:, -1] = x[:, -1]
    q[:, m // 2] = x[:, n // 2]          # an exact interior knot (tie) inside the sorted run
    q = np.sort(q, axis=1)
    yp1 = rng.normal(size=B).astype(dt)
    ypn = rng.normal(size=B).astype(dt)
    spec = workloads.ConfigSpec(0, "t", B, n, m, "f32" if dt == np.float32 else "f64", bc, 1, 0)
    check_fused(api, workloads.Workload(spec, x, y, q, yp1, ypn, bc, workloads.FLAG_Q_SORTED))


def test_tile_eval_wrong_sorted_hint_and_bad_data(api):
    """The sorted hint is only a hint: unsorted queries, out-of-range / NaN queries and a curve
    with bad knots give the oracle's answer (and the split path's bits) in the fused kernel."""
    wl = workloads.generate(4, batch=4, n=2048, m=8192)
    rng = np.random.default_rng(3)
    wl.q[1] = rng.permutation(wl.q[1])          # unsorted despite the flag
    wl.q[2, 100] = wl.x[2, 0] - 1.0             # below the range
    wl.q[2, 101] = np.nan
    wl.q[3, 5000] = wl.x[3, -1] + 1.0           # above the range
    check_fused(api, wl)
    wl.x[0, 1000] = wl.x[0, 999]                # curve 0: a repeated knot -> NaN y2 and out
    x, y, q, yp1, ypn = _dev(wl)
    api.status()
    y2, out, idx = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags)
    assert api.status() & api.STATUS_BAD_KNOTS
    assert torch.isnan(y2[0]).all() and torch.isfinite(y2[1:]).all()
    y2s = api.build(x, y, wl.bc, yp1, ypn)
    outs, idxs = api.evaluate(x, y, y2s, q, wl.flags)
    api.status()
    assert torch.equal(idx, idxs) and torch.equal(out.view(torch.int8), outs.view(torch.int8))


# ---- k_build_eval_warp: many K1h-sized curves (cfg2), the automatic path ----------------------

def check_auto(api, wl, nthreads=8):
    """The automatic spline_build_eval path against the oracle and bitwise against the split
    path (K1h + k_eval_curvewarp), with and without y2 / idx."""
    tol = parity.tol_for(wl.np_dtype)
    x, y, q, yp1, ypn = _dev(wl)
    api.status()
    y2, out, idx = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags)
    bits = api.status()
    y2_ref = parity.oracle_build(wl, nthreads)
    out_ref, idx_ref, nbad = oracle.evaluate(wl.x, wl.y, y2_ref, wl.q, nthreads=nthreads)
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    good = np.all(np.isfinite(y2_ref), axis=1)
    e2 = parity.y2_rel_err(y2.cpu().numpy()[good], y2_ref[good], wl.x[good], wl.y[good])
    eo = parity.out_rel_err(out.cpu().numpy()[good], out_ref[good], wl.y[good])
    assert np.all(e2 <= tol) and np.all(eo <= tol), (e2.max(), eo.max())
    assert bool(bits & api.STATUS_Q_OUT_OF_RANGE) == bool(nbad)
    assert bool(bits & api.STATUS_BAD_KNOTS) == (not good.all())
    y2s, outs, idxs = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_SPLIT)
    api.status()
    assert torch.equal(y2.view(torch.int8), y2s.view(torch.int8))
    assert torch.equal(idx, idxs) and torch.equal(out.view(torch.int8), outs.view(torch.int8))
    none, out2, none2 = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, want_y2=False, want_idx=False)
    api.status()
    assert none is None and none2 is None and torch.equal(out2.view(torch.int8), out.view(torch.int8))


@pytest.mark.parametrize("kw", [dict(batch=4096), dict(batch=1000, m=4), dict(batch=2999, m=1000),
                                dict(batch=700, n=32, m=64), dict(batch=650, n=16, m=12),
                                dict(batch=20000, m=8)])
def test_build_eval_warp_cfg2(api, kw):
    """cfg2-shaped calls big enough for k_build_eval_warp: warp ranges that are not whole groups of
    16 curves, fewer query vectors than lanes (m = 4), many per lane (m = 1000), n = 16/32/64."""
    check_auto(api, workloads.generate(2, **kw))


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_build_eval_warp_f64_n16(api, bc):
    rng = np.random.default_rng(50 + bc)
    B, n, m = 1500, 16, 90
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.01, axis=1)
    y = np.cumsum(rng.normal(size=(B, n)), axis=1)
    q = rng.uniform(x[:, :1], x[:, -1:], (B, m))
    q[:, :4] = x[:, [0, n - 1, 7, 1]]  # both ends and interior knots (ties)
    spec = workloads.ConfigSpec(0, "t", B, n, m, "f64", bc, 0, 0)
    check_auto(api, workloads.Workload(spec, x, y, q, rng.normal(size=B), rng.normal(size=B), bc, 0))


def test_build_eval_warp_bad_data(api):
    """Bad knots (NaN y2 and out for that curve only, BAD_KNOTS), out-of-range and NaN queries in
    the middle of a warp's range, on the automatic path."""
    wl = workloads.generate(2, batch=1200, m=256)
    wl.x[17, 30] = wl.x[17, 29]
    wl.y[600, 0] = np.inf
    wl.q[5, 3] = wl.x[5, -1] + 1.0
    wl.q[1100, 255] = np.nan
    wl.q[18, 0] = wl.x[18, 0] - 1e-3
    check_auto(api, wl)
