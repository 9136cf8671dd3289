"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle, element by element.

Sizes span several tiles / CTAs and a ragged tail; full BASELINE sizes are covered in
test_gpu_fullsize.py.  Every case is seeded (paper_2001_09253_b200.workloads).
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


# ------------------------------------------------------------ the five configs, scaled

@pytest.mark.parametrize("kw", [dict(), dict(batch=3)])
def test_cfg1(api, kw):
    parity.check_case(api, workloads.generate(1, **kw))


@pytest.mark.parametrize("kw", [dict(batch=4096), dict(batch=1001, m=255), dict(batch=77, n=63, m=31)])
def test_cfg2_k1_thomas_f32(api, kw):
    parity.check_case(api, workloads.generate(2, **kw))


@pytest.mark.parametrize("kw", [dict(batch=20000), dict(batch=4099, m=33), dict(batch=50, n=3, m=7),
                                dict(batch=1001, n=5, m=12), dict(batch=33, m=28), dict(batch=70001, n=4, m=4)])
def test_cfg3_uniform_f32(api, kw):
    parity.check_case(api, workloads.generate(3, **kw))
    parity.check_case(api, workloads.generate(3, **kw), flags=0)  # same answer without the hint


@pytest.mark.parametrize("kw", [dict(batch=6, n=4096, m=16384), dict(batch=5, n=1000, m=3001),
                                dict(batch=3, n=129, m=2048), dict(batch=2, n=3000, m=100)])
def test_cfg4_tile_sorted_f64(api, kw):
    parity.check_case(api, workloads.generate(4, **kw))
    parity.check_case(api, workloads.generate(4, **kw), flags=0)


@pytest.mark.parametrize("kw", [dict(n=(1 << 17), m=1 << 18), dict(n=(1 << 17) + 123, m=10007),
                                dict(n=600 * 4096 + 17, m=1 << 16)])
def test_cfg5_spike_f64(api, kw):
    parity.check_case(api, workloads.generate(5, **kw), nthreads=8)


# ------------------------------------------------------------ every kernel x dtype

@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n", [3, 5, 16, 32, 64, 128, 129, 700, 4096, 4097, 9000, 70000])
@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_build_all_paths(api, dt, n, bc):
    rng = np.random.default_rng(n * 10 + bc)
    B = 3
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.05, axis=1).astype(dt)
    y = np.cumsum(rng.normal(size=(B, n)), axis=1).astype(dt)
    yp1 = rng.normal(size=B).astype(dt)
    ypn = rng.normal(size=B).astype(dt)
    wl = workloads.Workload(workloads.CONFIGS[2], x, y, x[:, :4].copy(), yp1, ypn, bc, 0)
    wl.spec = workloads.ConfigSpec(0, "t", B, n, 4, "f32" if dt == np.float32 else "f64", bc, 0, 0)
    parity.check_case(api, wl, y2_only=True)
    if not bc & 1 or not bc & 2:
        _, _, y2 = parity.gpu_build(api, wl)
        y2 = y2.cpu().numpy()
        if not bc & 1:
            assert np.all(y2[:, 0] == 0)
        if not bc & 2:
            assert np.all(y2[:, -1] == 0)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n,m,flags", [(16, 1000, 0), (64, 256, 1), (8, 32, 2), (4096, 20000, 1),
                                       (4096, 3000, 0), (5000, 4000, 0), (200000, 5000, 0), (200000, 5000, 1)])
def test_eval_all_paths_with_ties(api, dt, n, m, flags):
    """Queries on exact knots (interior ties, x_0, x_{n-1}), out of range and NaN; bit-exact idx."""
    rng = np.random.default_rng(n + m)
    B = 2
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.01, axis=1).astype(dt)
    y = rng.normal(size=(B, n)).astype(dt)
    y2 = rng.normal(size=(B, n)).astype(dt)
    q = rng.uniform(x[:, :1], x[:, -1:], (B, m)).astype(dt)
    q[:, : m // 10] = x[:, rng.integers(0, n, m // 10)][0]          # exact knot hits
    q[:, 0], q[:, 1] = x[:, 0], x[:, -1]
    q[:, 2] = x[:, 0] - 1
    q[:, 3] = x[:, -1] + 1
    q[:, 4] = np.nan
    q[1] = x[1, :1] + (q[0] - x[0, :1])  # different curve, shifted queries
    if flags & 1:
        q = np.sort(q, axis=1)  # NaN sorts to the end
    out_ref, idx_ref, nbad = oracle.evaluate(x, y, y2, q)
    api.status()
    out, idx = api.evaluate(parity.to_dev(x), parity.to_dev(y), parity.to_dev(y2), parity.to_dev(q), flags)
    bits = api.status()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    e = parity.out_rel_err(out.cpu().numpy(), out_ref, y)
    assert np.all(e <= parity.tol_for(dt))
    assert (bits & api.STATUS_Q_OUT_OF_RANGE) == (api.STATUS_Q_OUT_OF_RANGE if nbad else 0)


def test_wrong_hints_do_not_change_results(api):
    wl = workloads.generate(2, batch=500)  # unsorted, non-uniform
    x, y, y2 = parity.gpu_build(api, wl)
    q = parity.to_dev(wl.q)
    base = api.evaluate(x, y, y2, q, 0)
    for flags in (1, 2, 3):
        o, i = api.evaluate(x, y, y2, q, flags)
        assert torch.equal(i, base[1])
        assert torch.allclose(o, base[0], rtol=0, atol=0, equal_nan=True)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [6, 16, 32, 64, 1000, 20000])
def test_bad_knots_status_and_nan(api, n, dt):
    rng = np.random.default_rng(n)
    x = np.cumsum(rng.uniform(0.5, 1.5, (4, n)), axis=1).astype(dt)
    y = rng.normal(size=(4, n)).astype(dt)
    x[1, n // 2] = x[1, n // 2 - 1]  # duplicate knot
    y[2, 1] = np.inf
    api.status()
    y2 = api.build(parity.to_dev(x), parity.to_dev(y), 0).cpu().numpy()
    bits = api.status()
    assert bits & api.STATUS_BAD_KNOTS
    assert np.all(np.isnan(y2[1])) and np.all(np.isnan(y2[2]))
    ref, _ = oracle.build_y2(x[[0, 3]], y[[0, 3]], 0)
    assert np.all(parity.y2_rel_err(y2[[0, 3]], ref) <= parity.tol_for(dt))


def test_idx_optional_and_empty(api):
    wl = workloads.generate(2, batch=64)
    x, y, y2 = parity.gpu_build(api, wl)
    q = parity.to_dev(wl.q)
    o1, i1 = api.evaluate(x, y, y2, q, 0)
    o2, i2 = api.evaluate(x, y, y2, q, 0, want_idx=False)
    assert i2 is None and torch.equal(o1, o2)
    e = torch.empty((64, 0), dtype=x.dtype, device=x.device)
    o3, _ = api.evaluate(x, y, y2, e, 0)
    assert o3.shape == (64, 0)
    z = torch.empty((0, 64), dtype=x.dtype, device=x.device)
    assert api.build(z, z, 0).shape == (0, 64)


def test_linear_and_cubic_closed_forms_gpu(api):
    """Closed forms through the GPU path: linear data -> y2 == 0; clamped cubic reproduced."""
    x = np.linspace(-1.0, 2.0, 300)
    y = 3 * x - 2
    y2 = api.build(parity.to_dev(x), parity.to_dev(y), 0).cpu().numpy()
    assert np.max(np.abs(y2)) <= 1e-12 * 6 * 3 / (3 / 299)   # reading c2's fallback scale
    f = lambda t: 1 - t + 0.5 * t ** 2 + 0.25 * t ** 3
    fp = lambda t: -1 + t + 0.75 * t ** 2
    for n in (50, 3000, 20000):
        xx = np.linspace(-2.0, 2.0, n)
        y2 = api.build(parity.to_dev(xx), parity.to_dev(f(xx)), 3, fp(-2.0), fp(2.0)).cpu().numpy()
        # conditioning (reading c16): the rounding of y (eps max|y| per value) enters
        # dd_j = (y_{j+1} - y_j)/h as 2 eps max|y|/h, d_j = 6(dd_j - dd_{j-1}) as 24 eps max|y|/h,
        # and the solve divides by the diagonal 4h: |dy2| <~ 6 eps max|y| / h^2 -- 4x headroom
        # (the oracle, doing the same arithmetic in the same precision, has the same error)
        h = xx[1] - xx[0]
        bound = 4 * 6 * np.finfo(np.float64).eps * np.max(np.abs(f(xx))) / h ** 2
        assert np.max(np.abs(y2 - (1 + 1.5 * xx))) <= bound, (n, np.max(np.abs(y2 - (1 + 1.5 * xx))), bound)


@pytest.mark.parametrize("cid,kw", [(2, dict(batch=40000, m=64)), (2, dict(batch=40000, m=256)),
                                    (3, dict(batch=300000, m=8)), (4, dict(batch=700, n=64, m=512))])
def test_persistent_multi_item(api, cid, kw):
    """Enough curves that every persistent CTA (K1 pipeline, staged eval) runs several items."""
    parity.check_case(api, workloads.generate(cid, **kw))


def test_bad_knots_in_multi_tile_pipeline(api):
    rng = np.random.default_rng(77)
    B, n = 30000, 64
    x = np.cumsum(rng.uniform(0.5, 1.5, (B, n)), axis=1).astype(np.float32)
    y = rng.normal(size=(B, n)).astype(np.float32)
    bad = rng.choice(B, 50, replace=False)
    x[bad, 10] = x[bad, 9]
    api.status()
    y2 = api.build(parity.to_dev(x), parity.to_dev(y), 0).cpu().numpy()
    assert api.status() & api.STATUS_BAD_KNOTS
    assert np.all(np.isnan(y2[bad]))
    good = np.setdiff1d(np.arange(B), bad)
    assert np.all(np.isfinite(y2[good]))


@pytest.mark.parametrize("world,n,bc", [(2, 20000, 0), (3, 50001, 3), (8, 1 << 18, 0), (4, 9000, 1)])
def test_spike_seam_emulated_ranks(api, world, n, bc):
    """The multi-GPU SPIKE seam with G ranks emulated on one GPU (the kernels of different
    ranks never wait on one another, so running them one after another is exact): every
    rank's reduce, an all-gather by concatenation, every rank's finish -> the oracle's y2."""
    from paper_2001_09253_b200 import dist as sdist
    wl = workloads.generate(5, n=n, m=16)
    x, y = parity.to_dev(wl.x[0]), parity.to_dev(wl.y[0])
    s0 = torch.full((1,), 0.3, dtype=x.dtype, device=x.device)
    s1 = torch.full((1,), -0.2, dtype=x.dtype, device=x.device)
    recs, wss = [], []
    for r in range(world):
        rb, re = sdist.shard_rows(n, world, r)
        ws = api.spike_workspace(n, rb, re, x.dtype, x.device)
        rec = torch.empty(6, dtype=x.dtype, device=x.device)
        api.spike_reduce(x, y, rb, re, bc, s0, s1, rec, ws)
        recs.append(rec)
        wss.append(ws)
    allr = torch.cat(recs)
    parts = []
    for r in range(world):
        rb, re = sdist.shard_rows(n, world, r)
        y2s = torch.empty(re - rb, dtype=x.dtype, device=x.device)
        api.spike_finish(x, y, rb, re, bc, s0, s1, allr, world, r, y2s, wss[r])
        parts.append(y2s)
    y2 = torch.cat(parts).cpu().numpy()
    ref, _ = oracle.build_y2(wl.x[0], wl.y[0], bc, [0.3], [-0.2])
    assert parity.y2_rel_err(y2[None], ref[None]).max() <= 1e-12


def test_spike_record_matches_dense_block(api):
    """The CUDA block record equals the dense-solve record of the same rows (seam contract)."""
    import seam_ref
    wl = workloads.generate(5, n=3000, m=16)
    ops = seam_ref.SeamRefOps(wl.x[0], wl.y[0], 3, 0.5, 0.25)
    x, y = parity.to_dev(wl.x[0]), parity.to_dev(wl.y[0])
    s0 = torch.full((1,), 0.5, dtype=x.dtype, device=x.device)
    s1 = torch.full((1,), 0.25, dtype=x.dtype, device=x.device)
    for rb, re in [(0, 1200), (1200, 3000), (700, 2900)]:
        ws = api.spike_workspace(3000, rb, re, x.dtype, x.device)
        rec = torch.empty(6, dtype=x.dtype, device=x.device)
        api.spike_reduce(x, y, rb, re, 3, s0, s1, rec, ws)
        ref = torch.empty(6, dtype=torch.float64)
        ops.reduce(None, None, rb, re, 3, None, None, ref, None)
        g, r = rec.cpu().numpy(), ref.numpy()
        scale = np.array([abs(r[0]) + abs(r[3])] * 6)
        scale[[1, 2, 4, 5]] = 1.0
        assert np.all(np.abs(g - r) <= 1e-12 * scale), (g, r)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_gather_probe_matches_eval(api, dt):
    """The gather-ceiling probe evaluates at known intervals: with spline_eval's
    idx it reproduces spline_eval's out bitwise through both access patterns."""
    wl = workloads.generate(5, n=(1 << 17) + 5, m=50000)
    x = parity.to_dev(wl.x.astype(dt))
    y = parity.to_dev(wl.y.astype(dt))
    q = parity.to_dev(wl.q.astype(dt))
    q[0, :3] = float("nan")
    y2 = api.build(x, y, 0)
    out, idx = api.evaluate(x, y, y2, q, 0)
    for mode in (0, 1):
        o, i = api.gather_probe(x, y, y2, q, idx, mode)
        assert torch.equal(i, idx)
        assert torch.equal(o.view(torch.int8), out.view(torch.int8))
    api.status()


def test_tile_solve_batch_beyond_grid_y(api):
    """K2 (one CTA per curve) with more than 65535 curves: the 1-D launch covers any batch."""
    rng = np.random.default_rng(99)
    B, n = 70000, 200
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.05, axis=1).astype(np.float32)
    y = np.cumsum(rng.normal(size=(B, n)), axis=1).astype(np.float32)
    spec = workloads.ConfigSpec(0, "t", B, n, 4, "f32", 0, 0, 0)
    wl = workloads.Workload(spec, x, y, x[:, :4].copy(), None, None, 0, 0)
    parity.check_case(api, wl, y2_only=True)


def _sorted_case(rng, dt, B, n, m, kind):
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.01, axis=1).astype(dt)
    y = rng.normal(size=(B, n)).astype(dt)
    y2 = rng.normal(size=(B, n)).astype(dt)
    if kind == "clustered":  # 90% of the queries in 1% of the range; the sparse rest gives
        lo, hi = x[:, :1], x[:, -1:]  # tiles whose window overflows shared memory
        q = np.concatenate([rng.uniform(lo, hi, (B, m // 10)),
                            rng.uniform(lo, lo + 0.01 * (hi - lo), (B, m - m // 10))], axis=1)
    else:
        q = rng.uniform(x[:, :1], x[:, -1:], (B, m))
    q = q.astype(dt)
    k = min(m // 8, n)
    q[:, :k] = x[:, rng.integers(0, n, k)][0]  # exact knot hits
    q[:, k], q[:, k + 1], q[:, k + 2], q[:, k + 3] = x[:, 0], x[:, -1], x[:, 0] - 1, x[:, -1] + 1
    if kind == "nan":
        q[:, k + 4] = np.nan
    if kind != "unsorted":
        q = np.sort(q, axis=1)  # NaN sorts to the end
    if kind == "nearly":  # sorted but for 1% of adjacent pairs swapped: a hint that is mostly right
        sw = rng.choice(m - 1, m // 100, replace=False)
        q[:, sw], q[:, sw + 1] = q[:, sw + 1].copy(), q[:, sw].copy()
    return x, y, y2, q


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("B,n,m,kind", [(3, 4096, 65536, "dense"), (2, 129, 8 * 1024 + 8, "nan"),
                                        (5, 3, 64, "dense"), (2, 2000, 40000, "clustered"), (3, 100, 3000, "dense"),
                                        (2, 500, 8192, "unsorted"), (1, 257, 4100, "dense"),
                                        (3, 1000, 40000, "nearly")])
def test_sorted_edge_cases(api, dt, B, n, m, kind):
    """SPLINE_Q_SORTED (k_eval_sorted): ties, both ends, out of range, NaN, ragged runs, dense
    and clustered query densities, a wrong hint and a mostly-right one (adjacent pairs swapped:
    the fast path's slot verification) all match the oracle, idx bit-exact; out is
    bitwise the unsorted path's (same make_cub / cub_eval arithmetic)."""
    rng = np.random.default_rng(n * 7 + m)
    x, y, y2, q = _sorted_case(rng, dt, B, n, m, kind)
    out_ref, idx_ref, nbad = oracle.evaluate(x, y, y2, q)
    t = parity.to_dev
    api.status()
    out, idx = api.evaluate(t(x), t(y), t(y2), t(q), 1)
    bits = api.status()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    e = parity.out_rel_err(out.cpu().numpy(), out_ref, y)
    assert np.all(e <= parity.tol_for(dt))
    assert (bits & api.STATUS_Q_OUT_OF_RANGE) == (api.STATUS_Q_OUT_OF_RANGE if nbad else 0)
    out_u, idx_u = api.evaluate(t(x), t(y), t(y2), t(q), 0)
    assert (api.status() & api.STATUS_Q_OUT_OF_RANGE) == (api.STATUS_Q_OUT_OF_RANGE if nbad else 0)
    assert torch.equal(idx, idx_u)
    assert torch.equal(torch.nan_to_num(out, 7.0).view(torch.int8), torch.nan_to_num(out_u, 7.0).view(torch.int8))


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("cid,kw", [(2, dict(batch=5000)), (2, dict(batch=700, m=252)), (4, dict(batch=7, n=300, m=1000)),
                                    (3, dict(batch=3000)), (5, dict(n=(1 << 15) + 3, m=4096))])
def test_build_eval_host_equals_device(api, cid, kw, pinned):
    """spline_build_eval_host (host arrays, chunked through internal streams) gives bitwise the
    device call's y2, out, idx -- several chunks, ragged last chunk, pageable or pinned memory."""
    wl = workloads.generate(cid, **kw)
    t = parity.to_dev
    h = lambda a: torch.from_numpy(a).pin_memory() if pinned else torch.from_numpy(a).clone()
    s1 = wl.yp1 if wl.bc & 1 else None
    s2 = wl.ypn if wl.bc & 2 else None
    dv = lambda a: t(a) if a is not None else None
    hv = lambda a: h(a) if a is not None else None
    api.status()
    y2d, od, idd = api.build_eval(t(wl.x), t(wl.y), t(wl.q), wl.bc, dv(s1), dv(s2), wl.flags)
    bits_d = api.status()
    y2h, oh, idh = api.build_eval_host(h(wl.x), h(wl.y), h(wl.q), wl.bc, hv(s1), hv(s2), wl.flags)
    bits_h = api.status()
    assert bits_h == bits_d
    assert torch.equal(y2h.view(torch.int8), y2d.cpu().view(torch.int8))
    assert torch.equal(idh, idd.cpu())
    assert torch.equal(oh.view(torch.int8), od.cpu().view(torch.int8))


@pytest.mark.slow
def test_build_eval_host_one_long_curve(api):
    """One curve with enough queries that spline_build_eval_host streams them in chunks after the
    build (the one-curve pipeline): bitwise the device call."""
    wl = workloads.generate(5, n=100003, m=14_000_000)
    t = parity.to_dev
    h = lambda a: torch.from_numpy(a).pin_memory()
    api.status()
    y2d, od, idd = api.build_eval(t(wl.x), t(wl.y), t(wl.q), wl.bc, None, None, wl.flags)
    y2h, oh, idh = api.build_eval_host(h(wl.x), h(wl.y), h(wl.q), wl.bc, None, None, wl.flags)
    assert api.status() == 0
    assert torch.equal(y2h.view(torch.int8), y2d.cpu().view(torch.int8))
    assert torch.equal(idh, idd.cpu())
    assert torch.equal(oh.view(torch.int8), od.cpu().view(torch.int8))


@pytest.mark.parametrize("kw", [dict(batch=20000), dict(batch=1001, n=5, m=12), dict(batch=77, n=8, m=32)])
@pytest.mark.parametrize("bc", [0, 3])
def test_build_eval_default_equals_build_then_eval(api, kw, bc):
    """spline_build_eval without a path hint (short fp32 curves: the solve+eval small kernel) gives
    bitwise spline_build followed by spline_eval, and the oracle's answer."""
    wl = workloads.generate(3, **kw)
    t = parity.to_dev
    B = wl.x.shape[0]
    rng = np.random.default_rng(B)
    s1 = t(rng.normal(size=B).astype(np.float32)) if bc & 1 else None
    s2 = t(rng.normal(size=B).astype(np.float32)) if bc & 2 else None
    x, y, q = t(wl.x), t(wl.y), t(wl.q)
    api.status()
    y2a, oa, ia = api.build_eval(x, y, q, bc, s1, s2, wl.flags)
    y2b = api.build(x, y, bc, s1, s2)
    ob, ib = api.evaluate(x, y, y2b, q, wl.flags)
    assert api.status() == 0
    assert torch.equal(y2a.view(torch.int8), y2b.view(torch.int8))
    assert torch.equal(ia, ib)
    assert torch.equal(oa.view(torch.int8), ob.view(torch.int8))


def test_build_eval_host_edge_cases(api):
    """Host entry: m = 0 builds only; no y2 / no idx outputs; a single curve with few queries."""
    wl = workloads.generate(2, batch=50, m=8)
    t = parity.to_dev
    x, y, q = torch.from_numpy(wl.x), torch.from_numpy(wl.y), torch.from_numpy(wl.q)
    s1, s2 = torch.from_numpy(wl.yp1), torch.from_numpy(wl.ypn)
    y2d = api.build(t(wl.x), t(wl.y), wl.bc, t(wl.yp1), t(wl.ypn)).cpu()
    e = q[:, :0].contiguous()
    y2h, oh, ih = api.build_eval_host(x, y, e, wl.bc, s1, s2)
    assert torch.equal(y2h.view(torch.int8), y2d.view(torch.int8)) and oh.shape == (50, 0)
    _, od, _ = api.build_eval(t(wl.x), t(wl.y), t(wl.q), wl.bc, t(wl.yp1), t(wl.ypn), want_y2=False, want_idx=False)
    z, oh, ih = api.build_eval_host(x, y, q, wl.bc, s1, s2, want_y2=False, want_idx=False)
    assert z is None and ih is None and torch.equal(oh.view(torch.int8), od.cpu().view(torch.int8))
    y2h, oh, ih = api.build_eval_host(x[0], y[0], q[0], wl.bc, s1[:1], s2[:1])
    assert oh.shape == (8,) and ih.shape == (8,)
    assert api.status() == 0


@pytest.mark.parametrize("cid,kw", [(1, dict()), (1, dict(batch=3)), (2, dict(batch=5, m=1000)),
                                    (2, dict(batch=16, n=32, m=64)), (2, dict(batch=1, n=16, m=8192))])
def test_build_eval_tiny_equals_build_then_eval(api, cid, kw):
    """spline_build_eval without a hint on a few K1h-sized curves (the one-CTA-per-curve kernel):
    bitwise spline_build then spline_eval, including out-of-range and NaN queries."""
    wl = workloads.generate(cid, **kw)
    q = wl.q.copy()
    q[:, 0], q[:, 1] = wl.x[:, 0] - 1, np.nan
    t = parity.to_dev
    s1 = t(wl.yp1) if wl.bc & 1 else None
    s2 = t(wl.ypn) if wl.bc & 2 else None
    x, y, qd = t(wl.x), t(wl.y), t(q)
    api.status()
    y2a, oa, ia = api.build_eval(x, y, qd, wl.bc, s1, s2, wl.flags)
    y2b = api.build(x, y, wl.bc, s1, s2)
    ob, ib = api.evaluate(x, y, y2b, qd, wl.flags)
    assert api.status() == api.STATUS_Q_OUT_OF_RANGE
    assert torch.equal(y2a.view(torch.int8), y2b.view(torch.int8))
    assert torch.equal(ia, ib)
    assert torch.equal(torch.nan_to_num(oa, 7.0).view(torch.int8), torch.nan_to_num(ob, 7.0).view(torch.int8))
    out_ref, idx_ref, _ = oracle.evaluate(wl.x, wl.y, y2b.cpu().numpy(), q)
    np.testing.assert_array_equal(ia.cpu().numpy(), idx_ref)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("B,n,m", [(1000, 40, 64), (700, 3, 8), (650, 64, 2), (900, 17, 130)])
def test_curvewarp_shapes(api, dt, B, n, m):
    """k_eval_curvewarp (n <= 64, >= 4 curves per SM) across n (Eytzinger depth 2..6), ragged
    query counts per lane and both dtypes, with ties, ends, out-of-range and NaN queries."""
    rng = np.random.default_rng(B + n + m)
    x = np.cumsum(rng.exponential(1.0, (B, n)) + 0.01, axis=1).astype(dt)
    y = rng.normal(size=(B, n)).astype(dt)
    y2 = rng.normal(size=(B, n)).astype(dt)
    q = rng.uniform(x[:, :1] - 0.5, x[:, -1:] + 0.5, (B, m)).astype(dt)
    q[:, 0] = x[:, min(1, n - 1)]
    if m > 1:
        q[:, 1] = np.nan
    out_ref, idx_ref, nbad = oracle.evaluate(x, y, y2, q)
    api.status()
    out, idx = api.evaluate(parity.to_dev(x), parity.to_dev(y), parity.to_dev(y2), parity.to_dev(q), 0)
    bits = api.status()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    e = parity.out_rel_err(out.cpu().numpy(), out_ref, y)
    assert np.all(e <= parity.tol_for(dt))
    assert (bits & api.STATUS_Q_OUT_OF_RANGE) == (api.STATUS_Q_OUT_OF_RANGE if nbad else 0)


# ------------------------------------------- one long curve: queries bucketed by L2-sized chunks

@pytest.mark.parametrize("n,m", [((1 << 23) + 77, 1 << 22), (1 << 24, (1 << 21) + 13)])
def test_long_curve_bucketed_eval(api, n, m):
    """Curves far larger than L2 with many unsorted queries take the bucketed eval
    (k_bucket_scatter -> k_bucket_eval -> k_bucket_gather): the oracle's idx bit for bit and out
    within tolerance, including knot ties at chunk boundaries, both ends, out of range and NaN --
    and bitwise the record-gather path (SPLINE_NO_BUCKET)."""
    wl = workloads.generate(5, n=n, m=m)
    K = (24 << 20) // 32                                   # chunk width of the fp64 path (24 MB of 32 B knots)
    ties = [wl.x[0, k] for k in range(0, n - 1, K)] + [wl.x[0, K - 1], wl.x[0, K + 1], wl.x[0, 2 * K - 1]]
    wl.q[0, :len(ties)] = ties                             # queries ON chunk-boundary knots
    wl.q[0, 100] = wl.x[0, -1]
    wl.q[0, 101] = wl.x[0, 0]
    wl.q[0, 102] = -0.5
    wl.q[0, 103] = 2.0
    wl.q[0, 104] = np.nan
    wl.q[0, 105] = np.nextafter(wl.x[0, -1], 2.0)
    api.status()
    x, y, y2 = parity.gpu_build(api, wl)
    y2_ref = parity.oracle_build(wl)
    assert parity.y2_rel_err(y2.cpu().numpy(), y2_ref).max() <= 1e-12
    q = parity.to_dev(wl.q)
    out_ref, idx_ref, nbad = oracle.evaluate(wl.x, wl.y, y2_ref, wl.q, nthreads=16)
    assert nbad == 4
    out, idx = api.evaluate(x, y, parity.to_dev(y2_ref), q, 0)
    assert api.status() == api.STATUS_Q_OUT_OF_RANGE
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    assert parity.out_rel_err(out.cpu().numpy(), out_ref, wl.y).max() <= 1e-12
    out_r, idx_r = api.evaluate(x, y, parity.to_dev(y2_ref), q, api.NO_BUCKET)
    api.status()
    assert torch.equal(idx, idx_r) and torch.equal(out.view(torch.int8), out_r.view(torch.int8))
    _, none = api.evaluate(x, y, parity.to_dev(y2_ref), q, 0, want_idx=False)  # no idx output
    assert none is None
    api.status()


@pytest.mark.parametrize("grid", ["jitter40", "exp"])
def test_long_curve_bucketed_eval_nonuniform(api, grid):
    """The bucketed eval on long curves whose knots stray far from the interval guess: a grid
    jittered by +-40% of a cell (the packing's deviation band covers ~80% of the queries) and
    exponential gaps (the guess misses by thousands of intervals: the general correction) -- idx
    bit for bit against the oracle, out within tolerance, bitwise the record-gather path."""
    rng = np.random.default_rng(11 if grid == "exp" else 12)
    n, m = (1 << 23) + 5, (1 << 21) + 3
    if grid == "exp":
        x = np.cumsum(rng.exponential(1.0, n))
    else:
        x = np.arange(n, dtype=np.float64) + rng.uniform(-0.4, 0.4, n)
    x = (x - x[0]) / (x[-1] - x[0])
    y = np.cumsum(rng.normal(0.0, 1.0 / np.sqrt(n), n))
    y2 = rng.normal(0.0, 1.0, n)
    q = rng.uniform(-0.01, 1.01, m)
    q[:4] = x[0], x[-1], x[n // 2], np.nan
    x, y, y2, q = x[None], y[None], y2[None], q[None]
    out_ref, idx_ref, nbad = oracle.evaluate(x, y, y2, q, nthreads=16)
    t = parity.to_dev
    api.status()
    out, idx = api.evaluate(t(x), t(y), t(y2), t(q), 0)
    assert api.status() == api.STATUS_Q_OUT_OF_RANGE and nbad > 0
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_ref)
    assert parity.out_rel_err(out.cpu().numpy(), out_ref, y).max() <= 1e-12
    out_r, idx_r = api.evaluate(t(x), t(y), t(y2), t(q), api.NO_BUCKET)
    api.status()
    assert torch.equal(idx, idx_r) and torch.equal(out.view(torch.int8), out_r.view(torch.int8))


@pytest.mark.parametrize("world,n,bc", [(2, 300001, 0), (8, (1 << 20) + 5, 3), (3, 4096 * 7, 1)])
def test_recompute_build_emulated_ranks(api, world, n, bc):
    """§8(e)(ii) recompute-instead-of-gather, G ranks emulated on one GPU: each rank's tile records
    (whole tiles), concatenated, then the full finish -> bitwise spline_build's y2 (the same tiles,
    the same merges) and the oracle's within tolerance."""
    from paper_2001_09253_b200 import dist as sdist
    api.status()
    wl = workloads.generate(5, n=n, m=16)
    x, y = parity.to_dev(wl.x[0]), parity.to_dev(wl.y[0])
    s0 = torch.full((1,), 0.3, dtype=x.dtype, device=x.device)
    s1 = torch.full((1,), -0.2, dtype=x.dtype, device=x.device)
    ts = api.spike_tile_rows(x.dtype)
    ntiles = -(-n // ts)
    ws = api.spike_workspace(n, 0, n, x.dtype, x.device)
    recs = torch.empty(ntiles, 6, dtype=x.dtype, device=x.device)
    for r in range(world):
        t0, t1, rb, re = sdist.shard_tiles(n, ts, world, r)
        if t1 > t0:
            api.spike_tile_records(x, y, rb, re, bc, s0, s1, recs[t0:t1], ws)
    y2 = torch.empty(n, dtype=x.dtype, device=x.device)
    api.spike_finish_tiles(x, y, bc, s0, s1, recs, y2, ws)
    ref_gpu = api.build(x[None], y[None], bc, 0.3, -0.2)[0]
    assert api.status() == 0
    assert torch.equal(y2.view(torch.int8), ref_gpu.view(torch.int8))
    ref, _ = oracle.build_y2(wl.x[0], wl.y[0], bc, [0.3], [-0.2])
    assert parity.y2_rel_err(y2.cpu().numpy()[None], ref[None]).max() <= 1e-12
