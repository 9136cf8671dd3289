"""Host-side checks of the seeded generators (-m "not gpu")."""
import numpy as np
import pytest

from paper_2001_09253_b200 import workloads


@pytest.mark.parametrize("cid,kw", [(1, {}), (2, dict(batch=512)), (3, dict(batch=2048)),
                                    (4, dict(batch=8, n=512, m=4096)), (5, dict(n=1 << 14, m=1 << 16))])
def test_generated_inputs_valid(cid, kw):
    wl = workloads.generate(cid, **kw)
    assert wl.x.dtype == wl.np_dtype and wl.q.dtype == wl.np_dtype
    assert np.all(np.diff(wl.x, axis=1) > 0), "knots must strictly increase (c11)"
    assert np.all(np.isfinite(wl.y))
    assert np.all(wl.q >= wl.x[:, :1]) and np.all(wl.q <= wl.x[:, -1:])
    if wl.flags & workloads.FLAG_Q_SORTED:
        assert np.all(np.diff(wl.q, axis=1) >= 0)
    if wl.bc:
        assert wl.yp1.shape == (wl.batch,) and np.all(np.isfinite(wl.yp1))
    b = workloads.generate(cid, **kw)
    np.testing.assert_array_equal(wl.q, b.q)   # seeded, deterministic
    c = workloads.generate(cid, shard=1, **kw)
    assert not np.array_equal(wl.y, c.y)       # shards differ


def test_cfg_shapes_match_baseline():
    s = workloads.CONFIGS
    assert (s[1].batch, s[1].n, s[1].m, s[1].dtype) == (1, 16, 1000, "f64")
    assert (s[2].batch, s[2].n, s[2].m, s[2].dtype) == (65536, 64, 256, "f32")
    assert (s[3].batch, s[3].n, s[3].m, s[3].dtype) == (1 << 20, 8, 32, "f32")
    assert (s[4].batch, s[4].n, s[4].m, s[4].dtype) == (4096, 4096, 16 * 4096, "f64")
    assert (s[5].batch, s[5].n, s[5].m, s[5].dtype) == (1, 1 << 26, 1 << 28, "f64")


def test_cfg1_ends_pinned():
    wl = workloads.generate(1)
    assert wl.x[0, 0] == 0.0 and wl.x[0, -1] == 1.0
