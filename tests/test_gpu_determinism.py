"""Race stress (compute-sanitizer is closed on this pool -- profiles/r02/compute_sanitizer_closed.log):
the kernels with shared-memory hand-offs (mbarrier phases, named barriers, last-warp refills,
merge trees) run many times while another stream keeps the SMs busy with unrelated work, so the
CTA schedule differs from run to run; every run must give the same bits.  A race on a stage, a
window or a tree level shows up as a run that differs."""
import pytest
import torch

import parity
from paper_2001_09253_b200 import workloads

pytestmark = pytest.mark.gpu

CASES = [("k_fused_staged warp-owned", 2, dict(batch=2000), 4), ("k_fused_staged chunked", 2, dict(batch=1, m=60000), 4),
         ("k_fused_staged SOLVE_REGS", 3, dict(batch=5000), 4), ("k_eval_warps + K1 pipe", 2, dict(batch=3000, n=100, m=300), 0),
         ("k_eval_staged TABLE", 4, dict(batch=4, n=1500, m=20000, ), 0), ("k_tile_eval", 4, dict(batch=40, n=3000, m=30000), 4),
         ("k_tile + k_eval_sorted", 4, dict(batch=40, n=3000, m=30000), 0), ("K3-K5 + records", 5, dict(n=300000, m=100000), 0),
         ("k_build_eval_tiny", 1, dict(batch=9), 0), ("k_eval_small<true>", 3, dict(batch=50000), 0),
         ("K1h + k_eval_curvewarp", 2, dict(batch=5000), 0)]


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_09253_b200 import api as a
    a.status()
    return a


@pytest.mark.parametrize("name,cid,kw,fl", CASES, ids=[c[0] for c in CASES])
def test_repeated_runs_identical_under_load(api, name, cid, kw, fl):
    wl = workloads.generate(cid, **kw)
    t = parity.to_dev
    x, y, q = t(wl.x), t(wl.y), t(wl.q)
    yp1 = t(wl.yp1) if wl.yp1 is not None else None
    ypn = t(wl.ypn) if wl.ypn is not None else None
    flags = wl.flags | (api.PATH_FUSED if fl else 0)
    ref = [r.clone() for r in api.build_eval(x, y, q, wl.bc, yp1, ypn, flags)]
    noise = torch.cuda.Stream()
    big = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for it in range(12):
        with torch.cuda.stream(noise):
            for _ in range(it % 4):
                big.mul_(1.0000001)  # SM pressure on another stream, a different amount each run
        got = api.build_eval(x, y, q, wl.bc, yp1, ypn, flags)
        torch.cuda.synchronize()
        for a, b in zip(ref, got):
            assert torch.equal(a.view(torch.int8), b.view(torch.int8)), f"{name}: run {it} differs"
    assert api.status() == 0
