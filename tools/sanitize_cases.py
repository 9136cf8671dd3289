"""Small cases through every kernel with shared-memory hand-offs or trees, for compute-sanitizer
(one tool per run):  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
Each case is also checked against the split path / its own consistency so a silent race would
show up as a mismatch too."""
import os
import sys

os.environ.setdefault("FASTSPLINE_BUCKET_MIN_N", "150000")  # the bucketed eval on a small curve
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, dist as sdist, workloads

t = lambda a: torch.from_numpy(a).cuda() if a is not None else None


def run(name, cid, flags_extra=0, **kw):
    wl = workloads.generate(cid, **kw)
    x, y, q, yp1, ypn = t(wl.x), t(wl.y), t(wl.q), t(wl.yp1), t(wl.ypn)
    a = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | flags_extra)
    b = api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_SPLIT)
    torch.cuda.synchronize()
    same = all(torch.equal(u.view(torch.int8), v.view(torch.int8)) for u, v in zip(a, b))
    print(f"{name:40s} {'ok' if same else 'MISMATCH'}", flush=True)
    assert same


run("k_build_eval_tiny (cfg1)", 1)
run("K1h + k_eval_curvewarp (cfg2)", 2, batch=600)
run("k_fused_staged warp-owned (cfg2)", 2, api.PATH_FUSED, batch=64)
run("k_fused_staged chunked (one curve)", 2, api.PATH_FUSED, batch=1, m=10000)
run("k_eval_small<true> (cfg3)", 3, batch=1000)
run("k_fused_staged SOLVE_REGS (cfg3)", 3, api.PATH_FUSED, batch=300)
run("K1 pipe + k_eval_warps (n=100)", 2, batch=64, n=100, m=300)
run("k_eval_staged TABLE (n=1000)", 4, batch=2, n=1000, m=5000, flags_extra=0)
run("k_tile<FULL> + k_eval_sorted (cfg4)", 4, batch=3, n=1000, m=8000)
run("k_tile_eval (cfg4, PATH_FUSED)", 4, api.PATH_FUSED, batch=3, n=1000, m=8000)
run("K3/K4/K5 + records eval", 5, n=100000, m=5000)
run("K3/K4/K5 + bucketed eval", 5, n=200000, m=1 << 18)
# the multi-GPU seam, 3 ranks emulated
wl = workloads.generate(5, n=60000, m=16)
x, y = t(wl.x[0]), t(wl.y[0])
recs, wss, parts = [], [], []
for r in range(3):
    rb, re = sdist.shard_rows(60000, 3, r)
    ws = api.spike_workspace(60000, rb, re, x.dtype, x.device)
    rec = torch.empty(6, dtype=x.dtype, device=x.device)
    api.spike_reduce(x, y, rb, re, 0, None, None, rec, ws)
    recs.append(rec)
    wss.append(ws)
allr = torch.cat(recs)
for r in range(3):
    rb, re = sdist.shard_rows(60000, 3, r)
    y2s = torch.empty(re - rb, dtype=x.dtype, device=x.device)
    api.spike_finish(x, y, rb, re, 0, None, None, allr, 3, r, y2s, wss[r])
    parts.append(y2s)
ref = api.build(x[None], y[None])[0]
torch.cuda.synchronize()
print(f"{'k4_top seam (3 emulated ranks)':40s} {'ok' if torch.allclose(torch.cat(parts), ref, rtol=1e-12) else 'MISMATCH'}")
h = [torch.from_numpy(a).pin_memory() for a in (workloads.generate(2, batch=2000).x,)]
print("status", api.status())
