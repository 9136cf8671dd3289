"""spline_build_eval with PATH_FUSED vs PATH_SPLIT vs no hint, queued steps, for a scaled config.
python tools/cmp_paths.py CFG BATCH"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, workloads

cid, B = int(sys.argv[1]), int(sys.argv[2])
wl = workloads.generate(cid, batch=B)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x, y, q, yp1, ypn = t(wl.x), t(wl.y), t(wl.q), t(wl.yp1), t(wl.ypn)
y2 = torch.empty_like(x); out = torch.empty_like(q); idx = torch.empty(q.shape, dtype=torch.int32, device='cuda')
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')


def run(fl, K=30):
    f = lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | fl, y2=y2, out=out, idx=idx)
    for _ in range(10):
        f()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in ev:
        flush.zero_()
        a.record(); f(); b.record()
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ev) * 1e3


for rep in range(2):
    print("cfg%d batch %d m %d: fused %.1f us  split %.1f us  auto %.1f us" % (
        cid, B, wl.m, run(api.PATH_FUSED), run(api.PATH_SPLIT), run(0)))
