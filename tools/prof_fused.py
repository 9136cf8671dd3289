"""Run spline_build_eval of one config a few times (for ncu captures).  python tools/prof_fused.py CFG [ITERS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, workloads

cid = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.generate(cid)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x, y, q, yp1, ypn = t(wl.x), t(wl.y), t(wl.q), t(wl.yp1), t(wl.ypn)
y2 = torch.empty_like(x)
out = torch.empty_like(q)
idx = torch.empty(q.shape, dtype=torch.int32, device="cuda")
for _ in range(iters):
    api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_FUSED, y2=y2, out=out, idx=idx)
torch.cuda.synchronize()
assert api.status() == 0
print("ok", cid)
