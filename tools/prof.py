"""The kernels of one config's timed paths, once each (for ncu captures):
  the bench step (spline_build_eval, the library's own path choice), then the split path's build
  and eval kernels (bench.py's per-kernel rooflines).   python tools/prof.py CFG [ITERS] [--x-shared]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, workloads

cid = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 1
wl = workloads.generate(cid)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x = t(wl.x[0]) if "--x-shared" in sys.argv else t(wl.x)
y, q, yp1, ypn = t(wl.y), t(wl.q), t(wl.yp1), t(wl.ypn)
y2 = torch.empty_like(y)
out = torch.empty_like(q)
idx = torch.empty(q.shape, dtype=torch.int32, device="cuda")
for _ in range(iters):
    torch.cuda.nvtx.range_push(f"cfg{cid}:step")
    api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, y2=y2, out=out, idx=idx)
    torch.cuda.nvtx.range_pop()
    torch.cuda.nvtx.range_push(f"cfg{cid}:build")
    api.build(x, y, wl.bc, yp1, ypn, out=y2)
    torch.cuda.nvtx.range_pop()
    torch.cuda.nvtx.range_push(f"cfg{cid}:eval")
    api.evaluate(x, y, y2, q, wl.flags, out=out, idx=idx)
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
assert api.status() == 0
print("ok", cid)
