"""End-to-end (host arrays) step: copies then kernels on one stream vs spline_build_eval_host.
python tools/cmp_e2e.py CFG"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, workloads

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workloads.generate(cid)
pin = lambda a: torch.from_numpy(a).pin_memory() if a is not None else None
hx, hy, hq = pin(wl.x), pin(wl.y), pin(wl.q)
s1 = pin(wl.yp1) if wl.bc & 1 else None
s2 = pin(wl.ypn) if wl.bc & 2 else None
hy2 = torch.empty(hx.shape, dtype=hx.dtype).pin_memory()
ho = torch.empty(hq.shape, dtype=hq.dtype).pin_memory()
hi = torch.empty(hq.shape, dtype=torch.int32).pin_memory()
dx, dy, dq = hx.cuda(), hy.cuda(), hq.cuda()
d1 = s1.cuda() if s1 is not None else None
d2 = s2.cuda() if s2 is not None else None
y2, out, idx = torch.empty_like(dx), torch.empty_like(dq), torch.empty(dq.shape, dtype=torch.int32, device="cuda")


def seq():
    dx.copy_(hx, non_blocking=True); dy.copy_(hy, non_blocking=True); dq.copy_(hq, non_blocking=True)
    if d1 is not None: d1.copy_(s1, non_blocking=True)
    if d2 is not None: d2.copy_(s2, non_blocking=True)
    api.build_eval(dx, dy, dq, wl.bc, d1, d2, wl.flags, y2=y2, out=out, idx=idx)
    hy2.copy_(y2, non_blocking=True); ho.copy_(out, non_blocking=True); hi.copy_(idx, non_blocking=True)


def host():
    api.build_eval_host(hx, hy, hq, wl.bc, s1, s2, wl.flags, y2=hy2, out=ho, idx=hi, sync=False)


def timeit(f, K=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


for rep in range(3):
    print("cfg%d copies+kernels %.3f ms   build_eval_host %.3f ms" % (cid, timeit(seq), timeit(host)))
