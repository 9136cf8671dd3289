"""Step time with steps queued back to back (bench.py's protocol) vs one step at a time.
python tools/cmp_queue.py CFG"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, workloads

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workloads.generate(cid)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x, y, q, yp1, ypn = t(wl.x), t(wl.y), t(wl.q), t(wl.yp1), t(wl.ypn)
y2 = torch.empty_like(x); out = torch.empty_like(q); idx = torch.empty(q.shape, dtype=torch.int32, device='cuda')
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
f = lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, y2=y2, out=out, idx=idx)
for _ in range(50):
    f()
torch.cuda.synchronize()


def queued(K=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in ev:
        flush.zero_()
        a.record(); f(); b.record()
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ev) * 1e3


def single(K=20):
    ts = []
    for _ in range(K):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(); f(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.mean(ts) * 1e3


for rep in range(3):
    print("cfg%d queued %.1f us   one-at-a-time %.1f us" % (cid, queued(), single()))
