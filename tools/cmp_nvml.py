"""Does NVML clock polling (bench.py's ClockSampler) perturb a µs-sized timed step?
python tools/cmp_nvml.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2001_09253_b200 import api, workloads

wl = workloads.generate(1)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x, y, q = t(wl.x), t(wl.y), t(wl.q)
y2 = torch.empty_like(x); out = torch.empty_like(q); idx = torch.empty(q.shape, dtype=torch.int32, device='cuda')
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
f = lambda: api.build_eval(x, y, q, wl.bc, None, None, wl.flags, y2=y2, out=out, idx=idx)
for _ in range(200):
    f()
torch.cuda.synchronize()


def run(sampler):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    for a, b in ev:
        flush.zero_()
        a.record(); f(); b.record()
    torch.cuda.synchronize()
    if ctx:
        ctx.__exit__()
    return statistics.mean(a.elapsed_time(b) for a, b in ev) * 1e3


for rep in range(3):
    print("no sampler %.1f us   sampler %.1f us" % (run(False), run(True)))
