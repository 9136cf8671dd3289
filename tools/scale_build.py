"""Build-kernel scaling probe: time spline_build on cfg-shaped inputs at several batch sizes.
python tools/scale_build.py CFG"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_09253_b200 import api, workloads

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
base = workloads.CONFIGS[cid].batch
for mult in (0.25, 1, 4, 16):
    B = int(base * mult)
    wl = workloads.generate(cid, batch=B, m=4)
    t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
    x, y, yp1, ypn = t(wl.x), t(wl.y), t(wl.yp1), t(wl.ypn)
    y2 = torch.empty_like(x)
    for _ in range(3):
        api.build(x, y, wl.bc, yp1, ypn, out=y2)
    ts = []
    for _ in range(15):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        api.build(x, y, wl.bc, yp1, ypn, out=y2)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    nb = 3 * x.element_size() * x.numel()
    print(f"cfg{cid} batch {B:8d}: {ms * 1e3:8.1f} us  {nb / ms / 1e6:8.1f} GB/s")
