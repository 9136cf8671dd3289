"""PCIe ceiling of the box for the host path (spline_build_eval_host): pinned H2D, D2H, and both
directions at once (2 streams), 1 GiB each.   python tools/pcie_probe.py"""
import json

import torch

N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
bi = timed(both)
print(json.dumps({"probe": "pcie_pinned", "bytes": N, "h2d_GBps": N / h2d / 1e9, "d2h_GBps": N / d2h / 1e9,
                  "bidirectional_GBps_each": N / bi / 1e9, "bidirectional_GBps_total": 2 * N / bi / 1e9}))
