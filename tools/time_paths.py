"""Quick CUDA-event timing of the build/eval paths of one config (not the bench contract).
python tools/time_paths.py CFG [ITERS]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import api, workloads

cid = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = workloads.generate(cid)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x, y, q, yp1, ypn = t(wl.x), t(wl.y), t(wl.q), t(wl.yp1), t(wl.ypn)
y2 = torch.empty_like(x)
out = torch.empty_like(q)
idx = torch.empty(q.shape, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.zeros(128 << 20, dtype=torch.float32, device="cuda")
MODE = os.environ.get("FLUSH", "wr")
s = 4 if wl.x.dtype.itemsize == 4 else 8
B, n, m = wl.batch, wl.n, wl.m


def timeit(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        if MODE in ("w", "wr"):
            flush.zero_()
        if MODE in ("wr", "r"):
            flush_r.sum()  # clean the L2: read 256 MiB so no dirty flush lines drain inside the timed region
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


paths = {
    "build": (lambda: api.build(x, y, wl.bc, yp1, ypn, out=y2), 3 * s * B * n),
    "eval": (lambda: api.evaluate(x, y, y2, q, wl.flags, out=out, idx=idx), (2 * s + 4) * B * m + 3 * s * B * n),
    "build+eval": (lambda: (api.build(x, y, wl.bc, yp1, ypn, out=y2),
                            api.evaluate(x, y, y2, q, wl.flags, out=out, idx=idx)),
                   (2 * s + 4) * B * m + 3 * s * B * n + 3 * s * B * n),
    "step (auto)": (lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, y2=y2, out=out, idx=idx),
                    (2 * s + 4) * B * m + 3 * s * B * n + 3 * s * B * n),
    "step (no y2)": (lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, want_y2=False, out=out, idx=idx),
                     (2 * s + 4) * B * m + 3 * s * B * n + 3 * s * B * n),
    "split": (lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_SPLIT, y2=y2, out=out, idx=idx),
              (2 * s + 4) * B * m + 3 * s * B * n + 3 * s * B * n),
    "fused(y2)": (lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_FUSED, y2=y2, out=out, idx=idx),
                  (2 * s + 4) * B * m + 3 * s * B * n),
    "fused(no y2)": (lambda: api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags | api.PATH_FUSED, want_y2=False, out=out, idx=idx),
                     (2 * s + 4) * B * m + 2 * s * B * n),
}
assert api.status() == 0
only = os.environ.get("ONLY")  # comma-separated path names
for name, (fn, nbytes) in paths.items():
    if only and name not in only.split(","):
        continue
    ms = timeit(fn)
    print(f"cfg{cid} {name:14s} {ms * 1e3:9.1f} us  {nbytes / ms / 1e6:8.1f} GB/s  {B * m / ms / 1e6:9.2f} Gq/s")
assert api.status() == 0
