"""Per-phase SM cycles of tile_solve (needs a -DFS_TILE_PHASES=1 build of the library).
python tools/tile_phases.py CFG [ITERS [BATCH]]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_09253_b200 import _lib, api, workloads

cid = int(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kw = {"batch": int(sys.argv[3])} if len(sys.argv) > 3 else {}
wl = workloads.generate(cid, **kw)
t = lambda a: torch.from_numpy(a).cuda() if a is not None else None
x, y, yp1, ypn = t(wl.x), t(wl.y), t(wl.yp1), t(wl.ypn)
lib = _lib.load()
fn = lib.spline_debug_tile_phases
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
buf = (ctypes.c_ulonglong * 8)()
api.build(x, y, wl.bc, yp1, ypn)
torch.cuda.synchronize()
fn(buf)
for _ in range(iters):
    api.build(x, y, wl.bc, yp1, ypn)
torch.cuda.synchronize()
fn(buf)
names = ["stage", "neighbours", "leaf sweep", "tree up", "tree down", "back-sub", "y2 store"]
tiles = wl.batch * max(1, -(-wl.n // 4096)) * iters
tot = sum(buf[:7])
print(f"cfg{cid}: {tiles} tile runs; cycles per tile (thread 0), share")
for k, nm in enumerate(names):
    print(f"  {nm:12s} {buf[k] / tiles:9.0f}  {buf[k] / max(tot, 1):5.1%}")
print(f"  {'total':12s} {tot / tiles:9.0f}")
