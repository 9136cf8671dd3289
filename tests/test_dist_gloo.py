"""Multi-rank orchestration of paper_2001_09253_b200.dist on CPU: gloo, world size 2 and 3.

The long-curve build (row partition -> per-rank block record -> all_gather of the
records -> redundant reduced solve -> per-rank finish -> all_gather of y2 shards) must
reproduce the oracle's y2; the statistics reduction must MAX/SUM across ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import seam_ref
from paper_2001_09253_b200 import dist as sdist
from paper_2001_09253_b200 import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, bc, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.generate(5, n=n, m=16)
        x, y = wl.x[0], wl.y[0]
        yp1, ypn = 0.7, -0.4
        ops = seam_ref.SeamRefOps(x, y, bc, yp1, ypn)
        y2s, (rb, re) = sdist.build_long_curve(torch.from_numpy(x), torch.from_numpy(y), bc, yp1, ypn, ops=ops)
        assert (rb, re) == sdist.shard_rows(n, world, rank)
        full = sdist.gather_curve(y2s, n)
        stats = sdist.reduce_stats({"err": float(rank + 1), "n_bad": 1.0})
        if rank == 0:
            q.put((full.numpy(), stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,bc", [(2, 500, 0), (3, 1001, 3), (2, 7, 1)])
def test_long_curve_build_gloo(world, n, bc):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), n, bc, q), nprocs=world, start_method="spawn")
    full, stats = q.get()
    wl = workloads.generate(5, n=n, m=16)
    ref, _ = oracle.build_y2(wl.x[0], wl.y[0], bc, [0.7], [-0.4])
    assert np.max(np.abs(full - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert stats == {"err": float(world), "n_bad": float(world)}


def test_shard_ranges_cover_rows():
    for n in (3, 10, 1 << 20):
        for world in (1, 2, 3, 8):
            rs = [sdist.shard_rows(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
