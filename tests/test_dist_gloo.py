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


def _worker_batched(rank, world, port, q):
    """Strong-scaling orchestration of the batched configs (bench.py --scaling strong): rank r
    takes curves [rB/G, (r+1)B/G) of the config, computes them (the oracle stands in for the
    per-rank GPU step here), and the shards' union is the whole batch; reduce_stats SUMs counts."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = workloads.generate(2, batch=53, m=12)
        full.q[7, 3] = full.x[7, 0] - 1.0                    # one out-of-range query (curve 7)
        b0, b1 = sdist.shard_batch(full.batch, world, rank)
        wl = workloads.slice_batch(full, b0, b1)
        y2, _ = oracle.build_y2(wl.x, wl.y, wl.bc, wl.yp1, wl.ypn)
        out, idx, nbad = oracle.evaluate(wl.x, wl.y, y2, wl.q)
        parts = [None] * world
        dist.all_gather_object(parts, (b0, b1, out, idx))
        stats = sdist.reduce_stats({"n_idx_out_of_range": float(nbad), "step_ms": float(rank + 1)})
        if rank == 0:
            q.put((parts, stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batched_strong_scaling_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker_batched, args=(world, _free_port(), q), nprocs=world, start_method="spawn")
    parts, stats = q.get()
    full = workloads.generate(2, batch=53, m=12)
    full.q[7, 3] = full.x[7, 0] - 1.0
    y2, _ = oracle.build_y2(full.x, full.y, full.bc, full.yp1, full.ypn)
    out, idx, nbad = oracle.evaluate(full.x, full.y, y2, full.q)
    assert [p[0] for p in parts] == [sdist.shard_batch(53, world, r)[0] for r in range(world)]
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), out)
    np.testing.assert_array_equal(np.concatenate([p[3] for p in parts]), idx)
    assert stats == {"n_idx_out_of_range": float(nbad), "step_ms": float(world)} and nbad == 1


def _worker_recompute(rank, world, port, n, bc, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = workloads.generate(5, n=n, m=16)
        x, y = wl.x[0], wl.y[0]
        ops = seam_ref.SeamRefOps(x, y, bc, 0.7, -0.4)
        y2 = sdist.build_long_curve_recompute(torch.from_numpy(x), torch.from_numpy(y), bc, 0.7, -0.4, ops=ops)
        ref, _ = oracle.build_y2(x, y, bc, [0.7], [-0.4])
        q.put((rank, float(np.max(np.abs(y2.numpy() - ref)) / np.max(np.abs(ref)))))  # small items: no pipe stall
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,bc", [(2, 4500, 0), (3, 7001, 3), (4, 2500, 1)])
def test_long_curve_recompute_gloo(world, n, bc):
    """§8(e)(ii): tile records all-gathered (whole tiles per rank, padded slabs), the full y2
    recomputed on EVERY rank; each rank's y2 is the oracle's."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker_recompute, args=(world, _free_port(), n, bc, q), nprocs=world, start_method="spawn")
    got = dict(q.get() for _ in range(world))
    assert sorted(got) == list(range(world))
    assert max(got.values()) <= 1e-12, got
