"""Multi-GPU spline: one process per GPU, torch.distributed (NCCL over NVLink) as plumbing.

Two parallel decompositions:

* Batched configurations (independent curves): rank r owns curves
  [r*B/G, (r+1)*B/G) and their queries.  No collective on the data path; the only
  collective is the final statistics reduction (``reduce_stats``).

* One long curve (BASELINE cfg5): the tridiagonal system's rows are partitioned,
  rank r owning rows [r*n/G, (r+1)*n/G) (``shard_rows``).  Each rank reduces its rows
  to one 6-scalar block record on its GPU (``spline_spike_reduce``), the G records are
  all-gathered (48 B per rank in fp64 -- the only exchange of the build), every rank
  solves the G-record reduced system redundantly and finishes its own rows
  (``spline_spike_finish``).  SURVEY.md Appendix A; the merge algebra is in
  csrc/build_tile.cuh.  Evaluation needs the whole curve on every rank: the y2 shards
  are all-gathered, then each rank evaluates its shard of the queries.

``ops`` (default: the CUDA library via ``api``) is injectable so the orchestration
(row ranges, gather order, seams) can be exercised on CPU with the gloo backend.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range [begin, end) of rank `rank` among `world` (balanced)."""
    return n * rank // world, n * (rank + 1) // world


def shard_batch(batch: int, world: int, rank: int) -> tuple[int, int]:
    return batch * rank // world, batch * (rank + 1) // world


class CudaOps:
    """The product path: every arithmetic step runs in libfastspline's kernels."""

    def __init__(self):
        from . import api
        self.api = api

    def workspace(self, n, rb, re, dtype, device):
        return self.api.spike_workspace(n, rb, re, dtype, device)

    def reduce(self, x, y, rb, re, bc, yp1, ypn, record, ws):
        self.api.spike_reduce(x, y, rb, re, bc, yp1, ypn, record, ws)

    def finish(self, x, y, rb, re, bc, yp1, ypn, all_records, world, rank, y2_shard, ws):
        self.api.spike_finish(x, y, rb, re, bc, yp1, ypn, all_records, world, rank, y2_shard, ws)

    def evaluate(self, x, y, y2, q, flags):
        return self.api.evaluate(x, y, y2, q, flags)

    def tile_rows(self, dtype):
        return self.api.spike_tile_rows(dtype)

    def tile_records(self, x, y, rb, re, bc, yp1, ypn, recs, ws):
        self.api.spike_tile_records(x, y, rb, re, bc, yp1, ypn, recs, ws)

    def finish_tiles(self, x, y, bc, yp1, ypn, all_recs, y2, ws):
        self.api.spike_finish_tiles(x, y, bc, yp1, ypn, all_recs, y2, ws)


def _slope(v, like):
    if v is None:
        return None
    if isinstance(v, torch.Tensor):
        return v.reshape(1).to(dtype=like.dtype, device=like.device)
    return torch.full((1,), float(v), dtype=like.dtype, device=like.device)


def build_long_curve(x: torch.Tensor, y: torch.Tensor, bc: int = 0, yp1=None, ypn=None, group=None, ops=None,
                     workspace=None):
    """Second derivatives of ONE long curve, rows partitioned over the process group.

    x, y: the full curve (n,), replicated on every rank.  Returns (y2_shard, (begin, end)):
    y2 for this rank's rows only.  One all_gather of 6 scalars per rank.
    """
    ops = ops or CudaOps()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = x.shape[-1]
    rb, re = shard_rows(n, world, rank)
    s0, s1 = _slope(yp1, x), _slope(ypn, x)
    ws = workspace if workspace is not None else ops.workspace(n, rb, re, x.dtype, x.device)
    record = torch.empty(6, dtype=x.dtype, device=x.device)
    ops.reduce(x, y, rb, re, bc, s0, s1, record, ws)
    if world > 1:
        all_records = torch.empty(6 * world, dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(all_records, record, group=group)
    else:
        all_records = record
    y2_shard = torch.empty(re - rb, dtype=x.dtype, device=x.device)
    ops.finish(x, y, rb, re, bc, s0, s1, all_records, world, rank, y2_shard, ws)
    return y2_shard, (rb, re)


def shard_tiles(n: int, tile_rows: int, world: int, rank: int) -> tuple[int, int, int, int]:
    """Whole tiles [t0, t1) of rank `rank` and their rows [rb, re) (the recompute build)."""
    ntiles = -(-n // tile_rows)
    t0, t1 = shard_batch(ntiles, world, rank)
    return t0, t1, t0 * tile_rows, min(t1 * tile_rows, n)


def build_long_curve_recompute(x: torch.Tensor, y: torch.Tensor, bc: int = 0, yp1=None, ypn=None, group=None,
                               ops=None, workspace=None):
    """Recompute instead of communicate: the FULL y2 (n,) on every rank.
    Each rank reduces its own whole tiles to tile records (K3); the records of all tiles are
    all-gathered (48 B per tile in fp64 -- 0.75 MB for cfg5's 16,384 tiles, instead of the 512 MB
    y2); every rank then solves the reduced system and finishes every tile itself (K4 + K5)."""
    ops = ops or CudaOps()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = x.shape[-1]
    ts = ops.tile_rows(x.dtype)
    ntiles = -(-n // ts)
    t0, t1, rb, re = shard_tiles(n, ts, world, rank)
    s0, s1 = _slope(yp1, x), _slope(ypn, x)
    ws = workspace if workspace is not None else ops.workspace(n, 0, n, x.dtype, x.device)
    per = -(-ntiles // world)  # equal slabs for all_gather_into_tensor (the last ones padded)
    slab = torch.zeros(per, 6, dtype=x.dtype, device=x.device)
    if t1 > t0:
        ops.tile_records(x, y, rb, re, bc, s0, s1, slab[: t1 - t0], ws)
    if world > 1:
        allr = torch.empty(per * world, 6, dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(allr, slab, group=group)
        parts = [allr[r * per: r * per + (shard_batch(ntiles, world, r)[1] - shard_batch(ntiles, world, r)[0])]
                 for r in range(world)]
        recs = torch.cat(parts).contiguous()
    else:
        recs = slab[:ntiles].contiguous()
    y2 = torch.empty(n, dtype=x.dtype, device=x.device)
    ops.finish_tiles(x, y, bc, s0, s1, recs, y2, ws)
    return y2


def gather_curve(y2_shard: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """All-gather the y2 shards of a row-partitioned curve into the full (n,) array."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return y2_shard
    sizes = [shard_rows(n, world, r) for r in range(world)]
    if len({e - b for b, e in sizes}) == 1:
        full = torch.empty(n, dtype=y2_shard.dtype, device=y2_shard.device)
        dist.all_gather_into_tensor(full, y2_shard, group=group)
        return full
    # uneven shards: gather equal-size padded slabs, then trim
    mx = max(e - b for b, e in sizes)
    slab = torch.zeros(mx, dtype=y2_shard.dtype, device=y2_shard.device)
    slab[: y2_shard.numel()] = y2_shard
    full = torch.empty(mx * world, dtype=y2_shard.dtype, device=y2_shard.device)
    dist.all_gather_into_tensor(full, slab, group=group)
    return torch.cat([full[r * mx: r * mx + (e - b)] for r, (b, e) in enumerate(sizes)])


def eval_long_curve(x, y, y2_full, q_shard, flags: int = 0, ops=None):
    """Evaluate this rank's shard of queries on the (replicated) full curve."""
    ops = ops or CudaOps()
    return ops.evaluate(x, y, y2_full, q_shard, flags)


def reduce_stats(stats: dict, group=None) -> dict:
    """The final error / statistics reduction: MAX of error ratios and times, SUM of counts."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return dict(stats)
    out = {}
    for k, v in stats.items():
        op = dist.ReduceOp.SUM if k.startswith("n_") else dist.ReduceOp.MAX
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op, group=group)
        out[k] = t.item()
    return out
