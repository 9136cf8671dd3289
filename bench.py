#!/usr/bin/env python
"""bench.py -- cubic-spline build + eval on B200 (arXiv 2001.09253 hot path).

One step = the whole hot path over one batch: spline_build (validate, assemble rows,
forward elimination, back-substitution) then spline_eval (locate + Eq. nr_formula),
through the C ABI, on inputs resident in HBM.  Default workload: BASELINE.json
configs[3], cfg4 (4,096 curves x 4,096 knots, fp64 -- the paper's binary64, P:1747-1748 --,
clamped, 16 sorted queries per knot): the largest batched configuration on one GPU.  The other
configurations via --config (cfg2 = configs[1], the fp32 many-curve case).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): weak scaling -- every rank builds and evaluates
its own shard of curves (same shape, its own seed); no collective on the data path.
Timing: CUDA events on the launching stream around every step, L2 flushed (256 MiB
write) between steps outside the events, barrier + synchronize around the K steps, max
over ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spline build+eval knots/s and queries/s; achieved HBM GB/s vs B200 peak"
SPEC_HBM_GBS = 8000.0  # BASELINE.json's "~8 TB/s" denominator (context)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="batched configs on N GPUs: strong = rank r owns curves [rB/N, (r+1)B/N) of the config "
                         "(SURVEY §8(e)); weak = every rank its own full-size batch (seeded per rank)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cfg5-mode", default="recompute", choices=["recompute", "gather"],
                    help="cfg5 on N GPUs (SURVEY §8(e)): recompute = tile records all-gathered, every rank "
                         "finishes the whole curve; gather = the rank-record seam, then an all-gather of y2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--x-shared", action="store_true",
                    help="shared-knot mode (SPLINE_X_SHARED): one knot vector for the batch (configs whose recipe "
                         "has one grid: cfg3)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ablation", action="store_true",
                    help="SURVEY §8(f) rows 2-3: the paper's control-point sweep (n = 4 .. 2^20) with its "
                         "interpolation variants and no-op loop, ns/point p16/p50/p84 (one JSON line)")
    ap.add_argument("--sweep-points", type=int, default=14)
    ap.add_argument("--reps", type=int, default=7)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_for(workload_key: str, kernel: str):
    """Per-launch DRAM traffic of the kernel from the current ncu capture (profiles/traffic.json,
    written by tools/traffic_capture.py): dram__bytes_read.sum + the bytes the kernel WROTE --
    the larger of dram__bytes_write.sum and the L2 write sectors from the SMs
    (lts__t_sectors_srcunit_tex_op_write.sum x 32 B), because writes still dirty in L2 when the
    kernel ends reach DRAM only later and dram__bytes_write.sum misses them."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    e = d.get(workload_key, {}).get(kernel)
    if isinstance(e, dict):
        return e.get("traffic"), {k: v for k, v in e.items() if k != "traffic"} | {"source": d.get("_source")}
    return e, None


def pstats(ms):
    """Median with p16 / p84 (the paper's own summary of a timing distribution)
    and the mean."""
    a = np.asarray(ms, dtype=np.float64)
    p16, p50, p84 = np.percentile(a, [16, 50, 84])
    return {"median": float(p50), "p16": float(p16), "p84": float(p84), "mean": float(a.mean()), "n": int(a.size)}


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            h = None
            try:
                bus = torch.cuda.get_device_properties(dev_index).pci_bus_id
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hh = pynvml.nvmlDeviceGetHandleByIndex(i)
                    b = pynvml.nvmlDeviceGetPciInfo(hh).busId
                    b = b.decode() if isinstance(b, bytes) else b
                    if b.lower().endswith(bus.lower()[-7:]):
                        h = hh
            except Exception:
                h = None
            self.h = h if h is not None else pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        rs = [name for bit, name in self.REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": rs, "samples": len(self.samples)}


def long_curve_cfg(n, s):
    return n > 256 * (16 if s == 8 else 32)


def algorithmic_bytes(B, n, m, s, xshared=False):
    """build 3 s B/knot (read x, y; write y2) + 2 s per clamped curve;
    eval (2 s + 4) B/query (read q; write out, int32 idx) + 3 n s per curve (x, y, y2).
    Shared-knot mode: x is read once for the batch (n s), not per curve."""
    xb = s * n if xshared else s * B * n
    build = 2 * s * B * n + xb
    evalb = (2 * s + 4) * B * m + 2 * n * s * B + xb
    return build, evalb


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, timed on the host cores (rank 0 only).
    Each step is one whole build + eval pass of the SAME workload as our arm when K + W such
    passes fit the time budget (~3 min); otherwise of a bounded sample of it (curves; for the
    one-curve cfg5, queries), chosen from one timed full pass and stated in `sample`."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2001_09253_b200 import workloads
    spec = workloads.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    budget = 180.0
    wl = workloads.generate(args.config)

    def one_pass(w):
        t0 = time.perf_counter()
        y2, _ = oracle.build_y2(w.x, w.y, w.bc, w.yp1, w.ypn, nthreads=cores)
        oracle.evaluate(w.x, w.y, y2, w.q, nthreads=cores)
        return time.perf_counter() - t0

    full = wl
    if args.config == 5:  # a full pass is ~10-20 s of host work: probe with a query sample first
        probe = workloads.Workload(wl.spec, wl.x, wl.y, wl.q[:, : 1 << 22], wl.yp1, wl.ypn, wl.bc, wl.flags)
        per = one_pass(probe) * wl.m / probe.m
    else:
        per = one_pass(wl)
    frac = min(1.0, budget / max(per * (args.steps + args.warmup), 1e-9))
    if frac < 1.0:
        if args.config == 5:
            mm = max(1 << 16, int(wl.m * frac))
            wl = workloads.Workload(wl.spec, wl.x, wl.y, wl.q[:, :mm], wl.yp1, wl.ypn, wl.bc, wl.flags)
        else:
            bb = max(1, int(wl.batch * frac))
            sl = lambda a: None if a is None else a[:bb]
            wl = workloads.Workload(wl.spec, wl.x[:bb], wl.y[:bb], wl.q[:bb], sl(wl.yp1), sl(wl.ypn), wl.bc, wl.flags)
    times = []
    for it in range(args.warmup + args.steps):
        t = one_pass(wl)
        if it >= args.warmup:
            times.append(t)
    st = pstats([t * 1e3 for t in times])
    t = st["median"] * 1e-3
    qps = wl.batch * wl.m / t
    same = wl.batch == full.batch and wl.m == full.m
    sample = (f"{'the full workload' if same else 'a sample'}: {wl.batch} curves x n={wl.n} x m={wl.m} of {spec.name} "
              f"per step (build + eval, {cores} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": st["median"], "step_ms_stats": st,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle; inputs widened)",
            "data": "synthetic (seeded, BASELINE.json config recipe)",
            "config": {"workload": spec.name, "batch": wl.batch, "n": wl.n, "m": wl.m, "same_config": same},
            "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "knots_per_s": wl.batch * wl.n / t}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, wl_full):
    import oracle
    cores = os.cpu_count() or 1
    wl = wl_full
    if wl.x.ndim == 1:  # shared knots: the oracle takes one row per curve
        from paper_2001_09253_b200 import workloads
        wl = workloads.Workload(wl.spec, np.tile(wl.x, (wl.batch, 1)), wl.y, wl.q, wl.yp1, wl.ypn, wl.bc, wl.flags)
    if args.config in (4, 5):  # bound the sample to ~10-30 s of CPU work
        from paper_2001_09253_b200 import workloads
        wl = workloads.generate(args.config, batch=64 if args.config == 4 else None,
                                n=None if args.config == 4 else 1 << 22, m=None if args.config == 4 else 1 << 24)
    # whole passes (build + eval) repeated until ~10 s of CPU work, for a stable number
    passes, t = 0, 0.0
    t0 = time.perf_counter()
    while passes == 0 or t < 10.0:
        y2, _ = oracle.build_y2(wl.x, wl.y, wl.bc, wl.yp1, wl.ypn, nthreads=cores)
        oracle.evaluate(wl.x, wl.y, y2, wl.q, nthreads=cores)
        passes += 1
        t = time.perf_counter() - t0
    return {"value": passes * wl.batch * wl.m / t, "unit": "queries/s", "cores": cores, "kind": "oracle",
            "sample": f"{passes} pass(es) of {wl.batch} curves x n={wl.n} x m={wl.m} (build + eval, {cores} "
                      f"threads), {t:.1f} s", "knots_per_s": passes * wl.batch * wl.n / t}


def run_long_curve_dist(args, world, rank, local, dev):
    """cfg5 on G GPUs (strong scaling): the one long curve's rows are partitioned (SPIKE:
    per-rank block record -> NCCL all_gather of 6 scalars per rank -> redundant reduced solve
    -> per-rank finish), the y2 shards are all-gathered (NCCL), and each rank evaluates its
    shard of the 2^28 queries.  All of it is inside the timed step."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2001_09253_b200 import api, workloads
    from paper_2001_09253_b200 import dist as sdist

    spec = workloads.CONFIGS[5]
    wl = workloads.generate(5, m=1)  # x, y identical on every rank (drawn before q)
    n, M = wl.n, spec.m
    qb, qe = sdist.shard_batch(M, world, rank)
    rng = np.random.default_rng([spec.seed, 1000 + rank])
    q = torch.from_numpy(rng.random(qe - qb)[None]).to(dev)
    x = torch.from_numpy(wl.x[0]).to(dev)
    y = torch.from_numpy(wl.y[0]).to(dev)
    rb, re = sdist.shard_rows(n, world, rank)
    ws = api.spike_workspace(n, rb, re, x.dtype, dev)
    out = torch.empty_like(q)
    idx = torch.empty(q.shape, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    wsf = api.spike_workspace(n, 0, n, x.dtype, dev) if args.cfg5_mode == "recompute" else None

    def step():
        if args.cfg5_mode == "recompute":  # §8(e)(ii): no y2 on the wire, every rank finishes all tiles
            y2 = sdist.build_long_curve_recompute(x, y, wl.bc, workspace=wsf)
        else:                              # §8(e)(i): rank records, then the y2 shards all-gathered
            y2s, _ = sdist.build_long_curve(x, y, wl.bc, workspace=ws)
            y2 = sdist.gather_curve(y2s, n)
        api.evaluate(x[None], y[None], y2[None], q, 0, out=out, idx=idx)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(K):
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([statistics.mean(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    if rank == 0:
        build_bytes, eval_bytes = algorithmic_bytes(1, n, M, 8)
        peak, peak_src = peaks()
        line = {"metric": METRIC, "value": M / (ms * 1e-3), "unit": "queries/s", "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded PCG64, BASELINE.json cfg5 recipe; per-rank query shards)",
                "config": {"workload": spec.name, "n": n, "m_total": M, "cfg5_mode": args.cfg5_mode,
                           "parallelism": (f"whole tiles sharded over {world} GPUs, tile records all-gathered (NCCL), "
                                           "every rank finishes the whole curve, queries sharded"
                                           if args.cfg5_mode == "recompute" else
                                           f"rows sharded over {world} GPUs (SPIKE, NCCL record all_gather), "
                                           "y2 all_gather, queries sharded"),
                           "l2": "inputs (1.5 GiB curve, 2 GiB queries) exceed L2"},
                "knots_per_s": n / (ms * 1e-3),
                "hbm_gbs_step_per_gpu": (build_bytes / world + eval_bytes / world) / (ms * 1e-3) / 1e9,
                "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": 7 * K,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def run_ablation(args):
    """The paper's timing experiment on one B200: control-point counts from the
    biased schedule, random curves (y = eps, x_i = x_{i-1} + eps), n uniformly spaced points
    per curve, fp64; every (n, variant) pair in a freshly shuffled order per repetition, L2
    flushed before each timed launch (CUDA events).  Each launch evaluates B = max(1, 2^22 / n)
    curves so that the GPU is filled; reported per point.  Variants: the product form, the
    paper's splint div/mul and newint orig/noinv, and the no-op (locate-only) loop."""
    import random

    import torch

    from paper_2001_09253_b200 import _lib, api, workloads
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # the paper's schedule, plus powers of two below 4096 (its coarse steps skip the short curves)
    sched = sorted(set(workloads.sweep_schedule(args.sweep_points)) | {1 << k for k in range(2, 12)})
    data = {}
    for n in sched:
        B = max(1, (1 << 22) // n)
        x, y, q = workloads.sweep_curves(n, B, seed=11)
        X, Y, Q = (torch.from_numpy(a).to(dev) for a in (x, y, q))
        Z = api.build(X, Y, api.BC_NATURAL)
        data[n] = (X, Y, Z, Q, torch.empty_like(Q), torch.empty(Q.shape, dtype=torch.int32, device=dev), B)
    forms = list(_lib.FORMS)
    times = {(n, f): [] for n in sched for f in forms}
    rng = random.Random(0)
    for _ in range(2):  # warm-up
        for n in sched:
            X, Y, Z, Q, O, I, B = data[n]
            for f in forms:
                api.evaluate_ablation(X, Y, Z, Q, f, out=O, idx=I)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        for _ in range(args.reps):
            order = [(n, f) for n in sched for f in forms]
            rng.shuffle(order)
            for n, f in order:
                X, Y, Z, Q, O, I, B = data[n]
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                api.evaluate_ablation(X, Y, Z, Q, f, out=O, idx=I)
                b.record()
                b.synchronize()
                times[(n, f)].append(a.elapsed_time(b) * 1e6 / (B * n))  # ns per point
    if api.status() != 0:
        raise RuntimeError("data-error status raised in the ablation sweep")
    rows = []
    for n in sched:
        row = {"n": n, "curves": data[n][6], "points": data[n][6] * n}
        for f in forms:
            p16, p50, p84 = np.percentile(times[(n, f)], [16, 50, 84])
            row[f] = {"p16": p16, "p50": p50, "p84": p84}
        rows.append(row)
    line = {"mode": "ablation", "metric": "ns per interpolated point (GPU-wide, B curves per launch)",
            "unit": "ns/point", "dtype": "f64", "kernel": "k_eval_sorted<FORM> (spline_eval_ablation)",
            "forms": forms, "reps": args.reps, "schedule": sched, "rows": rows, "clocks": clk.summary(),
            "data": "synthetic: the paper's random curves (y = eps, x_i = x_{i-1} + eps, eps ~ U(0,1)), "
                    "n uniformly spaced points per curve"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.ablation:
        run_ablation(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2001_09253_b200 import api, workloads

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test tooling only (tests/test_gpu_bench.py): FS_BENCH_BACKEND=gloo with FS_BENCH_ONE_GPU=1 runs
    # the N-rank orchestration with every rank on device 0 -- a functional check of the multi-rank
    # path on a one-GPU box, never a measurement (ranks sharing a GPU time each other)
    backend = os.environ.get("FS_BENCH_BACKEND", "nccl")
    if os.environ.get("FS_BENCH_ONE_GPU"):
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    if args.config == 5 and world > 1:
        run_long_curve_dist(args, world, rank, local, dev)
        dist.destroy_process_group()
        return

    from paper_2001_09253_b200 import dist as sdist
    spec = workloads.CONFIGS[args.config]
    # strong scaling (default): the config's batch split over the ranks -- the same inputs as at
    # N = 1; a batch smaller than the rank count (cfg1) runs as replicas (weak)
    scaling = args.scaling if spec.batch >= world else "weak"
    if scaling == "strong" and world > 1:
        full = workloads.generate(args.config)
        b0, b1 = sdist.shard_batch(full.batch, world, rank)
        wl = workloads.slice_batch(full, b0, b1)
        del full
    else:
        wl = workloads.generate(args.config, shard=rank)
    total_q = spec.batch * spec.m if (scaling == "strong" and world > 1) else world * wl.batch * wl.m
    B, n, m = wl.batch, wl.n, wl.m
    s = 4 if spec.dtype == "f32" else 8
    stream = torch.cuda.current_stream()

    def dev_t(a):
        return torch.from_numpy(a).to(dev) if a is not None else None

    if args.x_shared:
        if not np.all(wl.x == wl.x[0]):
            raise SystemExit("--x-shared: this configuration's curves do not share one grid")
        wl.x = np.ascontiguousarray(wl.x[0])  # (n,): one knot vector for the batch
    x, y, q = dev_t(wl.x), dev_t(wl.y), dev_t(wl.q)
    yp1, ypn = dev_t(wl.yp1), dev_t(wl.ypn)
    y2 = torch.empty_like(y)
    out = torch.empty_like(q)
    idx = torch.empty(q.shape, dtype=torch.int32, device=dev)
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.zeros(64 << 20, dtype=torch.float32, device=dev)

    class _Flush:
        """Between timed steps, outside the events: write 256 MiB (> the 126 MB L2: evicts it), then
        read 256 MiB so that the written lines are cleaned (written back) before the next step
        instead of draining inside it."""

        @staticmethod
        def zero_():
            flush_w.zero_()
            flush_r.sum()

    flush = _Flush()

    def step():  # the library's build+eval entry point: it picks fused or split per problem size
        api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, y2=y2, out=out, idx=idx)

    api.status()
    # untimed warm-up: at least W steps and 0.3 s, then one untimed pass of the timed protocol
    # itself (flush + events + step, queued): the first queued pass of a µs-sized step runs
    # measurably slower than the following ones
    t_end = time.perf_counter() + 0.3
    w = 0
    while w < max(args.warmup, 3) or time.perf_counter() < t_end:
        step()
        w += 1
        if w % 64 == 0:
            torch.cuda.synchronize()
    wev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    for k in range(args.steps):
        flush.zero_()
        wev[2 * k].record(stream)
        step()
        wev[2 * k + 1].record(stream)
    torch.cuda.synchronize()
    if api.status() != 0:
        raise RuntimeError("data-error status raised on the benchmark inputs")

    K = args.steps
    # the step: spline_build_eval (C ABI) -- one fused kernel for small problems (batch*m <= 2^17),
    # else build then eval back to back (the eval launch may overlap the build's drain:
    # programmatic dependent launch); CUDA events around it
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(K):
            flush.zero_()  # evict L2 (126 MB) between steps, outside the timed events
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_list = [ev[k][0].elapsed_time(ev[k][1]) for k in range(K)]
    step_st = pstats(step_list)
    step_ms = step_st["median"]
    # per-kernel breakdown (for the rooflines): each kernel timed alone, same flush protocol
    bev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for k in range(K):
        flush.zero_()
        bev[k][0].record(stream)
        api.build(x, y, wl.bc, yp1, ypn, out=y2)
        bev[k][1].record(stream)
        flush.zero_()
        bev[k][2].record(stream)
        api.evaluate(x, y, y2, q, wl.flags, out=out, idx=idx)
        bev[k][3].record(stream)
    torch.cuda.synchronize()
    build_ms = [bev[k][0].elapsed_time(bev[k][1]) for k in range(K)]
    eval_ms = [bev[k][2].elapsed_time(bev[k][3]) for k in range(K)]

    # ---- the fused single-kernel path (spline_build_eval, SPLINE_PATH_FUSED), same protocol
    fused_ms = 0.0
    tile_fusable = bool(wl.flags & workloads.FLAG_Q_SORTED) and 128 < n <= 256 * (16 if s == 8 else 32)
    fusable = (n <= 128 and (n * s) % 16 == 0 and m % (16 // s) == 0) or tile_fusable
    if fusable:
        ff = wl.flags | api.PATH_FUSED

        def fstep():
            api.build_eval(x, y, q, wl.bc, yp1, ypn, ff, y2=y2, out=out, idx=idx)

        for _ in range(3):
            fstep()
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            flush.zero_()
            fev[k][0].record(stream)
            fstep()
            fev[k][1].record(stream)
        torch.cuda.synchronize()
        fused_ms = statistics.mean(a.elapsed_time(b) for a, b in fev)
    # ---- the split path as one call (spline_build_eval with SPLINE_PATH_SPLIT), same protocol
    sf = wl.flags | api.PATH_SPLIT
    for _ in range(3):
        api.build_eval(x, y, q, wl.bc, yp1, ypn, sf, y2=y2, out=out, idx=idx)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        flush.zero_()
        sev[k][0].record(stream)
        api.build_eval(x, y, q, wl.bc, yp1, ypn, sf, y2=y2, out=out, idx=idx)
        sev[k][1].record(stream)
    torch.cuda.synchronize()
    split_ms = statistics.median(a.elapsed_time(b) for a, b in sev)
    build_st, eval_st = pstats(build_ms), pstats(eval_ms)
    t = torch.tensor([step_ms, build_st["median"], eval_st["median"], fused_ms, split_ms], dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, bms, ems, fused_ms, split_ms = t.tolist()

    # ---- cfg5: the random-gather ceiling: the same gathers at known intervals
    gather = None
    if long_curve_cfg(n, s):
        def probe_ms(mode):
            pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
            api.gather_probe(x, y, y2, q, idx, mode, out=pout, idx=pidx)
            for kk in range(K):
                flush.zero_()
                pev[kk][0].record(stream)
                api.gather_probe(x, y, y2, q, idx, mode, out=pout, idx=pidx)
                pev[kk][1].record(stream)
            torch.cuda.synchronize()
            return statistics.mean(a.elapsed_time(b) for a, b in pev)
        pout, pidx = torch.empty_like(out), torch.empty_like(idx)
        raw_ms, rec_ms = probe_ms(0), probe_ms(1)
        gather = {"raw_3array_ms": raw_ms, "records_ms": rec_ms, "eval_ms": None,
                  "note": "spline_gather_probe: evaluation at the already known intervals (no search); "
                          "records_ms includes building the records, like the eval path"}

    # ---- end to end through the public API with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        h_in = [torch.from_numpy(a).pin_memory() for a in (wl.x, wl.y, wl.q)]
        h_sl = [torch.from_numpy(a).pin_memory() if a is not None else None for a in (wl.yp1, wl.ypn)]
        h_y2 = torch.empty(y.shape, dtype=x.dtype).pin_memory()
        h_out = torch.empty(q.shape, dtype=q.dtype).pin_memory()
        h_idx = torch.empty(q.shape, dtype=torch.int32).pin_memory()

        def e2e_step():  # spline_build_eval_host: chunks of curves, copies overlapped with kernels
            api.build_eval_host(h_in[0], h_in[1], h_in[2], wl.bc, h_sl[0], h_sl[1], wl.flags, y2=h_y2, out=h_out,
                                idx=h_idx, sync=False)

        e2e_step()
        torch.cuda.synchronize()
        KE = max(1, min(args.e2e_steps, K))
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(KE):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / KE], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = sum(a.nbytes for a in (wl.x, wl.y, wl.q)) + sum(a.nbytes for a in (wl.yp1, wl.ypn) if a is not None)
        d2h = y.numel() * s + q.numel() * s + q.numel() * 4
        e2e = {"value": total_q / (te.item() * 1e-3), "unit": "queries/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": te.item(), "pinned": True,
               "path": "api.build_eval_host (C ABI spline_build_eval_host): pinned host in/out, the batch in chunks "
                       "whose H2D copies, kernels and D2H copies overlap on internal streams"}

    # the final statistics reduction (NCCL when N > 1): data-error bits, out-of-range and NaN counts
    # over all ranks' outputs, and the slowest rank's step time
    api.build_eval(x, y, q, wl.bc, yp1, ypn, wl.flags, y2=y2, out=out, idx=idx)
    bits = api.status()
    stats = sdist.reduce_stats({"status_bits": float(bits), "n_idx_out_of_range": float((idx < 0).sum().item()),
                                "n_out_nan": float(torch.isnan(out).sum().item()), "step_ms": step_ms})
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    bbytes, ebytes = algorithmic_bytes(B, n, m, s, args.x_shared)
    peak, peak_src = peaks()
    tkey = f"cfg{args.config}" + ("_xshared" if args.x_shared else "")
    etr, etr_d = traffic_for(tkey, "eval")
    btr, btr_d = traffic_for(tkey, "build")
    ach = ebytes / (ems * 1e-3) / 1e9
    wkey = f"cfg{args.config}"
    long_curve = n > 256 * (16 if s == 8 else 32)
    # the library's choice inside spline_build_eval (spline_abi.cu build_eval_t): one fused kernel
    # when the problem is small (batch*m <= 2^17) and fusable, else the two kernels
    small_step = s == 4 and n <= 8 and 0 < m <= 32 and m % 4 == 0  # k_eval_small<true>: solve + eval
    tiny_step = (n == 16 or (s == 4 and n in (32, 64))) and B <= 16 and m <= 8192 and m % (16 // s) == 0
    # many K1h-sized curves (cfg2): k_build_eval_warp solves and evaluates per warp
    warp_step = ((n == 16 or (s == 4 and n in (32, 64))) and B >= 4 * 148 and m > 0 and m % (16 // s) == 0
                 and not (wl.flags & workloads.FLAG_X_UNIFORM) and not args.x_shared and not small_step)
    fused_step = fusable and not tile_fusable and B * m <= (1 << 17) and not warp_step
    # mid-length curves with sorted queries (cfg4): k_tile_eval solves and evaluates in one kernel
    tile_step = False  # k_tile_eval runs on SPLINE_PATH_FUSED only (measured slower than split on cfg4)
    launches = 2 * K  # 1 build kernel + 1 eval kernel per step for configs 2-4
    if long_curve:
        # tiled SPIKE: reduce + top (grouped for one curve of > 128 tiles: up, root, down) + finish;
        # eval: pack records + gather
        ntiles = -(-n // (256 * (16 if s == 8 else 32)))
        bucketed = B == 1 and 3 * s * n > 4 * (24 << 20) and m >= (1 << 20) and m >= n // 4
        # build: memset + K3 + K4 (3 grouped launches for one curve of > 128 tiles, else 1) + K5;
        # eval: bucketed (count, pack, scan x2, scatter, eval, gather) or records (pack, gather)
        launches = ((5 if (B == 1 and ntiles > 128) else 3) + (7 if bucketed else 2)) * K
    if fused_step or small_step or tiny_step or tile_step or warp_step:
        launches = K
    one_kernel = fused_step or small_step or tiny_step or tile_step or warp_step
    xread = s * n if args.x_shared else s * B * n
    # §8(d)'s per-unit figures x the units one step processes: build 3s B/knot + eval (2s+4) B/query
    # + 3ns B/curve -- the same for one fused launch as for the two kernels; a fused kernel's own
    # minimum (x, y read once, y2 written once, never read back) is reported beside it
    step_bytes = bbytes + ebytes
    fused_min_bytes = (2 * s + 4) * B * m + 2 * s * B * n + xread
    if wl.flags & workloads.FLAG_Q_SORTED:
        ekern = "k_eval_sorted"
    elif s == 4 and n <= 8 and 0 < m <= 32 and m % 4 == 0:
        ekern = "k_eval_small"
    elif (n <= 64 and B >= 4 * 148 and m % (16 // s) == 0 and not (wl.flags & workloads.FLAG_X_UNIFORM)):
        ekern = "k_eval_curvewarp"
    elif long_curve and B == 1 and 3 * s * n > 4 * (24 << 20) and m >= (1 << 20) and m >= n // 4:
        ekern = "k_bucket_count + k_pack_knots + k_scan + k_bucket_scatter + k_bucket_eval + k_bucket_gather"
    elif long_curve or 3 * n * s > 200 * 1024:
        ekern = "k_pack_records + k_eval_records"
    elif n <= 512 and not (wl.flags & workloads.FLAG_X_UNIFORM) and B >= 8 and m < 2048:
        ekern = "k_eval_warps"
    else:
        ekern = "k_eval_staged"
    half = n == 16 or (s == 4 and n in (32, 64))  # K1h: half curves in registers
    bkern = ("k1_thomas_regs" if n <= 8 else "k1_thomas_half" if half else "k1_thomas_pipe" if n <= 128 else
             "k_tile<FULL>" if not long_curve else "k_tile<REDUCE> + k4_top + k_tile<FINISH>")
    split_roof = {"kernel": ekern, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                  "frac": ach / peak, "traffic": etr, "traffic_detail": etr_d, "peak_source": peak_src,
                  "algorithmic_bytes_per_launch": ebytes,
                  "build": {"kernel": bkern, "achieved": bbytes / (bms * 1e-3) / 1e9,
                            "frac": bbytes / (bms * 1e-3) / 1e9 / peak,
                            "algorithmic_bytes_per_launch": bbytes, "traffic": btr, "traffic_detail": btr_d}}
    if one_kernel:
        # the step IS one kernel: it is the dominant kernel; its launch is bracketed by the step's events
        skern = ("k_tile_eval" if tile_step else "k_eval_small<true>" if small_step else
                 "k_build_eval_tiny" if tiny_step else "k_build_eval_warp" if warp_step else "k_fused_staged")
        str_, str_d = traffic_for(tkey, "step")
        sach = step_bytes / (step_ms * 1e-3) / 1e9
        roof = {"kernel": skern, "bound": "hbm", "achieved": sach, "peak": peak, "unit": "GB/s", "frac": sach / peak,
                "traffic": str_, "traffic_detail": str_d, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": step_bytes,
                "note": "algorithmic bytes (SURVEY.md §8(d) per unit): build 3s B/knot + eval (2s+4) B/query "
                        "+ 3ns B/curve, for the build and eval units the one launch processes",
                "fused_min_bytes": fused_min_bytes,
                "fused_min_frac": fused_min_bytes / (step_ms * 1e-3) / 1e9 / peak,
                "fused_min_note": "the fused kernel's own minimum traffic: x, y read once, y2 written once "
                                  "and never read back, (2s+4) B/query",
                "split_path": split_roof}
    else:
        roof = split_roof
    line = {
        "metric": METRIC,
        "value": total_q / (step_ms * 1e-3),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "step_ms_stats": step_st,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": spec.dtype,
        "data": "synthetic (seeded PCG64, BASELINE.json config recipe; DESIGN.md input recipe)",
        "config": {"workload": spec.name + (" [shared knots: SPLINE_X_SHARED]" if args.x_shared else ""),
                   "batch_per_gpu": B, "n": n, "m": m, "bc": wl.bc, "flags": wl.flags, "x_shared": args.x_shared,
                   "l2": "flushed between steps, outside the timed events: 256 MiB written (evicts the 126 MB L2), "
                         "then 256 MiB read (cleans the written lines)",
                   "parallelism": (f"dp{world}: rank r owns curves [rB/{world}, (r+1)B/{world}) of the config, "
                                   "no data-path collective" if scaling == "strong" and world > 1 else
                                   f"dp{world}: {'replicas' if spec.batch < world else 'a full batch per rank'}, "
                                   "no data-path collective")},
        "stats": stats,
        "knots_per_s": (total_q // m) * n / (step_ms * 1e-3),
        "hbm_gbs_step": (bbytes + ebytes) / (step_ms * 1e-3) / 1e9,
        "frac_of_spec_8tbs_step": (bbytes + ebytes) / (step_ms * 1e-3) / 1e9 / SPEC_HBM_GBS,
        "build_ms": bms,
        "eval_ms": ems,
        "split_step_ms": split_ms,
        "build_ms_stats": build_st,
        "eval_ms_stats": eval_st,
        "timing": "CUDA events on the launching stream; value and ms_per_step use the median step "
                  "(p16 / p84 / mean in step_ms_stats), max over ranks",
        "build_gbs": bbytes / (bms * 1e-3) / 1e9,
        "step_roofline": {"bound": "hbm", "unit": "GB/s", "peak": peak,
                          "algorithmic_bytes": step_bytes, "achieved": step_bytes / (step_ms * 1e-3) / 1e9,
                          "frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak,
                          "note": "the whole timed step (build + eval), §8(d)'s per-unit bytes"},
        "step_path": ("fused (k_tile_eval: K2's solve, y2 kept on chip, sorted-run eval)" if tile_step else
                      "fused (k_eval_small<true>: K1r's solve + the small-curve eval)" if small_step else
                      "fused (k_build_eval_tiny: one CTA per curve, K1h's solve + eval)" if tiny_step else
                      "fused (k_build_eval_warp: K1h's solve per group of 16 curves, y2 staged on chip, "
                      "curvewarp eval)" if warp_step else
                      "fused (k_fused_staged)" if fused_step else "split (build kernel(s), then eval kernel(s))"),
        "roofline": roof,
        "fused": ({"kernel": "k_tile_eval" if tile_fusable else "k_fused_staged", "ms_per_step": fused_ms, "value": total_q / (fused_ms * 1e-3),
                   "unit": "queries/s", "algorithmic_bytes": (2 * s + 4) * B * m + 3 * s * B * n,
                   "hbm_gbs": ((2 * s + 4) * B * m + 3 * s * B * n) / (fused_ms * 1e-3) / 1e9,
                   "note": "spline_build_eval with SPLINE_PATH_FUSED (one launch; x, y read once, y2 written once)"}
                  if fusable else None),
        "cpu_baseline": None,
        "e2e": e2e,
        "gather_ceiling": (dict(gather, eval_ms=ems, eval_over_records_ceiling=gather["records_ms"] / ems)
                           if gather else None),
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args, wl)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
