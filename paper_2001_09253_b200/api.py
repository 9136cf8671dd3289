"""torch-tensor front end of the C ABI (include/spline.h).

PyTorch provides device memory and streams only; every step of build and eval runs
in libfastspline's sm_100a kernels.  All tensors are CUDA, C-contiguous, curve-major:
x, y, y2 (B, n); q, out (B, m); idx (B, m) int32; yp1, ypn (B,).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (BC_CLAMP_END, BC_CLAMP_START, BC_CLAMPED, BC_NATURAL, NO_BUCKET, PATH_FUSED,  # noqa: F401
                   PATH_SPLIT, Q_SORTED, STATUS_BAD_KNOTS, STATUS_Q_OUT_OF_RANGE, X_SHARED, X_UNIFORM)

_DT = {torch.float32: _lib.SPLINE_F32, torch.float64: _lib.SPLINE_F64}


def _stream(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_curves(x, *others):
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise ValueError("spline ops take CUDA tensors (no CPU fallback)")
    if x.dtype not in _DT:
        raise ValueError(f"dtype must be float32 or float64, got {x.dtype}")
    for t in (x, *others):
        if t is None:
            continue
        if t.device != x.device or t.dtype != x.dtype or not t.is_contiguous():
            raise ValueError("all arrays must be contiguous, on the same device, same dtype")


def _as2d(t):
    return t.unsqueeze(0) if t is not None and t.dim() == 1 else t


def _check_buf(t, shape, dtype, device, what, host=False):
    """A caller-supplied buffer the C library reads or writes in full: exact shape, dtype,
    placement (the curves' device, or a CPU tensor for the host entry) and contiguity."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{what} must be a torch tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{what} must be {dtype}, got {t.dtype}")
    if host:
        if t.device.type != "cpu":
            raise ValueError(f"{what} must be a CPU tensor (build_eval_host)")
    elif t.device != device:
        raise ValueError(f"{what} must be on {device}, got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")


def _curves(x, y):
    """The knots and values of a call: (x2d, y2d, shared, squeeze).  x (n,) with y (B, n) is the
    shared-knot mode (SPLINE_X_SHARED: one knot vector for the whole batch); x, y both (n,) is
    one curve; both (B, n) a batch."""
    if isinstance(x, torch.Tensor) and isinstance(y, torch.Tensor) and x.dim() == 1 and y.dim() == 2:
        if x.shape[0] != y.shape[1]:
            raise ValueError("shared knots: x must be (n,) for y (B, n)")
        return x.unsqueeze(0), y, True, False
    squeeze = x.dim() == 1
    x, y = _as2d(x), _as2d(y)
    if y.shape != x.shape:
        raise ValueError("x and y must have the same shape (or x (n,) shared by y (B, n))")
    return x, y, False, squeeze


def _slopes(v, B, like, host=False):
    """Per-curve clamped slope: a scalar is broadcast, a tensor must be (B,)."""
    if v is None:
        return None
    if not isinstance(v, torch.Tensor):
        return torch.full((B,), float(v), dtype=like.dtype, device="cpu" if host else like.device)
    return v


def build(x: torch.Tensor, y: torch.Tensor, bc: int = BC_NATURAL, yp1=None, ypn=None, out=None, stream=None):
    """Second derivatives y2 of the curves (x, y): (B, n) or (n,), or x (n,) shared by y (B, n).
    Returns y2 (y's shape)."""
    x, y, shared, squeeze = _curves(x, y)
    B, n = y.shape
    yp1, ypn = _slopes(yp1, B, x), _slopes(ypn, B, x)
    _check_curves(x, y)
    _check_buf(yp1, (B,), x.dtype, x.device, "yp1")
    _check_buf(ypn, (B,), x.dtype, x.device, "ypn")
    y2 = torch.empty_like(y) if out is None else _as2d(out)
    _check_buf(y2, y.shape, x.dtype, x.device, "y2 (out)")
    rc = _lib.load().spline_build(_p(x), _p(y), n, B, bc | (X_SHARED if shared else 0), _p(yp1), _p(ypn), _p(y2),
                                  _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_build")
    return y2[0] if squeeze else y2


def evaluate(x, y, y2, q, flags: int = 0, out=None, idx=None, want_idx: bool = True, stream=None):
    """Locate + evaluate queries q (B, m) on curves (B, n) (x may be (n,) shared by the batch).
    Returns (out, idx or None)."""
    x, y, shared, squeeze = _curves(x, y)
    y2, q = _as2d(y2), _as2d(q)
    B, n = y.shape
    m = q.shape[1]
    _check_curves(x, y, y2, q)
    if y2.shape != y.shape or q.dim() != 2 or q.shape[0] != B:
        raise ValueError("x, y, y2 must be (B, n) and q (B, m)")
    if shared:
        flags |= X_SHARED
    o = torch.empty_like(q) if out is None else _as2d(out)
    _check_buf(o, q.shape, q.dtype, q.device, "out")
    i = None
    if want_idx:
        i = torch.empty(q.shape, dtype=torch.int32, device=q.device) if idx is None else _as2d(idx)
        _check_buf(i, q.shape, torch.int32, q.device, "idx")
    rc = _lib.load().spline_eval(_p(x), _p(y), _p(y2), n, B, _p(q), m, _p(o), _p(i), flags, _DT[x.dtype],
                                 ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_eval")
    if squeeze:
        return o[0], (None if i is None else i[0])
    return o, i


def build_eval(x, y, q, bc: int = BC_NATURAL, yp1=None, ypn=None, flags: int = 0, want_y2: bool = True,
               y2=None, out=None, idx=None, want_idx: bool = True, stream=None):
    """Build + evaluate in one call (spline_build_eval; one fused kernel for n <= 128).
    Returns (y2 or None, out, idx or None); bitwise equal to build() then evaluate()."""
    x, y, shared, squeeze = _curves(x, y)
    q = _as2d(q)
    B, n = y.shape
    m = q.shape[1]
    yp1, ypn = _slopes(yp1, B, x), _slopes(ypn, B, x)
    _check_curves(x, y, q)
    if q.dim() != 2 or q.shape[0] != B:
        raise ValueError("x, y must be (B, n) and q (B, m)")
    if shared:
        flags |= X_SHARED
    _check_buf(yp1, (B,), x.dtype, x.device, "yp1")
    _check_buf(ypn, (B,), x.dtype, x.device, "ypn")
    z = None
    if want_y2:
        z = torch.empty_like(y) if y2 is None else _as2d(y2)
        _check_buf(z, y.shape, x.dtype, x.device, "y2")
    o = torch.empty_like(q) if out is None else _as2d(out)
    _check_buf(o, q.shape, q.dtype, q.device, "out")
    i = None
    if want_idx:
        i = torch.empty(q.shape, dtype=torch.int32, device=q.device) if idx is None else _as2d(idx)
        _check_buf(i, q.shape, torch.int32, q.device, "idx")
    rc = _lib.load().spline_build_eval(_p(x), _p(y), n, B, bc, _p(yp1), _p(ypn), _p(z), _p(q), m, _p(o), _p(i),
                                       flags, _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_build_eval")
    if squeeze:
        return (None if z is None else z[0]), o[0], (None if i is None else i[0])
    return z, o, i


def build_eval_host(x, y, q, bc: int = BC_NATURAL, yp1=None, ypn=None, flags: int = 0, want_y2: bool = True,
                    y2=None, out=None, idx=None, want_idx: bool = True, stream=None, sync: bool = True):
    """spline_build_eval_host: build + evaluate on HOST tensors (pinned for copy/compute overlap),
    chunked through the GPU.  Returns (y2 or None, out, idx or None) as CPU tensors; with
    sync=False the caller synchronises `stream` before reading them."""
    for t in (x, y, q):
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or not t.is_contiguous():
            raise ValueError("build_eval_host takes contiguous CPU tensors (pinned for overlap)")
    x, y, shared, squeeze = _curves(x, y)
    q = _as2d(q)
    B, n = y.shape
    m = q.shape[1]
    if q.shape[0] != B or y.dtype != x.dtype or q.dtype != x.dtype:
        raise ValueError("x, y must be (B, n) and q (B, m), one dtype")
    if shared:
        flags |= X_SHARED
    if x.dtype not in _DT:
        raise ValueError("dtype must be float32 or float64")
    pin = x.is_pinned()

    def host_like(shape, dtype):
        t = torch.empty(shape, dtype=dtype)
        return t.pin_memory() if pin else t

    yp1, ypn = _slopes(yp1, B, x, host=True), _slopes(ypn, B, x, host=True)
    _check_buf(yp1, (B,), x.dtype, None, "yp1", host=True)
    _check_buf(ypn, (B,), x.dtype, None, "ypn", host=True)
    z = (host_like(y.shape, x.dtype) if y2 is None else _as2d(y2)) if want_y2 else None
    o = host_like(q.shape, q.dtype) if out is None else _as2d(out)
    i = (host_like(q.shape, torch.int32) if idx is None else _as2d(idx)) if want_idx else None
    _check_buf(z, y.shape, x.dtype, None, "y2", host=True)
    _check_buf(o, q.shape, q.dtype, None, "out", host=True)
    _check_buf(i, q.shape, torch.int32, None, "idx", host=True)
    rc = _lib.load().spline_build_eval_host(_p(x), _p(y), n, B, bc, _p(yp1), _p(ypn), _p(z), _p(q), m, _p(o),
                                            _p(i), flags, _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_build_eval_host")
    if sync:
        (torch.cuda.current_stream() if stream is None else stream).synchronize()
    if squeeze:
        return (None if z is None else z[0]), o[0], (None if i is None else i[0])
    return z, o, i


def evaluate_ablation(x, y, y2, q, form: str, out=None, idx=None, stream=None):
    """spline_eval_ablation: the sorted-run eval kernel with one of the paper's interpolation
    variants (_lib.FORMS: record, splint_div, splint_mul, newint_orig, newint_noinv, noop)."""
    x, y, y2, q = _as2d(x), _as2d(y), _as2d(y2), _as2d(q)
    B, n = x.shape
    m = q.shape[1]
    _check_curves(x, y, y2, q)
    if y.shape != x.shape or y2.shape != x.shape or q.shape[0] != B:
        raise ValueError("x, y, y2 must be (B, n) and q (B, m)")
    if form not in _lib.FORMS:
        raise ValueError(f"form must be one of {sorted(_lib.FORMS)}")
    o = torch.empty_like(q) if out is None else _as2d(out)
    i = torch.empty(q.shape, dtype=torch.int32, device=q.device) if idx is None else _as2d(idx)
    _check_buf(o, q.shape, q.dtype, q.device, "out")
    _check_buf(i, q.shape, torch.int32, q.device, "idx")
    rc = _lib.load().spline_eval_ablation(_p(x), _p(y), _p(y2), n, B, _p(q), m, _p(o), _p(i), _lib.FORMS[form],
                                          _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_eval_ablation")
    return o, i


def gather_probe(x, y, y2, q, idx_in, mode: int, out=None, idx=None, stream=None):
    """spline_gather_probe (diagnostic): evaluate at the KNOWN intervals idx_in with no search --
    mode 0 gathers from x, y, y2; mode 1 through interval records.  Returns (out, idx)."""
    x, y, y2, q, idx_in = _as2d(x), _as2d(y), _as2d(y2), _as2d(q), _as2d(idx_in)
    B, n = x.shape
    m = q.shape[1]
    _check_curves(x, y, y2, q)
    if y.shape != x.shape or y2.shape != x.shape or q.shape[0] != B:
        raise ValueError("x, y, y2 must be (B, n) and q (B, m)")
    _check_buf(idx_in, q.shape, torch.int32, q.device, "idx_in")
    o = torch.empty_like(q) if out is None else _as2d(out)
    i = torch.empty(q.shape, dtype=torch.int32, device=q.device) if idx is None else _as2d(idx)
    _check_buf(o, q.shape, q.dtype, q.device, "out")
    _check_buf(i, q.shape, torch.int32, q.device, "idx")
    rc = _lib.load().spline_gather_probe(_p(x), _p(y), _p(y2), n, B, _p(q), m, _p(idx_in), _p(o), _p(i), mode,
                                         _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_gather_probe")
    return o, i


def status(stream=None) -> int:
    """Synchronise the stream, return and clear the data-error bits (STATUS_*)."""
    bits = ctypes.c_uint(0)
    rc = _lib.load().spline_status(ctypes.c_void_p(_stream(stream)), ctypes.byref(bits))
    _lib.check(rc, "spline_status")
    return bits.value


def spike_workspace(n: int, row_begin: int, row_end: int, dtype, device) -> torch.Tensor:
    nbytes = _lib.load().spline_spike_workspace_size(n, row_begin, row_end, _DT[dtype])
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def _check_spike(x, y, row_begin, row_end, yp1, ypn, workspace):
    _check_curves(x, y)
    if x.dim() != 1 or y.shape != x.shape:
        raise ValueError("the long-curve seam takes one curve: x, y of shape (n,)")
    n = x.shape[0]
    if not (0 <= row_begin < row_end <= n):
        raise ValueError("need 0 <= row_begin < row_end <= n")
    _check_buf(yp1, (1,), x.dtype, x.device, "yp1")
    _check_buf(ypn, (1,), x.dtype, x.device, "ypn")
    need = _lib.load().spline_spike_workspace_size(n, row_begin, row_end, _DT[x.dtype])
    if not (isinstance(workspace, torch.Tensor) and workspace.device == x.device and workspace.is_contiguous()
            and workspace.numel() * workspace.element_size() >= need):
        raise ValueError(f"workspace must be a contiguous device buffer of >= {need} bytes")
    return n


def spike_reduce(x, y, row_begin: int, row_end: int, bc: int, yp1, ypn, record, workspace, stream=None):
    n = _check_spike(x, y, row_begin, row_end, yp1, ypn, workspace)
    _check_buf(record, (6,), x.dtype, x.device, "record")
    rc = _lib.load().spline_spike_reduce(_p(x), _p(y), n, row_begin, row_end, bc, _p(yp1), _p(ypn), _p(record),
                                         _p(workspace), _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_spike_reduce")


def spike_finish(x, y, row_begin: int, row_end: int, bc: int, yp1, ypn, all_records, nranks: int, rank: int,
                 y2_shard, workspace, stream=None):
    n = _check_spike(x, y, row_begin, row_end, yp1, ypn, workspace)
    _check_buf(all_records, (6 * nranks,), x.dtype, x.device, "all_records")
    _check_buf(y2_shard, (row_end - row_begin,), x.dtype, x.device, "y2_shard")
    rc = _lib.load().spline_spike_finish(_p(x), _p(y), n, row_begin, row_end, bc, _p(yp1), _p(ypn),
                                         _p(all_records), nranks, rank, _p(y2_shard), _p(workspace),
                                         _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_spike_finish")


def spike_tile_rows(dtype) -> int:
    return int(_lib.load().spline_spike_tile_rows(_DT[dtype]))


def spike_tile_records(x, y, row_begin: int, row_end: int, bc: int, yp1, ypn, tile_records, workspace, stream=None):
    n = _check_spike(x, y, row_begin, row_end, yp1, ypn, workspace)
    ts = spike_tile_rows(x.dtype)
    _check_buf(tile_records, (-(-(row_end - row_begin) // ts), 6), x.dtype, x.device, "tile_records")
    rc = _lib.load().spline_spike_tile_records(_p(x), _p(y), n, row_begin, row_end, bc, _p(yp1), _p(ypn),
                                               _p(tile_records), _p(workspace), _DT[x.dtype],
                                               ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_spike_tile_records")


def spike_finish_tiles(x, y, bc: int, yp1, ypn, all_tile_records, y2, workspace, stream=None):
    n = _check_spike(x, y, 0, x.shape[-1], yp1, ypn, workspace)
    ts = spike_tile_rows(x.dtype)
    _check_buf(all_tile_records, (-(-n // ts), 6), x.dtype, x.device, "all_tile_records")
    _check_buf(y2, (n,), x.dtype, x.device, "y2")
    rc = _lib.load().spline_spike_finish_tiles(_p(x), _p(y), n, bc, _p(yp1), _p(ypn), _p(all_tile_records), _p(y2),
                                               _p(workspace), _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_spike_finish_tiles")


def build_dist(x, y, comm: int, bc: int = BC_NATURAL, yp1=None, ypn=None, y2_shard=None, stream=None):
    """spline_build_dist: this rank's rows of ONE long curve (x, y: the whole curve, (n,)) over an
    NCCL communicator given as its raw ncclComm_t handle (an int).  Rank r of G owns rows
    [r n / G, (r+1) n / G); returns (y2_shard, (row_begin, row_end)).  Collective: every rank calls."""
    _check_curves(x, y)
    if x.dim() != 1 or y.shape != x.shape:
        raise ValueError("build_dist takes one curve: x, y of shape (n,)")
    if not comm:
        raise ValueError("comm must be an initialised ncclComm_t handle")
    n = x.shape[0]
    yp1, ypn = _slopes(yp1, 1, x), _slopes(ypn, 1, x)
    _check_buf(yp1, (1,), x.dtype, x.device, "yp1")
    _check_buf(ypn, (1,), x.dtype, x.device, "ypn")
    nccl = _nccl_lib()
    G, r = ctypes.c_int(0), ctypes.c_int(0)
    if nccl.ncclCommCount(ctypes.c_void_p(comm), ctypes.byref(G)) or nccl.ncclCommUserRank(ctypes.c_void_p(comm),
                                                                                            ctypes.byref(r)):
        raise RuntimeError("ncclCommCount / ncclCommUserRank failed")
    rb, re = n * r.value // G.value, n * (r.value + 1) // G.value
    out = torch.empty(re - rb, dtype=x.dtype, device=x.device) if y2_shard is None else y2_shard
    _check_buf(out, (re - rb,), x.dtype, x.device, "y2_shard")
    rc = _lib.load().spline_build_dist(_p(x), _p(y), n, bc, _p(yp1), _p(ypn), _p(out), ctypes.c_void_p(comm),
                                       _DT[x.dtype], ctypes.c_void_p(_stream(stream)))
    _lib.check(rc, "spline_build_dist")
    return out, (rb, re)


_NCCL = None


def _nccl_lib():
    """The NCCL the process already uses (torch's), for communicator queries in the binding."""
    global _NCCL
    if _NCCL is None:
        import glob
        import os
        cands = []
        try:
            import nvidia.nccl
            for d in list(getattr(nvidia.nccl, "__path__", [])):  # a namespace package
                cands += glob.glob(os.path.join(d, "lib", "libnccl.so*"))
        except ImportError:
            pass
        cands.append("libnccl.so.2")
        for c in cands:
            try:
                _NCCL = ctypes.CDLL(c)
                break
            except OSError:
                continue
        if _NCCL is None:
            raise RuntimeError("libnccl.so.2 not found")
    return _NCCL


def version() -> str:
    return _lib.load().spline_version().decode()
