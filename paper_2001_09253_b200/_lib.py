"""ctypes binding of libfastspline.so (include/spline.h).  Argument marshalling only.

The library is REQUIRED: if it is missing or fails to load, every op raises.  There
is no CPU or eager-PyTorch fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

SPLINE_F32, SPLINE_F64 = 0, 1
SPLINE_OK, SPLINE_EINVAL, SPLINE_ECUDA, SPLINE_ENOMEM, SPLINE_ENCCL = 0, -1, -2, -3, -4
BC_NATURAL, BC_CLAMP_START, BC_CLAMP_END, BC_CLAMPED = 0, 1, 2, 3
Q_SORTED, X_UNIFORM, PATH_FUSED, PATH_SPLIT, NO_BUCKET, X_SHARED = 1, 2, 4, 8, 16, 32
STATUS_BAD_KNOTS, STATUS_Q_OUT_OF_RANGE = 1, 2
FORMS = {"record": 0, "splint_div": 1, "splint_mul": 2, "newint_orig": 3, "newint_noinv": 4, "noop": 5}

_ERR = {SPLINE_EINVAL: "SPLINE_EINVAL (invalid argument)", SPLINE_ECUDA: "SPLINE_ECUDA (CUDA error)",
        SPLINE_ENOMEM: "SPLINE_ENOMEM (out of device memory)", SPLINE_ENCCL: "SPLINE_ENCCL (NCCL unavailable or failed)"}

# name -> (restype, argtypes)
_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
SIGNATURES = {
    "spline_build": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _vp]),
    "spline_eval": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _i32, _i32, _vp]),
    "spline_build_eval": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _vp]),
    "spline_build_eval_host": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i32, _i32, _vp]),
    "spline_eval_ablation": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _i32, _i32, _vp]),
    "spline_gather_probe": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _i32, _i32, _vp]),
    "spline_build_f32": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "spline_build_f64": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "spline_eval_f32": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _i32, _vp]),
    "spline_eval_f64": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _i32, _vp]),
    "spline_status": (_i32, [_vp, ctypes.POINTER(ctypes.c_uint)]),
    "spline_spike_workspace_size": (_sz, [_i64, _i64, _i64, _i32]),
    "spline_spike_reduce": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp]),
    "spline_spike_finish": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _i32,
                                   _vp]),
    "spline_spike_tile_rows": (_i64, [_i32]),
    "spline_spike_tile_records": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp]),
    "spline_spike_finish_tiles": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "spline_build_dist": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp]),
    "spline_build_dist_f32": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "spline_build_dist_f64": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "spline_version": (ctypes.c_char_p, []),
}

_lib = None


def lib_path() -> str:
    return _build.LIB


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError(f"libfastspline.so not built ({path}); run __graft_entry__.build() "
                               "or python -m paper_2001_09253_b200._build -- there is no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != SPLINE_OK:
        raise RuntimeError(f"{what} failed: {_ERR.get(rc, rc)}")
