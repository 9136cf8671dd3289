"""Host-side checks of the C ABI (-m "not gpu"): the library loads, exports every symbol
that include/spline.h declares, and rejects bad arguments synchronously (no GPU needed:
argument errors return before any CUDA call)."""
import ctypes
import os
import re

import pytest

from paper_2001_09253_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "spline.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spline_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for required in ["spline_build", "spline_eval", "spline_build_f32", "spline_build_f64", "spline_eval_f32",
                     "spline_eval_f64", "spline_status", "spline_spike_reduce", "spline_spike_finish",
                     "spline_build_dist", "spline_build_dist_f32", "spline_build_dist_f64"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"binding lacks {name}"


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.lib_path()} 2>&1").read()
    assert "sm_100a" in out


def _build(*args):
    return _lib.load().spline_build(*args)


def test_einval_build():
    p = ctypes.c_void_p(16)
    F64 = _lib.SPLINE_F64
    assert _build(p, p, 2, 1, 0, None, None, p, F64, None) == _lib.SPLINE_EINVAL          # n < 3
    assert _build(p, p, 8, -1, 0, None, None, p, F64, None) == _lib.SPLINE_EINVAL         # batch < 0
    assert _build(p, p, 8, 1, 4, None, None, p, F64, None) == _lib.SPLINE_EINVAL          # bad bc
    assert _build(p, p, 8, 1, 1, None, None, p, F64, None) == _lib.SPLINE_EINVAL          # clamped, no yp1
    assert _build(p, p, 8, 1, 2, p, None, p, F64, None) == _lib.SPLINE_EINVAL             # clamped end, no ypn
    assert _build(None, p, 8, 1, 0, None, None, p, F64, None) == _lib.SPLINE_EINVAL       # NULL x
    assert _build(p, p, 8, 1, 0, None, None, p, 7, None) == _lib.SPLINE_EINVAL            # bad dtype
    assert _build(p, p, 1 << 31, 1, 0, None, None, p, F64, None) == _lib.SPLINE_EINVAL    # n >= 2^31
    assert _build(None, None, 8, 0, 0, None, None, None, F64, None) == _lib.SPLINE_OK     # empty batch


def test_einval_eval():
    lib = _lib.load()
    p = ctypes.c_void_p(16)
    F32 = _lib.SPLINE_F32
    assert lib.spline_eval(p, p, p, 2, 1, p, 4, p, None, 0, F32, None) == _lib.SPLINE_EINVAL   # n < 3
    assert lib.spline_eval(p, p, p, 8, 1, p, -1, p, None, 0, F32, None) == _lib.SPLINE_EINVAL  # m < 0
    assert lib.spline_eval(p, p, p, 8, 1, p, 4, p, None, 8, F32, None) == _lib.SPLINE_EINVAL   # unknown flag
    assert lib.spline_eval(p, p, p, 8, 1, p, 4, p, None, 64, F32, None) == _lib.SPLINE_EINVAL  # unknown flag
    assert lib.spline_eval(p, None, p, 8, 1, p, 4, p, None, 0, F32, None) == _lib.SPLINE_EINVAL  # NULL y
    assert lib.spline_eval(None, None, None, 8, 1, None, 0, None, None, 0, F32, None) == _lib.SPLINE_OK  # m == 0
    assert lib.spline_eval(None, None, None, 8, 0, None, 9, None, None, 0, F32, None) == _lib.SPLINE_OK  # B == 0


def test_einval_spike():
    lib = _lib.load()
    p = ctypes.c_void_p(16)
    F64 = _lib.SPLINE_F64
    assert lib.spline_spike_reduce(p, p, 100, 50, 40, 0, None, None, p, p, F64, None) == _lib.SPLINE_EINVAL
    assert lib.spline_spike_reduce(p, p, 100, 0, 101, 0, None, None, p, p, F64, None) == _lib.SPLINE_EINVAL
    assert lib.spline_spike_finish(p, p, 100, 0, 50, 0, None, None, p, 2, 2, p, p, F64, None) == _lib.SPLINE_EINVAL
    assert lib.spline_spike_workspace_size(1 << 26, 0, 1 << 26, F64) > 0


def test_no_oracle_in_product_package():
    """The product path never imports, loads or calls the oracle."""
    pkg = os.path.join(os.path.dirname(HEADER), "..", "paper_2001_09253_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f


def test_api_rejects_cpu_tensors():
    import torch
    from paper_2001_09253_b200 import api
    with pytest.raises(ValueError):
        api.build(torch.zeros(8, dtype=torch.float64), torch.zeros(8, dtype=torch.float64))


@pytest.mark.parametrize("entry", ["spline_build_eval", "spline_build_eval_host"])
def test_einval_build_eval(entry):
    lib = _lib.load()
    p = ctypes.c_void_p(16)
    F32, E = _lib.SPLINE_F32, _lib.SPLINE_EINVAL
    f = getattr(lib, entry)
    assert f(p, p, 2, 1, 0, None, None, p, p, 4, p, None, 0, F32, None) == E      # n < 3
    assert f(p, p, 8, 1, 0, None, None, p, p, -1, p, None, 0, F32, None) == E     # m < 0
    assert f(p, p, 8, 1, 1, None, None, p, p, 4, p, None, 0, F32, None) == E      # clamped, no yp1
    assert f(p, p, 8, 1, 0, None, None, p, None, 4, p, None, 0, F32, None) == E   # NULL q with m > 0
    assert f(p, p, 8, 1, 0, None, None, p, p, 4, None, None, 0, F32, None) == E   # NULL out
    assert f(p, p, 8, 1, 0, None, None, p, p, 4, p, None, 16, F32, None) == E     # unknown flag
    assert f(p, p, 8, 1, 5, None, None, p, p, 4, p, None, 0, F32, None) == E      # bad bc
    assert f(None, p, 8, 1, 0, None, None, p, p, 4, p, None, 0, F32, None) == E   # NULL x
    assert f(p, p, 8, 1, 0, None, None, p, p, 4, p, None, 12, F32, None) == E     # both path hints
    assert f(None, None, 8, 0, 0, None, None, None, None, 4, None, None, 0, F32, None) == _lib.SPLINE_OK


def test_einval_gather_probe():
    lib = _lib.load()
    p = ctypes.c_void_p(16)
    F64, E = _lib.SPLINE_F64, _lib.SPLINE_EINVAL
    assert lib.spline_gather_probe(p, p, p, 8, 1, p, 4, p, p, p, 2, F64, None) == E    # bad mode
    assert lib.spline_gather_probe(p, p, p, 2, 1, p, 4, p, p, p, 0, F64, None) == E    # n < 3
    assert lib.spline_gather_probe(p, p, p, 8, 1, p, 4, None, p, p, 0, F64, None) == E  # NULL idx_in
    assert lib.spline_gather_probe(None, None, None, 8, 0, None, 4, None, None, None, 0, F64, None) == _lib.SPLINE_OK


def test_einval_build_dist():
    lib = _lib.load()
    p = ctypes.c_void_p(16)
    F64, E = _lib.SPLINE_F64, _lib.SPLINE_EINVAL
    assert lib.spline_build_dist(p, p, 100, 0, None, None, p, None, F64, None) == E   # NULL communicator
    assert lib.spline_build_dist(p, p, 2, 0, None, None, p, p, F64, None) == E        # n < 3
    assert lib.spline_build_dist(p, p, 100, 1, None, None, p, p, F64, None) == E      # clamped, no yp1
    assert lib.spline_build_dist(p, p, 100, 0, None, None, p, p, 9, None) == E        # bad dtype
    assert lib.spline_build_dist(None, p, 100, 0, None, None, p, p, F64, None) == E   # NULL x


def test_build_dist_enccl_without_nccl():
    """NCCL is resolved at run time: with none loadable the distributed build returns SPLINE_ENCCL
    (before any CUDA or NCCL call), instead of failing to load the library."""
    import subprocess
    import sys
    code = ("import ctypes; from paper_2001_09253_b200 import _lib; p = ctypes.c_void_p(16); "
            "print(_lib.load().spline_build_dist(p, p, 100, 0, None, None, p, p, _lib.SPLINE_F64, None))")
    env = dict(os.environ, SPLINE_NCCL_LIB="/nonexistent/libnccl.so.2")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert int(out.stdout.strip().splitlines()[-1]) == _lib.SPLINE_ENCCL
