"""spline_build_dist through a real NCCL communicator (1 rank: one GPU on the box) -- the C-ABI
entry of the multi-GPU long-curve build; multi-rank orchestration is
covered by the emulated-rank seam tests and the gloo tests."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2001_09253_b200 import workloads

pytestmark = pytest.mark.gpu


class _UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_09253_b200 import api
    torch.cuda.set_device(0)
    nccl = api._nccl_lib()
    uid = _UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    c = ctypes.c_void_p()
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _UniqueId, ctypes.c_int]
    assert nccl.ncclCommInitRank(ctypes.byref(c), 1, uid, 0) == 0
    yield c.value
    nccl.ncclCommDestroy(c)


@pytest.mark.parametrize("n,bc,dt", [(1 << 18, 0, np.float64), (300001, 3, np.float64), (70000, 1, np.float32)])
def test_build_dist_one_rank_nccl(comm, n, bc, dt):
    from paper_2001_09253_b200 import api
    wl = workloads.generate(5, n=n, m=16)
    x, y = parity.to_dev(wl.x[0].astype(dt)), parity.to_dev(wl.y[0].astype(dt))
    api.status()
    y2, (rb, re) = api.build_dist(x, y, comm, bc, 0.25, -0.5)
    torch.cuda.synchronize()
    assert api.status() == 0 and (rb, re) == (0, n)
    ref, _ = oracle.build_y2(x.cpu().numpy(), y.cpu().numpy(), bc, [0.25], [-0.5])
    assert parity.y2_rel_err(y2.cpu().numpy()[None], ref[None]).max() <= parity.tol_for(dt)
    # bitwise the two-phase seam with G = 1 (reduce -> the record itself -> finish)
    s0 = torch.full((1,), 0.25, dtype=x.dtype, device=x.device)
    s1 = torch.full((1,), -0.5, dtype=x.dtype, device=x.device)
    ws = api.spike_workspace(n, 0, n, x.dtype, x.device)
    rec = torch.empty(6, dtype=x.dtype, device=x.device)
    api.spike_reduce(x, y, 0, n, bc, s0, s1, rec, ws)
    y2s = torch.empty(n, dtype=x.dtype, device=x.device)
    api.spike_finish(x, y, 0, n, bc, s0, s1, rec, 1, 0, y2s, ws)
    assert torch.equal(y2.view(torch.int8), y2s.view(torch.int8))


def test_build_dist_bad_knots_status(comm):
    from paper_2001_09253_b200 import api
    wl = workloads.generate(5, n=50000, m=16)
    wl.x[0, 1234] = wl.x[0, 1233]
    x, y = parity.to_dev(wl.x[0]), parity.to_dev(wl.y[0])
    api.status()
    y2, _ = api.build_dist(x, y, comm)
    assert api.status() == api.STATUS_BAD_KNOTS
    assert torch.isnan(y2).all()
