"""The README example, run as a check: PYTHONPATH=. python tools/readme_example.py"""

import torch
from paper_2001_09253_b200 import api

x = torch.cumsum(torch.rand(1024, 64, device="cuda") + 0.1, dim=1)   # [B][n] knots, increasing
y = torch.randn(1024, 64, device="cuda")
q = x[:, :1] + torch.rand(1024, 256, device="cuda") * (x[:, -1:] - x[:, :1])
y2, out, idx = api.build_eval(x, y, q, api.BC_NATURAL)               # device arrays, one call
assert api.status() == 0                                               # async data-error bits
y2h, outh, idxh = api.build_eval_host(x.cpu().pin_memory(), y.cpu().pin_memory(),
                                      q.cpu().pin_memory())            # host arrays, copies overlapped
print("ok", out.shape, outh.shape, bool(torch.equal(out.cpu(), outh)))
