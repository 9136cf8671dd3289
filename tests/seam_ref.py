"""Independent numpy model of the SPIKE seam contract of include/spline.h (test-only).

Used to exercise the multi-rank orchestration of paper_2001_09253_b200.dist on CPU (gloo):
the record of a row block [p, q] is (Gp, Vp, Wp, Gq, Vq, Wq) with
y_p = Gp - Vp y_{p-1} - Wp y_{q+1},  y_q = Gq - Vq y_{p-1} - Wq y_{q+1}
(SURVEY.md Appendix A), computed here by dense solves of the block."""
import numpy as np
import torch

import refmath


class SeamRefOps:
    def __init__(self, x, y, bc, yp1=0.0, ypn=0.0):
        M, d = refmath.dense_system(x, y, bc, yp1, ypn)
        self.M = np.array(M, dtype=np.float64)
        self.d = np.array(d, dtype=np.float64)

    def _block(self, rb, re):
        T = self.M[rb:re, rb:re]
        a = self.M[rb, rb - 1] if rb > 0 else 0.0
        c = self.M[re - 1, re] if re < self.M.shape[0] else 0.0
        return T, a, c

    def workspace(self, n, rb, re, dtype, device):
        return torch.empty(0)

    def reduce(self, x, y, rb, re, bc, yp1, ypn, record, ws):
        T, a, c = self._block(rb, re)
        m = re - rb
        e1 = np.zeros(m); e1[0] = a
        el = np.zeros(m); el[-1] = c
        G = np.linalg.solve(T, self.d[rb:re])
        V = np.linalg.solve(T, e1)
        W = np.linalg.solve(T, el)
        record.copy_(torch.tensor([G[0], V[0], W[0], G[-1], V[-1], W[-1]], dtype=record.dtype))

    def finish(self, x, y, rb, re, bc, yp1, ypn, all_records, world, rank, y2_shard, ws):
        R = all_records.reshape(world, 6).numpy()
        # unknowns u = (F_0, L_0, F_1, L_1, ...): first and last row of every rank block
        A = np.eye(2 * world)
        rhs = np.zeros(2 * world)
        for r in range(world):
            Gp, Vp, Wp, Gq, Vq, Wq = R[r]
            for row, (Gv, Vv, Wv) in ((2 * r, (Gp, Vp, Wp)), (2 * r + 1, (Gq, Vq, Wq))):
                rhs[row] = Gv
                if r > 0:
                    A[row, 2 * r - 1] += Vv   # y_{p-1} = last row of rank r-1
                if r < world - 1:
                    A[row, 2 * r + 2] += Wv   # y_{q+1} = first row of rank r+1
        u = np.linalg.solve(A, rhs)
        L = u[2 * rank - 1] if rank > 0 else 0.0
        Rv = u[2 * rank + 2] if rank < world - 1 else 0.0
        T, a, c = self._block(rb, re)
        b = self.d[rb:re].copy()
        b[0] -= a * L
        b[-1] -= c * Rv
        y2_shard.copy_(torch.tensor(np.linalg.solve(T, b), dtype=y2_shard.dtype))

    # ---- recompute instead of communicate: tiles of TILE rows act as the "ranks" of the seam
    TILE = 1000

    def tile_rows(self, dtype):
        return self.TILE

    def tile_records(self, x, y, rb, re, bc, yp1, ypn, recs, ws):
        for k, t0 in enumerate(range(rb, re, self.TILE)):
            self.reduce(x, y, t0, min(t0 + self.TILE, re), bc, yp1, ypn, recs[k], ws)

    def finish_tiles(self, x, y, bc, yp1, ypn, all_recs, y2, ws):
        n = y2.shape[0]
        nt = all_recs.shape[0]
        flat = all_recs.reshape(-1).cpu()
        for t in range(nt):
            rb, re = t * self.TILE, min((t + 1) * self.TILE, n)
            out = torch.empty(re - rb, dtype=y2.dtype)
            self.finish(x, y, rb, re, bc, yp1, ypn, flat, nt, t, out, ws)
            y2[rb:re] = out
