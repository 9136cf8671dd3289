// build_thomas.cuh -- K1: batched Thomas solve, one thread per curve (short curves, n <= 128).
//
// Method: the paper's new_second_derivative sweep -- forward elimination
// c'_j, d'_j, d' stored where y2 goes, back-substitution
// y2_j = d'_j - c'_j y2_{j+1} -- with the rows of Eq. init_val,
// the clamped start row and the clamped end row of P:1017-1018.
//
// Layout: global x/y/y2 are curve-major [B][n].  A CTA owns CPB consecutive curves: it
// stages their x and y with coalesced loads into shared memory tiles whose per-curve
// stride S = n|1 is odd, so that at sweep step j the 32 lanes (32 curves) read
// 32 distinct banks -- the "interleaved SoA" access of the north star, realised
// on-chip.  c' overwrites x and d' (then y2) overwrites y in place; the y2 tile is then
// written back with coalesced stores.  Validation (strictly increasing, finite knots,
// finite values and slopes) is fused into the sweep.
#pragma once
#include "common.cuh"

namespace fs {

constexpr int kK1Threads = 256;

// blockDim = 256 threads stage the tile (all loads in flight at once); the first CPB
// threads (one per curve) run the sweeps.
template <typename T>
__global__ void __launch_bounds__(kK1Threads, 4) k1_thomas_batched(const T *__restrict__ x, const T *__restrict__ y,
                                                                int n, int64_t batch, int bc,
                                                                const T *__restrict__ yp1, const T *__restrict__ ypn,
                                                                T *__restrict__ y2, int S, int CPB, FastDiv divn) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T *X = reinterpret_cast<T *>(smem_raw);
  T *Y = X + (size_t)CPB * S;

  const int64_t c0 = (int64_t)blockIdx.x * CPB;
  const int nc = (int)min64(CPB, batch - c0);
  const int tot = nc * n;
  const T *xb = x + c0 * n;
  const T *yb = y + c0 * n;

  // Stage: flat coalesced loads (UL per array per thread in flight), scattered into the
  // odd-stride tiles.
  constexpr int UL = sizeof(T) == 4 ? 16 : 8;
  for (int base = threadIdx.x; base < tot; base += UL * kK1Threads) {
    T vx[UL], vy[UL];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int e = base + u * kK1Threads;
      if (e < tot) {
        vx[u] = ld_stream(xb + e);
        vy[u] = ld_stream(yb + e);
      }
    }
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int e = base + u * kK1Threads;
      if (e < tot) {
        const int c = (int)divn.div((uint32_t)e);
        const int j = e - c * n;
        X[c * S + j] = vx[u];
        Y[c * S + j] = vy[u];
      }
    }
  }
  __syncthreads();

  const int t = threadIdx.x;
  if (t < nc) {
    T *Xc = X + t * S;
    T *Yc = Y + t * S;
    const int64_t cg = c0 + t;
    bool ok = true;

    T xo = Xc[0], yo = Yc[0];
    T xn = Xc[1], yn = Yc[1];
    ok = ok && finite(xo) && finite(yo) && finite(yn) && (xn > xo);
    T hprev = xn - xo;
    T ddprev = (yn - yo) / hprev;
    T cp, dp;
    if (bc & 1) {  // clamped start: c'_0 = 1/2, d'_0 = 3 (dd_0 - y'_0) / h_0
      const T s = yp1[cg];
      ok = ok && finite(s);
      cp = T(0.5);
      dp = T(3) * (ddprev - s) / hprev;
    } else {  // natural start
      cp = T(0);
      dp = T(0);
    }
    Xc[0] = cp;
    Yc[0] = dp;
    // Forward substitution over the interior rows; two loads per step.
    for (int j = 1; j < n - 1; ++j) {
      xo = xn;
      yo = yn;
      xn = Xc[j + 1];
      yn = Yc[j + 1];
      ok = ok && (xn > xo) && finite(yn);
      const T h = xn - xo;
      const T dd = (yn - yo) / h;
      const T inv = T(1) / (T(2) * (hprev + h) - hprev * cp);
      dp = (T(6) * (dd - ddprev) - hprev * dp) * inv;
      cp = h * inv;
      Xc[j] = cp;
      Yc[j] = dp;
      hprev = h;
      ddprev = dd;
    }
    ok = ok && finite(xn);
    // End row.
    if (bc & 2) {  // clamped end: a = h_{n-2}, b = 2 h_{n-2}, d = 6 (y'_{n-1} - dd_{n-2})
      const T e = ypn[cg];
      ok = ok && finite(e);
      const T inv = T(1) / (T(2) * hprev - hprev * cp);
      dp = (T(6) * (e - ddprev) - hprev * dp) * inv;
    } else {
      dp = T(0);
    }
    Yc[n - 1] = dp;
    // Backward substitution.
    for (int j = n - 2; j >= 0; --j) {
      dp = Yc[j] - Xc[j] * dp;
      Yc[j] = dp;
    }
    if (!ok) {
      const T nanv = qnan<T>();
      for (int j = 0; j < n; ++j) Yc[j] = nanv;
    }
    raise_status_warp(!ok, kBadKnots);
  }
  __syncthreads();

  T *y2b = y2 + c0 * n;
  for (int e = threadIdx.x; e < tot; e += kK1Threads) {
    const int c = (int)divn.div((uint32_t)e);
    const int j = e - c * n;
    y2b[e] = Y[c * S + j];
  }
}

}  // namespace fs
