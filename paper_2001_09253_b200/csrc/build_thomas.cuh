// build_thomas.cuh -- K1: batched Thomas solves for short curves (n <= 128).
//
// Method: the paper's new_second_derivative sweep -- forward elimination
// c'_j, d'_j stored in place, back-substitution
// y2_j = d'_j - c'_j y2_{j+1} -- on the rows of Eq. init_val, the
// clamped start row and the clamped end row of P:1017-1018.
//
// K1  (k1_thomas_babe, 3 <= n <= 128): two threads per curve run the same elimination
//     from both ends ("burn at both ends"): the top thread eliminates rows 0..k-1 downward
//     (c'_j, d'_j), the bottom thread rows n-1..k+1 upward (a''_j, d''_j), they meet at the
//     middle row k = n/2 through one shuffle, y2_k = (d_k - a_k d'_{k-1} - c_k d''_{k+1}) /
//     (b_k - a_k c'_{k-1} - c_k a''_{k+1}), and each back-substitutes outward.  Same flop
//     count as Thomas, half the dependency chain.  The CTA stages its curves' x, y with
//     coalesced loads into shared-memory tiles of odd stride S = n|1 (at a given step the
//     lanes of a warp hit distinct banks -- the north star's interleaved SoA, realised
//     on-chip); coefficients and y2 overwrite x, y in place; y2 leaves with coalesced stores.
// K1r (k1_thomas_regs, n <= 16): one thread per curve, everything in registers, 16-byte
//     vector loads/stores -- the few-control-point regime (BASELINE cfg3).
// Validation (strictly increasing finite knots, finite values and slopes) is
// fused: a bad curve's y2 is all NaN and SPLINE_STATUS_BAD_KNOTS is raised.
#pragma once
#include "common.cuh"

namespace fs {

constexpr int kK1Threads = 256;

// The two-ended sweep of one CTA tile: curve t = threadIdx.x/2 of the tile lives at
// Xc = X + t*S, Yc = Y + t*S (odd stride S); on return Yc holds y2 (or NaN).
template <typename T>
__device__ __forceinline__ void babe_tile(T *X, T *Y, int S, int n, int nc, int64_t c0, int bc,
                                          const T *__restrict__ yp1, const T *__restrict__ ypn) {
  const int t = threadIdx.x >> 1;       // curve within the CTA
  const bool top = (threadIdx.x & 1) == 0;
  const bool act = t < nc;              // pairs are lane-adjacent, so shuffles stay in-warp
  const int k = n >> 1;                 // meeting row, 1 <= k <= n-2
  T *Xc = X + (act ? t : 0) * S;
  T *Yc = Y + (act ? t : 0) * S;
  const int64_t cg = c0 + t;
  bool ok = true;
  T hb = T(0), ddb = T(0), cpb = T(0), dpb = T(0);  // this side's values at the seam
  if (act) {
    if (top) {
      // rows 0 .. k-1, downward
      T xo = Xc[0], yo = Yc[0];
      T xn = Xc[1], yn = Yc[1];
      ok = finite(xo) && finite(yo) && finite(xn) && finite(yn) && (xn > xo);
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
      for (int j = 1; j < k; ++j) {
        xo = xn;
        yo = yn;
        xn = Xc[j + 1];
        yn = Yc[j + 1];
        ok = ok && (xn > xo) && finite(xn) && finite(yn);
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
      hb = hprev;  // h_{k-1}
      ddb = ddprev;
      cpb = cp;    // c'_{k-1}
      dpb = dp;    // d'_{k-1}
    } else {
      // rows n-1 .. k+1, upward: y2_j = d''_j - a''_j y2_{j-1}
      T xo = Xc[n - 1], yo = Yc[n - 1];
      T xn = Xc[n - 2], yn = Yc[n - 2];
      ok = finite(xo) && finite(yo) && finite(xn) && finite(yn) && (xo > xn);
      T hnext = xo - xn;            // h_{n-2}
      T ddnext = (yo - yn) / hnext; // dd_{n-2}
      T ap, dp;
      if (bc & 2) {  // clamped end: a = h, b = 2h, d = 6 (y'_{n-1} - dd_{n-2})
        const T e = ypn[cg];
        ok = ok && finite(e);
        ap = T(0.5);
        dp = T(3) * (e - ddnext) / hnext;
      } else {  // natural end
        ap = T(0);
        dp = T(0);
      }
      Xc[n - 1] = ap;
      Yc[n - 1] = dp;
      for (int j = n - 2; j > k; --j) {
        xo = xn;
        yo = yn;
        xn = Xc[j - 1];
        yn = Yc[j - 1];
        ok = ok && (xo > xn) && finite(xn) && finite(yn);
        const T h = xo - xn;          // h_{j-1}
        const T dd = (yo - yn) / h;   // dd_{j-1}
        // row j: a = h_{j-1}, b = 2(h_{j-1} + h_j), c = h_j, d = 6(dd_j - dd_{j-1})
        const T inv = T(1) / (T(2) * (h + hnext) - hnext * ap);
        dp = (T(6) * (ddnext - dd) - hnext * dp) * inv;
        ap = h * inv;
        Xc[j] = ap;
        Yc[j] = dp;
        hnext = h;
        ddnext = dd;
      }
      hb = hnext;   // h_k
      ddb = ddnext; // dd_k
      cpb = ap;     // a''_{k+1}
      dpb = dp;     // d''_{k+1}
    }
  }
  // meet at row k: a_k = h_{k-1}, b_k = 2(h_{k-1} + h_k), c_k = h_k, d_k = 6(dd_k - dd_{k-1})
  const T o_h = __shfl_xor_sync(0xffffffffu, hb, 1);
  const T o_dd = __shfl_xor_sync(0xffffffffu, ddb, 1);
  const T o_cp = __shfl_xor_sync(0xffffffffu, cpb, 1);
  const T o_dp = __shfl_xor_sync(0xffffffffu, dpb, 1);
  const bool o_ok = __shfl_xor_sync(0xffffffffu, ok, 1);
  if (act) {
    ok = ok && o_ok;
    const T hk1 = top ? hb : o_h, ddk1 = top ? ddb : o_dd, cT = top ? cpb : o_cp, dT = top ? dpb : o_dp;
    const T hk = top ? o_h : hb, ddk = top ? o_dd : ddb, aB = top ? o_cp : cpb, dB = top ? o_dp : dpb;
    const T yk = (T(6) * (ddk - ddk1) - hk1 * dT - hk * dB) / (T(2) * (hk1 + hk) - hk1 * cT - hk * aB);
    T yv = yk;
    if (top) {
      Yc[k] = yk;
      for (int j = k - 1; j >= 0; --j) {
        yv = Yc[j] - Xc[j] * yv;
        Yc[j] = yv;
      }
    } else {
      for (int j = k + 1; j < n; ++j) {
        yv = Yc[j] - Xc[j] * yv;
        Yc[j] = yv;
      }
    }
    if (!ok) {  // both threads of the pair see the same ok
      const T nanv = qnan<T>();
      for (int j = top ? 0 : k + 1; j < (top ? k + 1 : n); ++j) Yc[j] = nanv;
    }
  }
  raise_status_warp(act && !ok && top, kBadKnots);

}

template <typename T>
__global__ void __launch_bounds__(kK1Threads) k1_thomas_babe(const T *__restrict__ x, const T *__restrict__ y, int n,
                                                             int64_t batch, int bc, const T *__restrict__ yp1,
                                                             const T *__restrict__ ypn, T *__restrict__ y2, int S,
                                                             FastDiv divn) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int CPB = blockDim.x / 2;  // blockDim = 2 x curves per CTA (<= 256)
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
  const int NT = blockDim.x;
  for (int base = threadIdx.x; base < tot; base += UL * NT) {
    T vx[UL], vy[UL];
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int e = base + u * NT;
      if (e < tot) {
        vx[u] = ld_stream(xb + e);
        vy[u] = ld_stream(yb + e);
      }
    }
#pragma unroll
    for (int u = 0; u < UL; ++u) {
      const int e = base + u * NT;
      if (e < tot) {
        const int c = (int)divn.div((uint32_t)e);
        const int j = e - c * n;
        X[c * S + j] = vx[u];
        Y[c * S + j] = vy[u];
      }
    }
  }
  __syncthreads();

  babe_tile(X, Y, S, n, nc, c0, bc, yp1, ypn);
  __syncthreads();

  T *y2b = y2 + c0 * n;
  for (int e = threadIdx.x; e < tot; e += NT) {
    const int c = (int)divn.div((uint32_t)e);
    const int j = e - c * n;
    y2b[e] = Y[c * S + j];
  }
}


// K1 pipelined: persistent CTAs.  One raw stage receives a tile's x, y by TMA bulk copy;
// it is transposed into the odd-stride tiles at once, and the next tile's copy is issued
// into it before the sweep starts, so the load of tile i+1 overlaps the sweep and the
// stores of tile i.  Requires n*sizeof(T) % 16 == 0 and 16-byte aligned x, y (else
// k1_thomas_babe).
template <typename T>
__global__ void __launch_bounds__(kK1Threads) k1_thomas_pipe(const T *__restrict__ x, const T *__restrict__ y, int n,
                                                             int64_t batch, int bc, const T *__restrict__ yp1,
                                                             const T *__restrict__ ypn, T *__restrict__ y2, int S,
                                                             int64_t ntiles, FastDiv divn) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int CPB = blockDim.x / 2;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
  T *Xr = reinterpret_cast<T *>(smem_raw + 16);
  T *Yr = Xr + (size_t)CPB * n;
  T *X = reinterpret_cast<T *>(smem_raw + 16 + ((2 * (size_t)CPB * n * sizeof(T) + 15) & ~(size_t)15));
  T *Y = X + (size_t)CPB * S;
  const int64_t G = gridDim.x;
  auto issue = [&](int64_t it) {  // thread 0 only
    if (it >= ntiles) return;
    const int64_t c0 = it * CPB;
    const int nc = (int)min64(CPB, batch - c0);
    const uint32_t bytes = (uint32_t)((size_t)nc * n * sizeof(T));
    mbar_expect_tx(bar, 2 * bytes);
    bulk_g2s(Xr, x + c0 * n, bytes, bar);
    bulk_g2s(Yr, y + c0 * n, bytes, bar);
  };
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  int64_t it = blockIdx.x;
  if (threadIdx.x == 0) issue(it);
  uint32_t phase = 0u;
  for (; it < ntiles; it += G) {
    const int64_t c0 = it * CPB;
    const int nc = (int)min64(CPB, batch - c0);
    const int tot = nc * n;
    mbar_wait(bar, phase);
    phase ^= 1u;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {  // to the odd-stride tiles
      const int c = (int)divn.div((uint32_t)e);
      const int j = e - c * n;
      X[c * S + j] = Xr[e];
      Y[c * S + j] = Yr[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) issue(it + G);  // raw stage consumed: next tile in flight
    babe_tile(X, Y, S, n, nc, c0, bc, yp1, ypn);
    __syncthreads();
    T *y2b = y2 + c0 * n;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      const int c = (int)divn.div((uint32_t)e);
      const int j = e - c * n;
      y2b[e] = Y[c * S + j];
    }
    __syncthreads();
  }
}

// K1r: one thread per curve, n <= NMAX, all in registers.
template <typename T, int NMAX>
__global__ void __launch_bounds__(256) k1_thomas_regs(const T *__restrict__ x, const T *__restrict__ y, int n,
                                                      int64_t batch, int bc, const T *__restrict__ yp1,
                                                      const T *__restrict__ ypn, T *__restrict__ y2, int vec) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= batch) return;
  T xv[NMAX], yv[NMAX];
  const T *xc = x + c * n, *yc = y + c * n;
  constexpr int VW = 16 / sizeof(T);
  if (vec) {  // n % VW == 0 and 16-byte aligned rows
    using VT = typename Vec16<T>::V;
#pragma unroll
    for (int j = 0; j < NMAX; j += VW) {
      if (j < n) {
        const VT a = __ldcs(reinterpret_cast<const VT *>(xc + j));
        const VT b = __ldcs(reinterpret_cast<const VT *>(yc + j));
#pragma unroll
        for (int i = 0; i < VW; ++i) {
          xv[j + i] = reinterpret_cast<const T *>(&a)[i];
          yv[j + i] = reinterpret_cast<const T *>(&b)[i];
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
      if (j < n) {
        xv[j] = ld_stream(xc + j);
        yv[j] = ld_stream(yc + j);
      } else {
        xv[j] = T(0);
        yv[j] = T(0);
      }
    }
  }
  bool ok = true;
  T cpv[NMAX], dpv[NMAX];
  T hprev = xv[1] - xv[0];
  T ddprev = (yv[1] - yv[0]) / hprev;
  if (bc & 1) {
    const T s = yp1[c];
    ok = ok && finite(s);
    cpv[0] = T(0.5);
    dpv[0] = T(3) * (ddprev - s) / hprev;
  } else {
    cpv[0] = T(0);
    dpv[0] = T(0);
  }
  T cpp = cpv[0], dpp = dpv[0];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j < n) {
      ok = ok && finite(xv[j]) && finite(yv[j]);
      if (j + 1 < n) ok = ok && (xv[j + 1] > xv[j]);
    }
  }
#pragma unroll
  for (int j = 1; j < NMAX - 1; ++j) {
    if (j < n - 1) {
      const T h = xv[j + 1] - xv[j];
      const T dd = (yv[j + 1] - yv[j]) / h;
      const T inv = T(1) / (T(2) * (hprev + h) - hprev * cpv[j - 1]);
      dpv[j] = (T(6) * (dd - ddprev) - hprev * dpv[j - 1]) * inv;
      cpv[j] = h * inv;
      cpp = cpv[j];
      dpp = dpv[j];
      hprev = h;
      ddprev = dd;
    }
  }
  T z[NMAX];
  T last = T(0);
  if (bc & 2) {
    const T e = ypn[c];
    ok = ok && finite(e);
    last = (T(6) * (e - ddprev) - hprev * dpp) / (T(2) * hprev - hprev * cpp);
  }
  T nxt = last;
#pragma unroll
  for (int j = NMAX - 1; j >= 0; --j) {
    if (j == n - 1) {
      z[j] = last;
    } else if (j < n - 1) {
      nxt = dpv[j] - cpv[j] * nxt;
      z[j] = nxt;
    } else {
      z[j] = T(0);
    }
  }
  if (!ok) {
#pragma unroll
    for (int j = 0; j < NMAX; ++j) z[j] = qnan<T>();
  }
  raise_status_warp(!ok, kBadKnots);
  T *zc = y2 + c * n;
  if (vec) {
    using VT = typename Vec16<T>::V;
#pragma unroll
    for (int j = 0; j < NMAX; j += VW) {
      if (j < n) {
        VT a;
#pragma unroll
        for (int i = 0; i < VW; ++i) reinterpret_cast<T *>(&a)[i] = z[j + i];
        *reinterpret_cast<VT *>(zc + j) = a;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
      if (j < n) zc[j] = z[j];
  }
}

}  // namespace fs
