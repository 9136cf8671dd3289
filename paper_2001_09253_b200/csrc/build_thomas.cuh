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

// Row stride of the transposed tiles of babe_tile.  A warp holds 16 curves x (top, bottom):
// at a step the top lanes touch row j and the bottom lanes row n-1-j of their curves.  With
// S = 2 mod 4 the 16 curves of one end fall on 16 distinct banks of one parity class (S t mod 32
// = 2 (u t mod 16), u odd), and for even n the two ends are n-1-2j (odd) banks apart, i.e. in the
// other parity class: every step is conflict-free.  Odd n: an odd stride (16 distinct banks
// per end; the two ends may share a bank).
__host__ __device__ constexpr int babe_stride(int n) { return (n & 1) ? n : ((n % 4 == 2) ? n : n + 2); }

// The two-ended sweep of one CTA tile: curve t = threadIdx.x/2 of the tile lives at
// Xc = X + t*S, Yc = Y + t*S (odd stride S); on return Yc holds y2 (or NaN).
// Both threads of a pair run the SAME instruction stream with a direction dir = +1 (top:
// rows 0, 1, .., k-1) or -1 (bottom: rows n-1, n-2, .., k+1), so a warp never diverges:
//   g_i  = (y_{j+dir} - y_j) / (x_{j+dir} - x_j)      (the divided difference of the step)
//   h_i  = dir (x_{j+dir} - x_j) > 0
//   row  : den = 2(h_c + h) - h_c c'_prev,  c' = h/den,  d' = (6 dir (g - g_c) - h_c d'_prev)/den
// where (h_c, g_c) belong to the interval already eliminated.  For dir = +1 this is the
// paper's forward sweep verbatim; for dir = -1 it is the same recurrence read
// from the other end.  Divisions are a correctly rounded reciprocal then a multiply.
// The clamped end slope a thread of babe_tile needs (top: yp1, bottom: ypn; 0 when that end is
// natural).  Callers issue this global load before staging the tile, so its latency is hidden.
template <typename T>
__device__ __forceinline__ T babe_slope(int64_t c0, int nc, int bc, const T *__restrict__ yp1,
                                        const T *__restrict__ ypn, int tid) {
  const int t = tid >> 1;
  const bool top = (tid & 1) == 0;
  const int64_t cg = c0 + (t < nc ? t : 0);
  if (top) return (bc & 1) ? yp1[cg] : T(0);
  return (bc & 2) ? ypn[cg] : T(0);
}

// The arithmetic of the two-ended sweep, shared by every kernel that runs it, with every
// rounding explicit (no compiler-chosen contraction), so all of them agree bitwise: the end
// row, one eliminated row, the meeting row and one back-substitution row.  dir = +1 (top) or
// -1 (bottom); d = x_{j+dir} - x_j, h = dir d > 0.
// End row: g = the divided difference; natural: c' = d' = 0; clamped (P:966-971 start,
// P:1017-1018 end): c' = 1/2, d' = 3 dir (g - y') / h.
template <typename T>
__device__ __forceinline__ bool babe_first(T xo, T yo, T xn, T yn, int dir, bool clamped, T sl, T &hc, T &gc, T &cp,
                                           T &dp) {
  const T d = r_sub(xn, xo);
  hc = (dir > 0) ? d : -d;
  bool ok = finite(xo) & finite(yo) & finite(xn) & finite(yn) & (hc > T(0));
  gc = r_mul(r_sub(yn, yo), nr_rcp(d));
  cp = T(0);
  dp = T(0);
  if (clamped) {
    ok &= finite(sl);
    cp = T(0.5);
    dp = r_mul(r_mul(T(3 * dir), r_sub(gc, sl)), nr_rcp(hc));
  }
  return ok;
}
// One row: den = 2(h_c + h) - h_c c'_prev, c' = h/den, d' = (6 dir (g - g_c) - h_c d'_prev)/den
// (P:714-718 read from either end); returns the row's validity (finite, strictly increasing).
template <typename T>
__device__ __forceinline__ bool babe_row(T xo, T yo, T xn, T yn, int dir, T &hc, T &gc, T &cp, T &dp) {
  const T d = r_sub(xn, xo);
  const T h = (dir > 0) ? d : -d;
  const bool ok = finite(xn) & finite(yn) & (h > T(0));
  const T g = r_mul(r_sub(yn, yo), nr_rcp(d));
  const T inv = nr_rcp(r_fma(-hc, cp, r_mul(T(2), r_add(hc, h))));
  dp = r_mul(r_fma(-hc, dp, r_mul(T(6 * dir), r_sub(g, gc))), inv);
  cp = r_mul(h, inv);
  hc = h;
  gc = g;
  return ok;
}
// Meet at row k (lanes 2t, 2t+1 hold the top and bottom sweeps of one curve): a_k = h_{k-1},
// b_k = 2(h_{k-1} + h_k), c_k = h_k, d_k = 6(dd_k - dd_{k-1}); both lanes return y2_k, and ok
// becomes the pair's.  Every lane of the warp must call it.
template <typename T> __device__ __forceinline__ T babe_meet(bool top, T hc, T gc, T cp, T dp, bool &ok) {
  const T o_h = __shfl_xor_sync(0xffffffffu, hc, 1);
  const T o_g = __shfl_xor_sync(0xffffffffu, gc, 1);
  const T o_cp = __shfl_xor_sync(0xffffffffu, cp, 1);
  const T o_dp = __shfl_xor_sync(0xffffffffu, dp, 1);
  const int o_ok = __shfl_xor_sync(0xffffffffu, (int)ok, 1);
  ok = ok & (o_ok != 0);
  const T hk1 = top ? hc : o_h, gk1 = top ? gc : o_g, cT = top ? cp : o_cp, dT = top ? dp : o_dp;
  const T hk = top ? o_h : hc, gk = top ? o_g : gc, aB = top ? o_cp : cp, dB = top ? o_dp : dp;
  const T num = r_fma(-hk, dB, r_fma(-hk1, dT, r_mul(T(6), r_sub(gk, gk1))));
  const T den = r_fma(-hk, aB, r_fma(-hk1, cT, r_mul(T(2), r_add(hk1, hk))));
  return r_mul(num, nr_rcp(den));
}
// Back-substitution: y_j = d'_j - c'_j y_{j+dir}
template <typename T> __device__ __forceinline__ T babe_back(T cb, T db, T yv) { return r_fma(-cb, yv, db); }

template <typename T>
__device__ __forceinline__ void babe_tile(unsigned *__restrict__ status, T *X, T *Y, int S, int n, int nc, int bc, T sl, T *dummy, int tid) {
  const int t = tid >> 1;  // curve within the tile (tid = thread index within the solving group)
  const bool top = (tid & 1) == 0;
  const bool act = t < nc;         // pairs are lane-adjacent, so shuffles stay in-warp
  const int k = n >> 1;            // meeting row, 1 <= k <= n-2
  const int dir = top ? 1 : -1;
  const int j0 = top ? 0 : n - 1;
  // inactive pairs (ragged last tile) run on a private scratch row, so no store is predicated
  T *Xc = act ? X + t * S : dummy;
  T *Yc = act ? Y + t * S : dummy + S;
  if (!act) {
    Xc[j0] = T(j0);
    Xc[j0 + dir] = T(j0 + dir);
  }
  // end row
  T xo = Xc[j0], yo = Yc[j0];
  T xn = Xc[j0 + dir], yn = Yc[j0 + dir];
  T hc, gc, cp, dp;
  bool ok = babe_first(xo, yo, xn, yn, dir, top ? (bc & 1) : (bc & 2), sl, hc, gc, cp, dp);
  // the row after next is loaded one step ahead (register rotation), so the shared-memory
  // latency is off the dependency chain; near the meeting row the look-ahead may read a row
  // of the other thread's half, a value that is never used
  T xnn = Xc[j0 + 2 * dir], ynn = Yc[j0 + 2 * dir];  // n >= 3
  Xc[j0] = cp;
  Yc[j0] = dp;
  int j = j0 + dir;
  auto step = [&]() {
    xo = xn;
    yo = yn;
    xn = xnn;
    yn = ynn;
    const int jp = min(max(j + 2 * dir, 0), n - 1);
    xnn = Xc[jp];
    ynn = Yc[jp];
    ok &= babe_row(xo, yo, xn, yn, dir, hc, gc, cp, dp);
    Xc[j] = cp;
    Yc[j] = dp;
    j += dir;
  };
  const int common = n - 2 - k;  // bottom's interior rows; the top has one more when n is even
#pragma unroll 2
  for (int i = 0; i < common; ++i) step();
  if (top && (k - 1 > common)) step();
  const T yk = babe_meet(top, hc, gc, cp, dp, ok);
  if (top) Yc[k] = yk;
  // back-substitution outward from the seam: y_j = d'_j - c'_j y_{j+dir}
  T yv = yk;
  int jj = k - dir;
  T cb = Xc[jj], db = Yc[jj];
  auto back = [&]() {
    const int jn = min(max(jj - dir, 0), n - 1);  // next row loaded ahead of this row's store
    const T cb2 = Xc[jn], db2 = Yc[jn];
    yv = babe_back(cb, db, yv);
    Yc[jj] = yv;
    cb = cb2;
    db = db2;
    jj -= dir;
  };
  const int bcommon = n - 1 - k;  // bottom's count; the top has k (one more when n is even)
#pragma unroll 2
  for (int i = 0; i < bcommon; ++i) back();
  if (top && (k > bcommon)) back();
  if (!ok) {  // both threads of the pair see the same ok
    const T nanv = qnan<T>();
    for (int r = top ? 0 : k + 1; r < (top ? k + 1 : n); ++r) Yc[r] = nanv;
  }
  raise_status_warp(status, act && !ok && top, kBadKnots);
}

template <typename T>
__global__ void __launch_bounds__(kK1Threads) k1_thomas_babe(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int n,
                                                             int64_t batch, int bc, const T *__restrict__ yp1,
                                                             const T *__restrict__ ypn, T *__restrict__ y2, int S,
                                                             FastDiv divn) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  pdl_trigger();
  const int CPB = blockDim.x / 2;  // blockDim = 2 x curves per CTA (<= 256)
  T *X = reinterpret_cast<T *>(smem_raw);
  T *Y = X + (size_t)CPB * S;
  T *dummy = Y + (size_t)CPB * S;  // 2S scratch for inactive pairs

  const int64_t c0 = (int64_t)blockIdx.x * CPB;
  const int nc = (int)min64(CPB, batch - c0);
  const int tot = nc * n;
  const T sl = babe_slope(c0, nc, bc, yp1, ypn, threadIdx.x);  // in flight during the staging
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

  babe_tile(status, X, Y, S, n, nc, bc, sl, dummy, threadIdx.x);
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
__global__ void __launch_bounds__(kK1Threads) k1_thomas_pipe(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int n,
                                                             int64_t batch, int bc, const T *__restrict__ yp1,
                                                             const T *__restrict__ ypn, T *__restrict__ y2, int S,
                                                             int64_t ntiles, FastDiv divn) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  pdl_trigger();
  const int CPB = blockDim.x / 2;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
  T *Xr = reinterpret_cast<T *>(smem_raw + 16);
  T *Yr = Xr + (size_t)CPB * n;
  T *X = reinterpret_cast<T *>(smem_raw + 16 + ((2 * (size_t)CPB * n * sizeof(T) + 15) & ~(size_t)15));
  T *Y = X + (size_t)CPB * S;
  T *dummy = Y + (size_t)CPB * S;  // 2S scratch for inactive pairs
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
    const T sl = babe_slope(c0, nc, bc, yp1, ypn, threadIdx.x);  // in flight during the staging
    mbar_wait(bar, phase);
    phase ^= 1u;
    // to the odd-stride tiles: 16-byte reads of the raw stage (n*sizeof(T) % 16 == 0, so a
    // vector never straddles two curves)
    constexpr int VW = 16 / sizeof(T);
    using VT = typename Vec16<T>::V;
    for (int e = threadIdx.x * VW; e < tot; e += blockDim.x * VW) {
      const int c = (int)divn.div((uint32_t)e);
      const int j = e - c * n;
      const VT a = *reinterpret_cast<const VT *>(Xr + e);
      const VT b = *reinterpret_cast<const VT *>(Yr + e);
      T *xd = X + c * S + j, *yd = Y + c * S + j;
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        xd[i] = reinterpret_cast<const T *>(&a)[i];
        yd[i] = reinterpret_cast<const T *>(&b)[i];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) issue(it + G);  // raw stage consumed: next tile in flight
    babe_tile(status, X, Y, S, n, nc, bc, sl, dummy, threadIdx.x);
    __syncthreads();
    T *y2b = y2 + c0 * n;
    for (int e = threadIdx.x * VW; e < tot; e += blockDim.x * VW) {
      const int c = (int)divn.div((uint32_t)e);
      const int j = e - c * n;
      const T *ys = Y + c * S + j;
      VT a;
#pragma unroll
      for (int i = 0; i < VW; ++i) reinterpret_cast<T *>(&a)[i] = ys[i];
      *reinterpret_cast<VT *>(y2b + e) = a;
    }
    __syncthreads();
  }
}

// The paper's sweep for one curve held in registers, n <= NMAX: forward
// elimination c'_j, d'_j, back-substitution.  s1 / sn are the
// clamped end slopes (read only when that bc bit is set).  z = y2, all NaN when the curve
// is invalid; returns validity.
template <typename T, int NMAX>
__device__ __forceinline__ bool thomas_regs(const T (&xv)[NMAX], const T (&yv)[NMAX], int n, int bc, T s1, T sn,
                                            T (&z)[NMAX]) {
  bool ok = true;
  T cpv[NMAX], dpv[NMAX];
  // (explicitly rounded, reciprocal + Newton then multiply, like the other solvers)
  T hprev = r_sub(xv[1], xv[0]);
  T ddprev = r_mul(r_sub(yv[1], yv[0]), nr_rcp(hprev));
  if (bc & 1) {
    ok = ok && finite(s1);
    cpv[0] = T(0.5);
    dpv[0] = r_mul(r_mul(T(3), r_sub(ddprev, s1)), nr_rcp(hprev));
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
      const T h = r_sub(xv[j + 1], xv[j]);
      const T dd = r_mul(r_sub(yv[j + 1], yv[j]), nr_rcp(h));
      const T inv = nr_rcp(r_fma(-hprev, cpv[j - 1], r_mul(T(2), r_add(hprev, h))));
      dpv[j] = r_mul(r_fma(-hprev, dpv[j - 1], r_mul(T(6), r_sub(dd, ddprev))), inv);
      cpv[j] = r_mul(h, inv);
      cpp = cpv[j];
      dpp = dpv[j];
      hprev = h;
      ddprev = dd;
    }
  }
  T last = T(0);
  if (bc & 2) {
    ok = ok && finite(sn);
    last = r_mul(r_fma(-hprev, dpp, r_mul(T(6), r_sub(sn, ddprev))), nr_rcp(r_fma(-hprev, cpp, r_mul(T(2), hprev))));
  }
  T nxt = last;
#pragma unroll
  for (int j = NMAX - 1; j >= 0; --j) {
    if (j == n - 1) {
      z[j] = last;
    } else if (j < n - 1) {
      nxt = r_fma(-cpv[j], nxt, dpv[j]);
      z[j] = nxt;
    } else {
      z[j] = T(0);
    }
  }
  if (!ok) {
#pragma unroll
    for (int j = 0; j < NMAX; ++j) z[j] = qnan<T>();
  }
  return ok;
}

// K1r: one thread per curve, n <= NMAX, all in registers.
template <typename T, int NMAX>
__global__ void __launch_bounds__(256) k1_thomas_regs(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int n,
                                                      int64_t batch, int bc, const T *__restrict__ yp1,
                                                      const T *__restrict__ ypn, T *__restrict__ y2, int vec,
                                                      int64_t xs) {
  pdl_trigger();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= batch) return;
  T xv[NMAX], yv[NMAX];
  const T *xc = x + c * xs, *yc = y + c * n;  // xs = n, or 0: one knot vector shared by the batch
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
  T z[NMAX];
  const bool ok = thomas_regs<T, NMAX>(xv, yv, n, bc, (bc & 1) ? yp1[c] : T(0), (bc & 2) ? ypn[c] : T(0), z);
  raise_status_warp(status, !ok, kBadKnots);
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


// K1h (k1_thomas_half, n = N in {16, 32, 64}, 16-byte-aligned curve rows): the two-ended sweep
// with each thread's half curve in REGISTERS -- no shared-memory tile, no transposition, no
// staging barrier.  Lane 2t (top) owns rows 0 .. K-1 of curve t, lane 2t+1 (bottom) rows
// N-1 .. K (K = N/2); "step s" is row s for the top and row N-1-s for the bottom, so both run
// one instruction stream.  Each thread loads / stores its half with 16-byte vectors (the bottom
// reverses the element order).  The arithmetic is babe_first/babe_row/babe_meet/babe_back, so
// y2 is bitwise the shared-memory K1's (and the fused kernel's).
constexpr int kK1hThreads = 128;
// One lane pair's curve cv (lane parity: top / bottom) -- the body of K1h, also called by the
// fused build+eval kernels.  Every lane of the warp must call it.  y2 (nullable) receives the
// curve's row in HBM; zs (nullable) is a 16-byte-aligned row in shared memory that receives it too.
template <typename T, int N>
__device__ __forceinline__ void k1h_solve(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int64_t batch, int bc,
                                          const T *__restrict__ yp1, const T *__restrict__ ypn, T *__restrict__ y2,
                                          int64_t cv, bool top, T *zs = nullptr) {
  constexpr int K = N / 2;
  constexpr int VW = 16 / sizeof(T);
  static_assert(K % VW == 0 && K >= 2 * VW, "each half is whole 16-byte vectors");
  using VT = typename Vec16<T>::V;
  const bool act = cv < batch;
  const int64_t c = act ? cv : batch - 1;  // a ragged last warp shadows the last curve, stores nothing
  const int dir = top ? 1 : -1;
  const int hoff = top ? 0 : K;            // this thread's half of the row
  const T sl = top ? ((bc & 1) ? yp1[c] : T(0)) : ((bc & 2) ? ypn[c] : T(0));
  T xs[K], ys[K];
  {
    const T *xh = x + c * N + hoff, *yh = y + c * N + hoff;
#pragma unroll
    for (int g = 0; g < K; g += VW) {
      const int o = top ? g : K - g - VW;
      const VT a = __ldg(reinterpret_cast<const VT *>(xh + o));
      const VT b = __ldg(reinterpret_cast<const VT *>(yh + o));
      const T *pa = reinterpret_cast<const T *>(&a), *pb = reinterpret_cast<const T *>(&b);
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        xs[g + e] = top ? pa[e] : pa[VW - 1 - e];
        ys[g + e] = top ? pb[e] : pb[VW - 1 - e];
      }
    }
  }
  // row K (the top's last neighbour) is the bottom thread's last step
  const T xK = __shfl_xor_sync(0xffffffffu, xs[K - 1], 1), yK = __shfl_xor_sync(0xffffffffu, ys[K - 1], 1);
  T hc, gc, cp, dp;
  T cpr[K], dpr[K];
  bool ok = babe_first(xs[0], ys[0], xs[1], ys[1], dir, top ? (bc & 1) : (bc & 2), sl, hc, gc, cp, dp);
  cpr[0] = cp;
  dpr[0] = dp;
#pragma unroll
  for (int s = 1; s < K - 1; ++s) {  // rows both threads eliminate
    ok &= babe_row(xs[s], ys[s], xs[s + 1], ys[s + 1], dir, hc, gc, cp, dp);
    cpr[s] = cp;
    dpr[s] = dp;
  }
  {  // the top's extra row K-1 (the bottom's step K-1 is the meeting row itself)
    T h2 = hc, g2 = gc, c2 = cp, d2 = dp;
    const bool ok2 = babe_row(xs[K - 1], ys[K - 1], xK, yK, dir, h2, g2, c2, d2);
    if (top) {
      ok &= ok2;
      hc = h2;
      gc = g2;
      cp = c2;
      dp = d2;
    }
    cpr[K - 1] = c2;
    dpr[K - 1] = d2;
  }
  const T yk = babe_meet(top, hc, gc, cp, dp, ok);
  // back-substitution outward from the seam; yo[s] = y2 of step s's row (dpr reused)
  T yv = yk;
  {
    const T yt = babe_back(cpr[K - 1], dpr[K - 1], yv);
    yv = top ? yt : yk;
    dpr[K - 1] = yv;  // top: row K-1; bottom: row K = the seam
  }
#pragma unroll
  for (int s = K - 2; s >= 0; --s) {
    yv = babe_back(cpr[s], dpr[s], yv);
    dpr[s] = yv;
  }
  if (!ok) {  // both threads of the pair see the same ok
#pragma unroll
    for (int s = 0; s < K; ++s) dpr[s] = qnan<T>();
  }
  raise_status_warp(status, act && !ok && top, kBadKnots);
  if (act) {
#pragma unroll
    for (int g = 0; g < K; g += VW) {
      VT a;
      T *pa = reinterpret_cast<T *>(&a);
#pragma unroll
      for (int e = 0; e < VW; ++e) pa[e] = top ? dpr[g + e] : dpr[g + VW - 1 - e];
      const int o = hoff + (top ? g : K - g - VW);
      if (y2) *reinterpret_cast<VT *>(y2 + c * N + o) = a;
      if (zs) *reinterpret_cast<VT *>(zs + o) = a;
    }
  }
}

template <typename T, int N>
__global__ void __launch_bounds__(kK1hThreads) k1_thomas_half(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y,
                                                              int64_t batch, int bc, const T *__restrict__ yp1,
                                                              const T *__restrict__ ypn, T *__restrict__ y2) {
  pdl_trigger();
  k1h_solve<T, N>(status, x, y, batch, bc, yp1, ypn, y2, ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 1,
                  (threadIdx.x & 1) == 0);
}

}  // namespace fs
