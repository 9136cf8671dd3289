// eval.cuh -- fused locate + evaluate kernels.
//
// Locate rule (reading c1): idx = the largest j in [0, n-2] with x_j <= q;
// -1 (and out = NaN, status bit) when q is outside [x_0, x_{n-1}] or NaN, because
// Eq. nr_formula only holds for x_j <= x <= x_{j+1}.  Every search below ends in
// comparisons against this rule, so guesses (sorted-run carry, uniform-grid index,
// interpolation guess) change speed, never idx.
// Evaluate: Eq. nr_formula, see nr_interp in common.cuh.
//
//  k_eval_staged : the curves' x, y, y2 fit in shared memory (3 n s bytes per curve).
//                  A CTA stages a group of curves (coalesced), then each thread
//                  locates its queries in shared memory:
//                    MODE_BSEARCH  -- bisection;
//                    MODE_SORTED   -- a warp takes a contiguous run of queries; the
//                                     bracket of the previous 32 is carried forward
//                                     (generalising the paper's forward scan)
//                                     and each lane gallops from it;
//                    MODE_UNIFORM  -- direct index (q-x_0)(n-1)/(x_{n-1}-x_0), corrected.
//  k_eval_global : long curves (beyond shared memory): interpolation guess in global
//                  memory, corrected by galloping + bisection; gathers x, y, y2.
#pragma once
#include "common.cuh"

namespace fs {

enum { MODE_BSEARCH = 0, MODE_SORTED = 1, MODE_UNIFORM = 2 };

// Largest j in [lo, n-2] with X[j] <= q, given X[lo] <= q <= X[n-1].
template <typename T> __device__ __forceinline__ int gallop_up(const T *X, int n, int lo, T q) {
  int step = 1, hi = min(lo + 1, n - 1);
  while (hi < n - 1 && X[hi] <= q) {
    lo = hi;
    step <<= 1;
    hi = min(lo + step, n - 1);
  }
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (X[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Largest j in [0, hi) with X[j] <= q, given X[0] <= q < X[hi].
template <typename T> __device__ __forceinline__ int gallop_down(const T *X, int hi, T q) {
  int step = 1, lo = max(hi - 1, 0);
  while (lo > 0 && X[lo] > q) {
    hi = lo;
    step <<= 1;
    lo = max(hi - step, 0);
  }
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (X[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

// From a guess g in [0, n-2]; requires X[0] <= q <= X[n-1].
template <typename T> __device__ __forceinline__ int locate_from(const T *X, int n, int g, T q) {
  if (X[g] > q) return gallop_down(X, g, q);
  return gallop_up(X, n, g, q);
}

template <typename T> __device__ __forceinline__ int bisect(const T *X, int n, T q) {
  int lo = 0, hi = n - 1;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (X[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

template <typename T, int MODE>
__device__ __forceinline__ void eval_one(const T *X, const T *Y, const T *Z, int n, T q, int &jcarry, T &val,
                                         int &j) {
  const T x0 = X[0], xn = X[n - 1];
  if (!(q >= x0 && q <= xn)) {  // out of range or NaN
    j = -1;
    val = qnan<T>();
    return;
  }
  if (MODE == MODE_BSEARCH) {
    j = bisect(X, n, q);
  } else if (MODE == MODE_SORTED) {
    j = (X[jcarry] <= q) ? gallop_up(X, n, jcarry, q) : bisect(X, n, q);
  } else {
    int g = (int)((q - x0) * (T)(n - 1) / (xn - x0));
    g = max(0, min(g, n - 2));
    j = locate_from(X, n, g, q);
  }
  val = nr_interp(q, X[j], X[j + 1], Y[j], Y[j + 1], Z[j], Z[j + 1]);
}

constexpr int kEvalThreads = 256;

// Grid: cpb > 1 -> blockIdx.x = group of cpb curves (all m queries each);
//       cpb == 1 -> blockIdx.x = curve * nchunks + chunk (queries [chunk*qchunk, ..)).
template <typename T, int MODE>
__global__ void __launch_bounds__(kEvalThreads) k_eval_staged(const T *__restrict__ x, const T *__restrict__ y,
                                                             const T *__restrict__ y2, int n, int64_t batch,
                                                             const T *__restrict__ q, int m, T *__restrict__ out,
                                                             int32_t *__restrict__ idx, int cpb, int nchunks,
                                                             int qchunk, FastDiv divn, FastDiv divm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *X = reinterpret_cast<T *>(smem_raw);
  T *Y = X + (size_t)cpb * n;
  T *Z = Y + (size_t)cpb * n;

  int64_t c0, k0, k1;
  int nc;
  if (cpb > 1) {
    c0 = (int64_t)blockIdx.x * cpb;
    nc = (int)min64(cpb, batch - c0);
    k0 = c0 * m;
    k1 = (c0 + nc) * m;
  } else {
    c0 = blockIdx.x / nchunks;
    const int ch = blockIdx.x - (int)(c0 * nchunks);
    nc = 1;
    k0 = c0 * m + (int64_t)ch * qchunk;
    k1 = min64(c0 * m + m, k0 + qchunk);
  }
  {
    const int tot = nc * n;
    const T *xs = x + c0 * n, *ys = y + c0 * n, *zs = y2 + c0 * n;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      X[e] = xs[e];
      Y[e] = ys[e];
      Z[e] = zs[e];
    }
  }
  __syncthreads();
  const int cnt = (int)(k1 - k0);
  const T *qb = q + k0;
  T *ob = out + k0;
  int32_t *ib = idx ? idx + k0 : nullptr;
  bool oor = false;

  if (MODE == MODE_SORTED) {
    // Each warp owns a contiguous run of the CTA's queries, 32 at a time.
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int per = ((cnt + nw - 1) / nw + 31) & ~31;
    const int wb = w * per, we = min(cnt, wb + per);
    int jcarry = 0;
    for (int base = wb; base < we; base += 32) {
      const int k = base + lane;
      const bool act = k < we;
      const int cl = (cpb > 1 && act) ? (int)divm.div((uint32_t)k) : 0;
      int j = -1;
      T val = T(0);
      if (act) {
        const T qq = ld_stream(qb + k);
        eval_one<T, MODE_SORTED>(X + cl * n, Y + cl * n, Z + cl * n, n, qq, jcarry, val, j);
        st_stream(ob + k, val);
        if (ib) st_stream(ib + k, (int32_t)j);
        oor |= (j < 0);
      }
      const int jmax = __reduce_max_sync(0xffffffffu, act ? j : -1);
      if (jmax >= 0) jcarry = jmax;
    }
  } else {
    constexpr int U = 4;
    for (int base = threadIdx.x; base < cnt; base += U * blockDim.x) {
      T qq[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * blockDim.x;
        qq[u] = (k < cnt) ? ld_stream(qb + k) : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * blockDim.x;
        if (k < cnt) {
          const int cl = (cpb > 1) ? (int)divm.div((uint32_t)k) : 0;
          int jc = 0, j;
          T val;
          eval_one<T, MODE>(X + cl * n, Y + cl * n, Z + cl * n, n, qq[u], jc, val, j);
          st_stream(ob + k, val);
          if (ib) st_stream(ib + k, (int32_t)j);
          oor |= (j < 0);
        }
      }
    }
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(kOutOfRange);
}

// Long curves: one query per thread-iteration, everything gathered from global memory.
template <typename T>
__global__ void __launch_bounds__(256) k_eval_global(const T *__restrict__ x, const T *__restrict__ y,
                                                     const T *__restrict__ y2, int n, int64_t batch,
                                                     const T *__restrict__ q, int64_t m, T *__restrict__ out,
                                                     int32_t *__restrict__ idx) {
  const int64_t total = batch * m;
  bool oor = false;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (batch == 1) ? 0 : k / m;
    const T *X = x + c * n;
    const T qq = ld_stream(q + k);
    const T x0 = __ldg(X), xn = __ldg(X + n - 1);
    int j = -1;
    T val = qnan<T>();
    if (qq >= x0 && qq <= xn) {
      int g = (int)((qq - x0) * (T)(n - 1) / (xn - x0));
      g = max(0, min(g, n - 2));
      j = locate_from(X, n, g, qq);
      const T *Y = y + c * n, *Z = y2 + c * n;
      val = nr_interp(qq, __ldg(X + j), __ldg(X + j + 1), __ldg(Y + j), __ldg(Y + j + 1), __ldg(Z + j),
                      __ldg(Z + j + 1));
    } else {
      oor = true;
    }
    st_stream(out + k, val);
    if (idx) st_stream(idx + k, (int32_t)j);
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(kOutOfRange);
}

}  // namespace fs
