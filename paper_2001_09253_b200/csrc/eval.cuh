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
constexpr int kStageHeader = 16;  // mbarrier (8 B) + pad, ahead of the staged arrays

// Grid: cpb > 1  -> blockIdx.x = group of cpb curves (all m queries of each);
//       cpb == 1 -> blockIdx.x = curve * nchunks + chunk (queries [chunk*qchunk, ..)).
// Staging: BULK -> one thread issues three cp.async.bulk copies (x, y, y2 of the CTA's
// curves, contiguous in HBM) completing on an mbarrier, while every thread already has
// its first batch of query loads in flight; otherwise coalesced loads + __syncthreads.
// Queries: each warp owns a contiguous run of the CTA's queries; lane l takes groups of V
// consecutive queries (one 16-byte vector load / store when V > 1), U groups per batch in
// flight.  MODE_SORTED carries the warp's bracket from one 32V-query step to the next.
template <typename T, int MODE, int V, bool BULK>
__global__ void __launch_bounds__(kEvalThreads) k_eval_staged(const T *__restrict__ x, const T *__restrict__ y,
                                                             const T *__restrict__ y2, int n, int64_t batch,
                                                             const T *__restrict__ q, int m, T *__restrict__ out,
                                                             int32_t *__restrict__ idx, int cpb, int nchunks,
                                                             int qchunk, FastDiv divm) {
  constexpr int U = sizeof(T) == 4 ? 4 : 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
  T *X = reinterpret_cast<T *>(smem_raw + kStageHeader);
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
  const int tot = nc * n;
  if (BULK) {
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(tot * sizeof(T));
      mbar_expect_tx(bar, 3 * bytes);
      bulk_g2s(X, x + c0 * n, bytes, bar);
      bulk_g2s(Y, y + c0 * n, bytes, bar);
      bulk_g2s(Z, y2 + c0 * n, bytes, bar);
    }
  } else {
    const T *xs = x + c0 * n, *ys = y + c0 * n, *zs = y2 + c0 * n;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      X[e] = xs[e];
      Y[e] = ys[e];
      Z[e] = zs[e];
    }
    __syncthreads();
  }

  const int ngroups = (int)(k1 - k0) / V;
  const T *qb = q + k0;
  T *ob = out + k0;
  int32_t *ib = idx ? idx + k0 : nullptr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int per = (ngroups + nw - 1) / nw;
  const int wb = w * per, we = min(ngroups, wb + per);
  bool oor = false, staged = !BULK;
  int jcarry = 0;
  for (int gb = wb; gb < we; gb += 32 * U) {
    T qv[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = gb + u * 32 + lane;
      if (g < we) VecIO<T, V>::load(qb + (int64_t)g * V, qv[u]);
    }
    if (!staged) {
      mbar_wait(bar, 0);
      staged = true;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = gb + u * 32 + lane;
      int jl = -1;
      if (g < we) {
        T val[V];
        int jj[V];
#pragma unroll
        for (int i = 0; i < V; ++i) {
          const int k = g * V + i;
          const int cl = (cpb > 1) ? (int)divm.div((uint32_t)k) : 0;
          eval_one<T, MODE>(X + cl * n, Y + cl * n, Z + cl * n, n, qv[u][i], jcarry, val[i], jj[i]);
          oor |= (jj[i] < 0);
          if (MODE == MODE_SORTED && jj[i] >= 0) jcarry = jj[i];
          jl = max(jl, jj[i]);
        }
        VecIO<T, V>::store(ob + (int64_t)g * V, val);
        if (ib) VecIO<T, V>::store_idx(ib + (int64_t)g * V, jj);
      }
      if (MODE == MODE_SORTED) {
        const int jmax = __reduce_max_sync(0xffffffffu, jl);
        if (jmax >= 0) jcarry = jmax;
      }
    }
  }
  if (!staged) mbar_wait(bar, 0);  // never leave a bulk copy in flight past the CTA's exit
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(kOutOfRange);
}

// Long curves (not stageable): locate in HBM.  Each thread carries U independent queries
// through the three dependent round trips (q -> x pair at the interpolation guess -> y, y2
// pairs) so that U x (threads per SM) gathers are in flight.  The guess
// (q - x_0)(n-1)/(x_{n-1} - x_0) is exact up to +-1 interval on near-uniform grids; any
// other outcome falls back to galloping + bisection (correct for every grid).
template <typename T>
__global__ void __launch_bounds__(256) k_eval_global(const T *__restrict__ x, const T *__restrict__ y,
                                                     const T *__restrict__ y2, int n, int64_t batch,
                                                     const T *__restrict__ q, int64_t m, T *__restrict__ out,
                                                     int32_t *__restrict__ idx) {
  constexpr int U = 4;
  const int64_t total = batch * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool oor = false;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += U * stride) {
    T qq[U], xa[U], xb[U];
    int g[U];
    int64_t off[U];
    bool act[U], in[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = base + u * stride;
      act[u] = k < total;
      qq[u] = act[u] ? ld_stream(q + k) : T(0);
      off[u] = act[u] ? ((batch == 1) ? 0 : (k / m) * n) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T *X = x + off[u];
      const T x0 = __ldg(X), xn = __ldg(X + n - 1);
      in[u] = act[u] && (qq[u] >= x0 && qq[u] <= xn);
      int gg = in[u] ? (int)((qq[u] - x0) * (T)(n - 1) / (xn - x0)) : 0;
      g[u] = max(0, min(gg, n - 2));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      xa[u] = __ldg(x + off[u] + g[u]);
      xb[u] = __ldg(x + off[u] + g[u] + 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (in[u] && !(xa[u] <= qq[u] && (qq[u] < xb[u] || g[u] == n - 2))) {
        const T *X = x + off[u];
        g[u] = locate_from(X, n, g[u], qq[u]);
        xa[u] = __ldg(X + g[u]);
        xb[u] = __ldg(X + g[u] + 1);
      }
    }
    T ya[U], yb[U], za[U], zb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = in[u] ? g[u] : 0;
      ya[u] = __ldg(y + off[u] + j);
      yb[u] = __ldg(y + off[u] + j + 1);
      za[u] = __ldg(y2 + off[u] + j);
      zb[u] = __ldg(y2 + off[u] + j + 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!act[u]) continue;
      const int64_t k = base + u * stride;
      T val = qnan<T>();
      int j = -1;
      if (in[u]) {
        j = g[u];
        val = nr_interp(qq[u], xa[u], xb[u], ya[u], yb[u], za[u], zb[u]);
      } else {
        oor = true;
      }
      st_stream(out + k, val);
      if (idx) st_stream(idx + k, (int32_t)j);
    }
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(kOutOfRange);
}

}  // namespace fs
