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
//                    MODE_TABLE    -- (unsorted default) packed knots + per-curve bucket
//                                     table bracketing each query, then bisection;
//                    MODE_BSEARCH  -- bisection (curves too large for the table);
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

enum { MODE_BSEARCH = 0, MODE_SORTED = 1, MODE_UNIFORM = 2, MODE_TABLE = 3 };

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
  if (MODE == MODE_SORTED) {
    j = (X[jcarry] <= q) ? gallop_up(X, n, jcarry, q) : bisect(X, n, q);
  } else {
    j = bisect(X, n, q);
  }
  val = nr_interp(q, X[j], X[j + 1], Y[j], Y[j + 1], Z[j], Z[j + 1]);
}

// ---- packed knots + bucket table (MODE_TABLE, MODE_UNIFORM) ---------------------------
// Per staged curve: K[j] = {x_j, y_j, y2_j, 1/h_j} (one 16/32-byte record per knot, so the
// gather is two vector loads and the per-query division becomes a multiply by the
// interval's precomputed reciprocal -- the paper's inv_ba), and for MODE_TABLE
// a bucket table over nb = n equal-width buckets of [x_0, x_{n-1}]:
//     bucket(v) = min(nb, (int)((v - x_0) * s)),   s = nb / (x_{n-1} - x_0)
//     Tb[b]     = max{ j in [0, n-2] : bucket(x_j) < b }   (Tb[0] = 0).
// bucket() is monotone in v, so for an in-range query q in bucket b the answer
// j* = max{ j : x_j <= q } satisfies Tb[b] <= j* <= Tb[b+1]: the table only brackets the
// search, which still ends in comparisons x_j <= q (bit-exact idx on any grid).
template <typename T> struct Knot { T x, y, z, ih; };

template <typename T> __device__ __forceinline__ int bucket_of(T v, T x0, T s, int nb) {
  const T f = (v - x0) * s;
  return (f >= T(0)) ? min((int)f, nb) : 0;  // f is NaN-free for finite knots
}

template <typename T>
__device__ __forceinline__ void eval_packed(const Knot<T> *K, const uint16_t *Tb, T s, int n, T q, int mode,
                                            T &val, int &j) {
  const T x0 = K[0].x, xn = K[n - 1].x;
  if (!(q >= x0 && q <= xn)) {
    j = -1;
    val = qnan<T>();
    return;
  }
  int lo, hi;
  if (mode == MODE_TABLE) {
    const int b = bucket_of(q, x0, s, n);
    lo = min((int)Tb[b], n - 2);  // clamps keep invalid (non-monotone) knots memory-safe
    hi = max(lo, min((int)Tb[b + 1], n - 2));
  } else {  // MODE_UNIFORM: direct index on the (hinted) uniform grid, then corrected
    int g = (int)((q - x0) * s);
    g = max(0, min(g, n - 2));
    if (K[g].x > q) {
      hi = g - 1;
      lo = (g >= 1 && K[g - 1].x <= q) ? g - 1 : 0;
    } else {
      lo = g; hi = n - 2;
      if (g + 1 <= n - 2 && K[g + 1].x > q) hi = g;  // the common case: settled in one compare
    }
  }
  while (lo < hi) {  // largest j in [lo, hi] with x_j <= q
    const int mid = (lo + hi + 1) >> 1;
    if (K[mid].x <= q) lo = mid;
    else hi = mid - 1;
  }
  j = lo;
  const Knot<T> a = K[j], b = K[j + 1];
  val = interp_core(q, a.x, b.x, a.y, b.y, a.z, b.z, a.ih);
}

constexpr int kEvalThreads = 256;
constexpr int kStageHeader = 16;  // mbarrier (8 B) + pad, ahead of the staged arrays

__host__ __device__ constexpr size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

// Shared-memory layout of one CTA: two raw stages (x, y, y2 of cpb curves each, filled by
// TMA bulk copies) + the packed knots / scales / bucket table of the item being evaluated.
template <typename T> struct StageLayout {
  size_t raw[2], knots, scale, table, total;
  __host__ __device__ StageLayout(int cpb, int n, bool packed, bool table_) {
    const size_t rawb = 3 * sizeof(T) * (size_t)cpb * n;
    raw[0] = kStageHeader;
    raw[1] = align16(raw[0] + rawb);
    size_t off = align16(raw[1] + rawb);
    knots = off;
    if (packed) off = align16(off + sizeof(Knot<T>) * (size_t)cpb * n);
    scale = off;
    if (packed) off = align16(off + sizeof(T) * (size_t)cpb);
    table = off;
    if (table_) off = align16(off + sizeof(uint16_t) * (size_t)cpb * (n + 2));
    total = off;
  }
};

// Work item `it`: curves [c0, c0+nc) and queries [k0, k1) (flat indices into q).
struct Item {
  int64_t c0, k0, k1;
  int nc;
};
__device__ __forceinline__ Item item_of(int64_t it, int64_t batch, int m, int cpb, int nchunks, int qchunk) {
  Item r;
  if (cpb > 1) {
    r.c0 = it * cpb;
    r.nc = (int)min64(cpb, batch - r.c0);
    r.k0 = r.c0 * m;
    r.k1 = (r.c0 + r.nc) * m;
  } else {
    r.c0 = it / nchunks;
    const int ch = (int)(it - r.c0 * nchunks);
    r.nc = 1;
    r.k0 = r.c0 * m + (int64_t)ch * qchunk;
    r.k1 = min64(r.c0 * m + m, r.k0 + qchunk);
  }
  return r;
}

// Persistent, double-buffered staged eval.  Grid = min(items, SMs x CTAs/SM); CTA b takes
// items b, b+G, b+2G, ...  Pipeline per CTA:
//   * raw stage s holds item i's x, y, y2 (cp.async.bulk -> mbarrier[s]); the copy for
//     item i+1 is already in flight in stage s^1 while item i is evaluated, and stage s is
//     refilled (item i+2) as soon as it has been consumed;
//   * query batches are register double-buffered: batch b+1 (possibly the next item's
//     first batch) is loaded before batch b is evaluated.
// Each warp owns a contiguous run of an item's queries; lane l takes groups of V
// consecutive queries (16-byte vectors when V > 1), U groups per batch.
template <typename T, int MODE, int V, bool BULK>
__global__ void __launch_bounds__(kEvalThreads) k_eval_staged(const T *__restrict__ x, const T *__restrict__ y,
                                                             const T *__restrict__ y2, int n, int64_t batch,
                                                             const T *__restrict__ q, int m, T *__restrict__ out,
                                                             int32_t *__restrict__ idx, int cpb, int nchunks,
                                                             int qchunk, int64_t nitems, FastDiv divn,
                                                             FastDiv divm) {
  constexpr int U = 4;
  constexpr bool PACKED = (MODE == MODE_TABLE || MODE == MODE_UNIFORM);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const StageLayout<T> L(cpb, n, PACKED, MODE == MODE_TABLE);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);  // bar[0], bar[1]
  Knot<T> *K = reinterpret_cast<Knot<T> *>(smem_raw + L.knots);
  T *Sc = reinterpret_cast<T *>(smem_raw + L.scale);
  uint16_t *Tb = reinterpret_cast<uint16_t *>(smem_raw + L.table);
  const int64_t G = gridDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;

  const size_t raw0 = L.raw[0], rawstep = L.raw[1] - L.raw[0];
  auto raw = [&](int s) { return reinterpret_cast<T *>(smem_raw + raw0 + (size_t)s * rawstep); };
  auto issue = [&](int64_t it, int s) {  // thread 0 only
    if (!BULK || it >= nitems) return;
    const Item I = item_of(it, batch, m, cpb, nchunks, qchunk);
    const uint32_t bytes = (uint32_t)((size_t)I.nc * n * sizeof(T));
    T *R = raw(s);
    mbar_expect_tx(bar + s, 3 * bytes);
    bulk_g2s(R, x + I.c0 * n, bytes, bar + s);
    bulk_g2s(R + (size_t)cpb * n, y + I.c0 * n, bytes, bar + s);
    bulk_g2s(R + 2 * (size_t)cpb * n, y2 + I.c0 * n, bytes, bar + s);
  };
  // The warp's group range of an item.
  auto wrange = [&](const Item &I, int &wb, int &we) {
    const int ng = (int)(I.k1 - I.k0) / V;
    const int per = (ng + nw - 1) / nw;
    wb = w * per;
    we = min(ng, wb + per);
  };
  auto load_batch = [&](const Item &I, int gb, int we, T (&qv)[U][V]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int g = gb + u * 32 + lane;
      if (g < we) VecIO<T, V>::load(q + I.k0 + (int64_t)g * V, qv[u]);
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  int64_t it = blockIdx.x;
  if (threadIdx.x == 0) {
    issue(it, 0);
    issue(it + G, 1);
  }
  T qa[U][V], qn[U][V];
  Item I = item_of(it < nitems ? it : 0, batch, m, cpb, nchunks, qchunk);
  int wb, we;
  wrange(I, wb, we);
  if (it < nitems) load_batch(I, wb, we, qa);
  bool oor = false;
  uint32_t phases = 0u;  // bit s = parity to wait for on bar[s]
  int s = 0;

  for (; it < nitems; it += G) {
    if (BULK) {
      mbar_wait(bar + s, (phases >> s) & 1u);
      phases ^= 1u << s;
    } else {  // unaligned inputs: synchronous coalesced staging
      T *R = raw(s);
      const int tot = I.nc * n;
      for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        R[e] = x[I.c0 * n + e];
        R[(size_t)cpb * n + e] = y[I.c0 * n + e];
        R[2 * (size_t)cpb * n + e] = y2[I.c0 * n + e];
      }
      __syncthreads();
    }
    const T *X = raw(s);
    const T *Y = X + (size_t)cpb * n;
    const T *Z = Y + (size_t)cpb * n;
    const int tot = I.nc * n;
    if (PACKED) {
      for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int c = (int)divn.div((uint32_t)e);
        const int j = e - c * n;
        const T xj = X[e];
        Knot<T> kk;
        kk.x = xj;
        kk.y = Y[e];
        kk.z = Z[e];
        kk.ih = (j < n - 1) ? r_rcp(r_sub(X[e + 1], xj)) : T(0);
        K[e] = kk;
        const T x0 = X[c * n], xn = X[c * n + n - 1];
        const T sc = (MODE == MODE_TABLE) ? (T)n / (xn - x0) : (T)(n - 1) / (xn - x0);
        if (j == 0) Sc[c] = sc;
        if (MODE == MODE_TABLE && j < n - 1) {
          uint16_t *Tc = Tb + c * (n + 2);
          if (j == 0) Tc[0] = 0;
          const int blo = bucket_of(xj, x0, sc, n);
          const int bhi = (j == n - 2) ? n + 1 : bucket_of(X[e + 1], x0, sc, n);
          for (int b = blo + 1; b <= bhi; ++b) Tc[b] = (uint16_t)j;
        }
      }
      __syncthreads();  // K/T built; raw stage s consumed
      if (threadIdx.x == 0) issue(it + 2 * G, s);
    }

    // next item's geometry (for the cross-item prefetch of its first batch)
    const int64_t itn = it + G;
    Item In = I;
    int wbn = 0, wen = 0;
    if (itn < nitems) {
      In = item_of(itn, batch, m, cpb, nchunks, qchunk);
      wrange(In, wbn, wen);
    }
    int jcarry = 0;
    for (int gb = wb; gb < we; gb += 32 * U) {
      const bool last = gb + 32 * U >= we;
      if (!last) load_batch(I, gb + 32 * U, we, qn);
      else if (itn < nitems) load_batch(In, wbn, wen, qn);
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
            const int cl = (cpb > 1) ? (int)divm.div((uint32_t)(I.k0 - I.c0 * m + k)) : 0;
            if (PACKED) {
              eval_packed(K + cl * n, Tb + cl * (n + 2), Sc[cl], n, qa[u][i], MODE, val[i], jj[i]);
            } else {
              eval_one<T, MODE>(X + cl * n, Y + cl * n, Z + cl * n, n, qa[u][i], jcarry, val[i], jj[i]);
              if (MODE == MODE_SORTED && jj[i] >= 0) jcarry = jj[i];
            }
            oor |= (jj[i] < 0);
            jl = max(jl, jj[i]);
          }
          VecIO<T, V>::store(out + I.k0 + (int64_t)g * V, val);
          if (idx) VecIO<T, V>::store_idx(idx + I.k0 + (int64_t)g * V, jj);
        }
        if (MODE == MODE_SORTED) {
          const int jmax = __reduce_max_sync(0xffffffffu, jl);
          if (jmax >= 0) jcarry = jmax;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < V; ++i) qa[u][i] = qn[u][i];
    }
    if (wb >= we && itn < nitems) load_batch(In, wbn, wen, qa);  // warp had no work in this item
    __syncthreads();  // everyone is done with K/T (and raw stage s) of item `it`
    if (!PACKED && threadIdx.x == 0) issue(it + 2 * G, s);
    I = In;
    wb = wbn;
    we = wen;
    s ^= 1;
  }
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
