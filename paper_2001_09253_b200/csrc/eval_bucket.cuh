// eval_bucket.cuh -- evaluation of ONE very long curve with many unsorted queries (BASELINE cfg5)
// with the queries bucketed by L2-sized chunks of the curve.
//
// On a curve whose x, y, y2 (3 s B per knot: 1.5 GB for cfg5) dwarf the 126 MB L2, every
// unsorted query costs a random DRAM access (the interval-record path, k_eval_records, runs at
// the HBM random-access rate: DESIGN.md).  Here the queries are first grouped by the chunk of
// K consecutive intervals they fall in (the GPU analogue of the paper's cache "goose neck",
// keep the working set in the fast level), each chunk is then evaluated while its
// 3 s K bytes sit in L2, and the results are put back in query order:
//
//   A1 k_bucket_count   per tile of kBkTile queries: the bucket of each query (chunk boundary
//                       x_{bK} comparisons after a guess; nb = out of range / NaN) and the
//                       tile's count per bucket, stored bucket-major: cnt[b * ntiles + t].
//   S  k_scan_*         exclusive scan of cnt in that order: the global bucket-major position
//                       of every (bucket, tile) run (block-level scan + a scan of block sums).
//   A2 k_bucket_scatter the same buckets again, a tile-local counting sort in shared memory,
//                       each run written to its global position (qs: queries bucket-major) and
//                       the query of each tile slot (perm, u16, tile-local order).
//   B  k_bucket_eval    ONE flat pass over qs in bucket-major order (blocks dispatched in
//                       order, so the GPU works on ~one chunk at a time): interpolation guess,
//                       galloping correction (the locate rule's answer on any grid), Eq.
//                       nr_formula in the factored form (bitwise the other eval kernels');
//                       results in the same bucket-major order (coalesced).  Each block
//                       prefetches (cp.async.bulk.prefetch.L2) its share of the NEXT chunk's knots.
//   C  k_bucket_gather  per tile: its runs found from the scanned counts (run (b, t) spans
//                       [start(b ntiles + t), start(b ntiles + t + 1)); its tile-local slots
//                       start at the sum of the tile's earlier runs), read back (contiguous
//                       runs), scattered to query order through perm in shared memory, written
//                       coalesced.  No per-query destination array.
//
// Algorithmic bytes are those of any eval ((2s+4) B/query + 3 s B/knot); this path moves the
// q-sized arrays a few more times, but every access is a stream, a contiguous run or an L2 hit
// instead of a random DRAM access.
#pragma once
#include "eval.cuh"

namespace fs {

#ifndef FS_BK_CNT_MINB
#define FS_BK_CNT_MINB 3  // A/B cfg5 eval: 9.18 ms at 3/3 vs 9.34 at 2/2 (count, scatter)
#endif
#ifndef FS_BK_SC_MINB
#define FS_BK_SC_MINB 3
#endif
constexpr int kBkTile = 4096;         // queries per tile (tile-local slots fit u16)
constexpr int kBkThreads = 256;
constexpr int kBkScThreads = 512;     // count / scatter / gather: 8 queries per thread
constexpr int kBkPerThread = kBkTile / kBkScThreads;
constexpr int kBkMaxBuckets = 512;    // in-range chunks per curve (+1 bucket: out of range / NaN)
#ifndef FS_BK_EVAL_ITERS
#define FS_BK_EVAL_ITERS 8
#endif
constexpr int kBkEvalIters = FS_BK_EVAL_ITERS;  // rounds of the flat evaluation per block
#ifndef FS_BK_EVAL_U
#define FS_BK_EVAL_U 2  // A/B cfg5 eval (with kBkSpec): U2 x 8 rounds 8.38 ms, U4 x 4 11.08 (spills), U1 x 16 8.42, U2 x 4 8.62
#endif
constexpr int kBkEvalPer = kBkThreads * FS_BK_EVAL_U * kBkEvalIters;  // queries per block of the flat evaluation (U per thread and round)
constexpr int kScanBlock = 4096;      // elements per block of the run-offset scan (4 per thread)

// bucket of q: b in [0, nb) with x_{bK} <= q < x_{(b+1)K} (the last bucket ends at x_{n-1}
// inclusive); nb for q outside [x_0, x_{n-1}] or NaN.  xb[0..nb-1] = x_{bK}, xb[nb] = x_{n-1};
// xp[b] = {xb[b], xb[b+1]} (one vector load for the guess's test); lo = x_0, hi = x_{n-1} in
// registers.  From the guess g = (q - x_0) sb (exact up to a step on near-uniform grids),
// verified against the boundaries, else a bisection: exact on any grid.
template <typename T> struct alignas(2 * sizeof(T)) BkPair { T a, b; };
template <typename T>
__device__ __forceinline__ int bucket_of_q(const T *xb, const BkPair<T> *xp, int nb, T q, T lo, T hi, T sb) {
  if (!(q >= lo && q <= hi)) return nb;
  const int g = max(0, min((int)((q - lo) * sb), nb - 1));
  const BkPair<T> pr = xp[g];
  if (pr.a <= q && (q < pr.b || g == nb - 1)) return g;  // the guess holds (near-uniform grids)
  int l = 0, h = nb;  // xb[l] <= q, and h == nb or xb[h] > q
  while (h - l > 1) {
    const int mid = (l + h) >> 1;
    if (xb[mid] <= q) l = mid;
    else h = mid;
  }
  return l;
}

// The chunk boundaries (and their pairs) in shared memory; returns the bucket guess scale.
template <typename T>
__device__ __forceinline__ T load_bounds(T *xb, BkPair<T> *xp, const T *__restrict__ x, int n, int64_t K, int nb) {
  for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
    const T v = (b < nb) ? __ldg(x + (int64_t)b * K) : __ldg(x + n - 1);
    xb[b] = v;
    if (b < nb) xp[b] = BkPair<T>{v, (b + 1 < nb) ? __ldg(x + (int64_t)(b + 1) * K) : __ldg(x + n - 1)};
  }
  return (T)(n - 1) / ((__ldg(x + n - 1) - __ldg(x)) * (T)K);  // buckets per unit of x (a guess)
}

template <typename T>
__global__ void __launch_bounds__(kBkScThreads, FS_BK_CNT_MINB) k_bucket_count(const T *__restrict__ x, int n, int64_t K, int nb,
                                                                  const T *__restrict__ q, int64_t m,
                                                                  int *__restrict__ cnt) {
  pdl_wait();
  __shared__ T xb[kBkMaxBuckets + 1];
  __shared__ BkPair<T> xp[kBkMaxBuckets];
  __shared__ int c[kBkMaxBuckets + 1];
  const int64_t ntiles = (m + kBkTile - 1) / kBkTile;
  const int64_t tile = blockIdx.x;
  const int64_t q0 = tile * kBkTile;
  const int nq = (int)min64(kBkTile, m - q0);
  const T sb = load_bounds(xb, xp, x, n, K, nb);
  const T lo = __ldg(x), hi = __ldg(x + n - 1);
  for (int b = threadIdx.x; b <= nb; b += kBkScThreads) c[b] = 0;
  T qv[kBkPerThread];
#pragma unroll
  for (int u = 0; u < kBkPerThread; ++u) {
    const int i = u * kBkScThreads + threadIdx.x;
    qv[u] = (i < nq) ? ld_stream(q + q0 + i) : T(0);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kBkPerThread; ++u)
    if (u * kBkScThreads + (int)threadIdx.x < nq) atomicAdd(&c[bucket_of_q(xb, xp, nb, qv[u], lo, hi, sb)], 1);
  __syncthreads();
  for (int b = threadIdx.x; b <= nb; b += kBkScThreads) cnt[(int64_t)b * ntiles + tile] = c[b];
}

// Exclusive scan of L ints in place, in blocks of kScanBlock; the block totals go to bsum and are
// scanned by k_scan_top (one CTA); consumers add bsum[i / kScanBlock] themselves.
__global__ void __launch_bounds__(1024) k_scan_blocks(int *__restrict__ a, int64_t L, int *__restrict__ bsum) {
  __shared__ int ws[32];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + 4 * threadIdx.x;
  int v[4], s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = (base + k < L) ? a[base + k] : 0;
    s += v[k];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    int t = ws[lane], ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += u;
    }
    ws[lane] = ti - t;
    if (lane == 31) bsum[blockIdx.x] = ti;
  }
  __syncthreads();
  int run = ws[w] + inc - s;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (base + k < L) a[base + k] = run;
    run += v[k];
  }
}
__global__ void __launch_bounds__(1024) k_scan_top(int *__restrict__ bsum, int nblk) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int b0 = 0; b0 < nblk; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const int v = (i < nblk) ? bsum[i] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
      int t = ws[lane], ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      ws[lane] = ti - t;
    }
    __syncthreads();
    const int c0 = carry;
    if (i < nblk) bsum[i] = c0 + ws[w] + inc - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + ws[31] + inc;
    __syncthreads();
  }
}

template <typename T> constexpr size_t bucket_scatter_smem() {
  return sizeof(T) * (kBkTile + kBkMaxBuckets + 1) + sizeof(BkPair<T>) * kBkMaxBuckets +
         sizeof(int) * (2 * kBkMaxBuckets + 3) + 2 * 2 * kBkTile;
}
template <typename T> constexpr size_t bucket_gather_smem() {
  return (sizeof(T) + 4) * kBkTile + (sizeof(int64_t) + sizeof(int)) * (kBkMaxBuckets + 1);
}

template <typename T>
__global__ void __launch_bounds__(kBkScThreads, FS_BK_SC_MINB) k_bucket_scatter(const T *__restrict__ x, int n, int64_t K, int nb,
                                                                    const T *__restrict__ q, int64_t m,
                                                                    const int *__restrict__ goff,
                                                                    const int *__restrict__ bsum,
                                                                    T *__restrict__ qs,
                                                                    uint16_t *__restrict__ perm) {
  extern __shared__ __align__(16) unsigned char bk_smem[];  // bucket_scatter_smem<T>() bytes
  T *sq = reinterpret_cast<T *>(bk_smem);                          // [kBkTile]
  BkPair<T> *xp = reinterpret_cast<BkPair<T> *>(sq + kBkTile);  // [kBkMaxBuckets] (16/8-byte aligned)
  T *xb = reinterpret_cast<T *>(xp + kBkMaxBuckets);               // [kBkMaxBuckets + 1]
  int *c = reinterpret_cast<int *>(xb + kBkMaxBuckets + 1);        // counts, then the run starts
  int *gb = c + kBkMaxBuckets + 2;                                 // global base of each run
  uint16_t *sp = reinterpret_cast<uint16_t *>(gb + kBkMaxBuckets + 1);
  uint16_t *sbk = sp + kBkTile;
  const int tid = threadIdx.x;
  const int64_t ntiles = (m + kBkTile - 1) / kBkTile;
  const int64_t tile = blockIdx.x;
  const int64_t q0 = tile * kBkTile;
  const int nq = (int)min64(kBkTile, m - q0);
  const T sb = load_bounds(xb, xp, x, n, K, nb);
  const T lo = __ldg(x), hi = __ldg(x + n - 1);
  for (int b = tid; b <= nb + 1; b += kBkScThreads) c[b] = 0;
  for (int b = tid; b <= nb; b += kBkScThreads) {
    const int64_t e = (int64_t)b * ntiles + tile;
    gb[b] = goff[e] + bsum[e / kScanBlock];
  }
  T qv[kBkPerThread];
  int bk[kBkPerThread], rk[kBkPerThread];
#pragma unroll
  for (int u = 0; u < kBkPerThread; ++u) {
    const int i = u * kBkScThreads + tid;
    qv[u] = (i < nq) ? ld_stream(q + q0 + i) : T(0);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kBkPerThread; ++u) {
    if (u * kBkScThreads + tid < nq) {
      bk[u] = bucket_of_q(xb, xp, nb, qv[u], lo, hi, sb);
      rk[u] = atomicAdd(&c[bk[u]], 1);  // rank inside the run (any order: results go back by perm)
    }
  }
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the nb + 1 counts by one warp
    int carry = 0;
    for (int b0 = 0; b0 <= nb; b0 += 32) {
      const int b = b0 + tid;
      const int v = (b <= nb) ? c[b] : 0;
      int s = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, s, o);
        if (tid >= o) s += t;
      }
      if (b <= nb) c[b] = carry + s - v;
      carry += __shfl_sync(0xffffffffu, s, 31);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kBkPerThread; ++u) {
    const int i = u * kBkScThreads + tid;
    if (i < nq) {
      const int s = c[bk[u]] + rk[u];
      sq[s] = qv[u];
      sp[s] = (uint16_t)i;
      sbk[s] = (uint16_t)bk[u];
    }
  }
  __syncthreads();
  for (int s = tid; s < nq; s += kBkScThreads) {
    const int b = sbk[s];
    const int64_t p = gb[b] + (s - c[b]);  // consecutive slots of a run: consecutive addresses
    st_stream(qs + p, sq[s]);
    perm[q0 + s] = sp[s];                  // the query of the tile's slot s
  }
}


// Knots interleaved for the evaluation: {x_j, y_j, y2_j, 0} (32 B fp64: one sector per knot), so an
// interval is two 32-byte loads instead of six scattered 8-byte ones.
template <typename T> struct alignas(4 * sizeof(T)) Knot { T x, y, z, pad; };

// The packing also measures how far the knots stray from the evaluation's interval guess
// f(q) = (q - x_0) (n-1) / (x_{n-1} - x_0): dev = max_j |f(x_j) - j| (atomicMax on the bits of a
// non-negative double into *dev, which the caller zeroes).  A query whose f lies farther than dev
// from every integer is inside the guessed interval, so k_bucket_eval loads the guess's neighbour
// knot only for the queries within dev of a cell boundary.
template <typename T>
__global__ void __launch_bounds__(256) k_pack_knots(const T *__restrict__ x, const T *__restrict__ y,
                                                    const T *__restrict__ y2, int64_t n, Knot<T> *__restrict__ kn,
                                                    unsigned long long *__restrict__ dev) {
  const double x0 = (double)__ldg(x), sc = (double)(n - 1) / ((double)__ldg(x + n - 1) - x0);
  double dmax = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    T v[4] = {ld_stream(x + j), ld_stream(y + j), ld_stream(y2 + j), T(0)};
    if constexpr (sizeof(T) == 8) st256(kn + j, reinterpret_cast<const double(&)[4]>(v));
    else *reinterpret_cast<float4 *>(kn + j) = make_float4(v[0], v[1], v[2], v[3]);
    const double d = fabs(((double)v[0] - x0) * sc - (double)j);
    dmax = (d > dmax || d != d) ? d : dmax;  // NaN knots: NaN (the eval then loads the neighbour always)
  }
  if (dev) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, dmax, o);
      dmax = (t > dmax || t != t) ? t : dmax;
    }
    if ((threadIdx.x & 31) == 0) {
      const double d = (dmax != dmax || dmax > 1.0) ? 1.0 : dmax;  // >= 0.5: every query is "near a boundary"
      atomicMax(dev, (unsigned long long)__double_as_longlong(d));
    }
  }
}
template <typename T> __device__ __forceinline__ Knot<T> ld_knot(const Knot<T> *p) {
  Knot<T> k;
  if constexpr (sizeof(T) == 8) {
    double v[4];
    ld256(p, v);
    k = Knot<T>{v[0], v[1], v[2], v[3]};
  } else {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(p));
    k = Knot<T>{v.x, v.y, v.z, v.w};
  }
  return k;
}

// The flat evaluation of the bucket-major queries; results in the same bucket-major order
// (coalesced; k_bucket_gather finds each tile's runs from the scan of the run counts).
#ifndef FS_BK_SPEC
#define FS_BK_SPEC 1  // A/B cfg5 eval: 8.38 vs 9.13 ms without (a miss of the guess costs no second round)
#endif
constexpr bool kBkSpec = FS_BK_SPEC != 0;  // the guess's likely neighbour knot loaded in the first round
#ifndef FS_BK_EVAL_MINB
#define FS_BK_EVAL_MINB 3
#endif
template <typename T>
__global__ void __launch_bounds__(kBkThreads, FS_BK_EVAL_MINB) k_bucket_eval(unsigned *__restrict__ status, const Knot<T> *__restrict__ kn,
                                                            int n, int64_t K, int nb, int64_t m,
                                                            const int *__restrict__ goff, const int *__restrict__ bsum,
                                                            const T *__restrict__ qs,
                                                            T *__restrict__ os, int32_t *__restrict__ is,
                                                            const unsigned long long *__restrict__ dev) {
  constexpr int U = kBkEvalPer / kBkEvalIters / kBkThreads;  // independent queries per thread in flight
  const int64_t ntiles = (m + kBkTile - 1) / kBkTile;
  const int64_t p0 = (int64_t)blockIdx.x * kBkEvalPer;
  if (threadIdx.x == 0) {
    // the bucket of this block's first position, then this block's share of the next chunk
    auto bstart = [&](int b) -> int64_t {
      if (b > nb) return m;
      const int64_t e = (int64_t)b * ntiles;
      return (int64_t)__ldg(goff + e) + __ldg(bsum + e / kScanBlock);
    };
    int lo = 0, hi = nb + 1;  // bstart(lo) <= p0 < bstart(hi)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (bstart(mid) <= p0) lo = mid;
      else hi = mid;
    }
    const int c = lo + 1;  // the next chunk
    if (lo < nb && c < nb) {
      const int64_t bs = bstart(lo), be = bstart(lo + 1);
      const int64_t c0 = (int64_t)c * K, c1 = min64((int64_t)(c + 1) * K + 1, (int64_t)n);
      const double f0 = (double)(p0 - bs) / (double)max((int64_t)1, be - bs);
      const double f1 = (double)(p0 + kBkEvalPer - bs) / (double)max((int64_t)1, be - bs);
      const int64_t s0 = c0 + (int64_t)(f0 * (double)(c1 - c0));
      const int64_t s1 = min64(c1, c0 + (int64_t)(f1 * (double)(c1 - c0)) + 1);
      if (s1 > s0) prefetch_l2_bulk(kn + s0, (uint32_t)((s1 - s0) * sizeof(Knot<T>)));
    }
  }
  const T x0 = __ldg(&kn[0].x), xn = __ldg(&kn[n - 1].x);
  const T sc = (T)(n - 1) / (xn - x0);
  // the band around the cell boundaries where the guess can miss (k_pack_knots' deviation, plus
  // a margin for the rounding of f in either precision); outside it only the guess's two knots
  // are loaded.  A miss outside the band (impossible up to that margin) still takes the general
  // correction below, so the band only decides speed.
  const double margin = 1e-3 + 8.0 * (double)n * (sizeof(T) == 8 ? 1.1102230246251565e-16 : 5.9604644775390625e-08);
  const T band = dev ? (T)fmin(__longlong_as_double((long long)__ldg(dev)) + margin, 0.5) : T(0.5);
  bool oor = false;
  // the block's positions in kBkEvalIters rounds of U per thread; the next round's queries and
  // the next round's queries are loaded before this round's knots are (two streams in flight)
  T qn[U];

#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t p = p0 + u * kBkThreads + threadIdx.x;
    qn[u] = (p < m) ? ld_stream(qs + p) : x0;
  }
  for (int it = 0; it < kBkEvalIters; ++it) {
    const int64_t pb = p0 + (int64_t)it * kBkThreads * U;
    if (pb >= m) break;
    T qq[U];
    int j[U];
    bool in[U];
    Knot<T> ka[U], kb[U], kc[U];
    bool up[U], risky[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const T v = qn[u];
      in[u] = (v >= x0) && (v <= xn);
      qq[u] = in[u] ? v : x0;
      const T f = r_mul(r_sub(qq[u], x0), sc);
      j[u] = max(0, min((int)f, n - 2));
      const T fr = f - (T)j[u];
      up[u] = fr >= T(0.5);  // which neighbour a miss of the guess most likely needs
      risky[u] = !(fr > band && fr < T(1) - band);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ka[u] = ld_knot(kn + j[u]);
      kb[u] = ld_knot(kn + j[u] + 1);
      // the likely neighbour in the same round (kBkSpec), for the queries near a cell boundary:
      // knot j-1 below the guess's middle, knot j+2 above it (clamped into the curve; only used
      // when it is the right one)
      if (kBkSpec && risky[u]) kc[u] = ld_knot(kn + (up[u] ? min(j[u] + 2, n - 1) : max(j[u] - 1, 0)));
    }
    if (it + 1 < kBkEvalIters) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = pb + (int64_t)kBkThreads * U + u * kBkThreads + threadIdx.x;
        qn[u] = (p < m) ? ld_stream(qs + p) : x0;
          }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kBkSpec && risky[u] && !(ka[u].x <= qq[u] && (qq[u] < kb[u].x || j[u] == n - 2))) {
        if (!up[u] && ka[u].x > qq[u] && j[u] > 0 && kc[u].x <= qq[u]) {  // one interval down
          j[u] -= 1;
          kb[u] = ka[u];
          ka[u] = kc[u];
        } else if (up[u] && !(ka[u].x > qq[u]) && j[u] + 2 <= n - 1 && qq[u] < kc[u].x) {  // one up
          j[u] += 1;
          ka[u] = kb[u];
          kb[u] = kc[u];
        }
      }
      if (!(ka[u].x <= qq[u] && (qq[u] < kb[u].x || j[u] == n - 2))) {  // the guess missed
        if (ka[u].x > qq[u] && j[u] > 0 && __ldg(&kn[j[u] - 1].x) <= qq[u]) {
          j[u] -= 1;  // one interval down (the usual miss on a jittered grid)
        } else if (!(ka[u].x > qq[u]) && j[u] + 2 <= n - 1 && qq[u] < __ldg(&kn[j[u] + 2].x)) {
          j[u] += 1;  // one interval up
        } else {      // any grid: bisection over the knots
          int lo = 0, hi = n - 1;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(&kn[mid].x) <= qq[u]) lo = mid;
            else hi = mid;
          }
          j[u] = lo;
        }
        ka[u] = ld_knot(kn + j[u]);
        kb[u] = ld_knot(kn + j[u] + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = pb + u * kBkThreads + threadIdx.x;
      if (p < m) {
        const T v = nr_interp(qq[u], ka[u].x, kb[u].x, ka[u].y, kb[u].y, ka[u].z, kb[u].z);
        st_stream(os + p, in[u] ? v : qnan<T>());
        if (is) st_stream(is + p, in[u] ? j[u] : -1);
        oor |= !in[u];
      }
    }
  }
  raise_status_warp(status, oor, kOutOfRange);
}

#ifndef FS_BK_GATHER_THREADS
#define FS_BK_GATHER_THREADS 512
#endif
constexpr int kBkGaThreads = FS_BK_GATHER_THREADS;  // the gather's CTA
// Tile t's results sit in nb + 1 runs of the bucket-major arrays: run (b, t) starts at the
// scanned offset of cnt entry e = b ntiles + t and ends where entry e + 1 starts (the scan is
// exclusive and bucket-major, so runs of one bucket follow each other tile by tile); inside
// the tile, bucket b's slots start at the sum of the tile's earlier runs -- the tile-local
// counting sort of k_bucket_scatter.  The gather copies the runs back through perm (slot ->
// query) into shared memory and writes the tile's results in query order, coalesced.
template <typename T>
__global__ void __launch_bounds__(kBkGaThreads, 2048 / kBkGaThreads) k_bucket_gather(const T *__restrict__ os, const int32_t *__restrict__ is,
                                                                   const uint16_t *__restrict__ perm, int64_t m,
                                                                   const int *__restrict__ goff, const int *__restrict__ bsum,
                                                                   int nb, T *__restrict__ out, int32_t *__restrict__ idx) {
  extern __shared__ __align__(16) unsigned char bk_smem[];  // bucket_gather_smem<T>() bytes
  T *so = reinterpret_cast<T *>(bk_smem);                          // [kBkTile]
  int32_t *si = reinterpret_cast<int32_t *>(so + kBkTile);         // [kBkTile]
  int64_t *gs = reinterpret_cast<int64_t *>(si + kBkTile);        // [kBkMaxBuckets + 1] global run starts
  int *ls = reinterpret_cast<int *>(gs + kBkMaxBuckets + 1);       // [kBkMaxBuckets + 1] tile-local run starts
  const int64_t ntiles = (m + kBkTile - 1) / kBkTile;
  const int64_t tile = blockIdx.x;
  const int64_t q0 = tile * kBkTile;
  const int nq = (int)min64(kBkTile, m - q0);
  const int64_t L = (int64_t)(nb + 1) * ntiles;
  auto start = [&](int64_t e) -> int64_t { return e >= L ? m : (int64_t)goff[e] + bsum[e / kScanBlock]; };
  const int tid = threadIdx.x;
  for (int b = tid; b <= nb; b += kBkGaThreads) {
    const int64_t e = (int64_t)b * ntiles + tile;
    const int64_t g = start(e);
    gs[b] = g;
    ls[b] = (int)(start(e + 1) - g);  // the run's length (its end: the next entry's start)
  }
  __syncthreads();
  if (tid < 32) {  // tile-local starts: exclusive scan of the run lengths (one warp)
    int carry = 0;
    for (int b0 = 0; b0 <= nb; b0 += 32) {
      const int b = b0 + tid;
      const int v = (b <= nb) ? ls[b] : 0;
      int sc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t2 = __shfl_up_sync(0xffffffffu, sc, o);
        if (tid >= o) sc += t2;
      }
      if (b <= nb) ls[b] = carry + sc - v;
      carry += __shfl_sync(0xffffffffu, sc, 31);
    }
  }
  __syncthreads();
  // each warp copies whole runs (buckets w, w + 16, ...): coalesced reads of the run, the
  // results land at their queries' places in shared memory
  const int lane = tid & 31, w = tid >> 5;
  for (int b = w; b <= nb; b += kBkGaThreads / 32) {
    const int64_t g = gs[b];
    const int s0 = ls[b];  // (bucket b's slots in the tile: [s0, s0 + run length))
    const int ln = (b < nb ? ls[b + 1] : nq) - s0;
    for (int r = lane; r < ln; r += 32) {
      const int i = perm[q0 + s0 + r];
      so[i] = ld_stream(os + g + r);
      if (idx) si[i] = __ldcs(is + g + r);
    }
  }
  __syncthreads();
  for (int i = tid; i < nq; i += kBkGaThreads) {
    st_stream(out + q0 + i, so[i]);
    if (idx) st_stream(idx + q0 + i, si[i]);
  }
}

}  // namespace fs
