// eval.cuh -- fused locate + evaluate kernels.
//
// Locate rule (reading c1): idx = the largest j in [0, n-2] with x_j <= q;
// -1 (and out = NaN, status bit) when q is outside [x_0, x_{n-1}] or NaN, because
// Eq. nr_formula only holds for x_j <= x <= x_{j+1}.  Every search below ends in
// comparisons against this rule, so guesses (bucket table, uniform-grid index, sorted-run
// carry, interpolation guess) change speed, never idx.
// Evaluate: Eq. nr_formula in the factored form of common.cuh (Cub: make_cub,
// cub_eval; explicitly rounded, so all kernels and hints give bitwise-identical out).
//
//  k_eval_staged : unsorted queries on curves that fit in shared memory.  Persistent CTAs,
//                  TMA bulk staging (double-buffered), packed interval records:
//                    MODE_BISECT  -- branch-free bisection over +inf-padded knots (short curves)
//                    MODE_TABLE   -- per-curve bucket table brackets each query
//                    MODE_UNIFORM -- direct index (q-x_0)(n-1)/(x_{n-1}-x_0), corrected
//                    MODE_BSEARCH -- bisection on the raw arrays (curves too big to pack)
//  k_eval_warps  : the same stages with per-warp curve ownership (no CTA barrier in the loop).
//  k_eval_curvewarp : n <= 64, many curves: one warp per curve, knots loaded directly (next
//                  curve prefetched), records + Eytzinger keys in a per-warp table.
//  k_eval_small  : fp32 n <= 8, m <= 32: a warp per 32 curves, per-lane record build; its
//                  SOLVE form also runs K1r's sweep (spline_build_eval).
//  k_build_eval_tiny : spline_build_eval on a few K1h-sized curves, one CTA per curve.
//  k_eval_sorted : SPLINE_Q_SORTED.  A warp walks a contiguous run of queries with a
//                  carried bracket (the paper's forward scan, made
//                  warp-cooperative); dense runs keep a window of interval records in
//                  shared memory, sparse runs read knots through L1, any n.
//  k_pack_records + k_eval_records : unsorted queries on long curves: interval records in
//                  an HBM workspace, one gather per query at the interpolation guess.
#pragma once
#include "build_thomas.cuh"
#include "common.cuh"

namespace fs {

enum { MODE_BSEARCH = 0, MODE_BISECT = 1, MODE_UNIFORM = 2, MODE_TABLE = 3 };

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

template <typename T>
__device__ __forceinline__ void eval_one(const T *X, const T *Y, const T *Z, int n, T q, T &val, int &j) {
  const T x0 = X[0], xn = X[n - 1];
  if (!(q >= x0 && q <= xn)) {  // out of range or NaN
    j = -1;
    val = qnan<T>();
    return;
  }
  j = bisect(X, n, q);
  val = nr_interp(q, X[j], X[j + 1], Y[j], Y[j + 1], Z[j], Z[j + 1]);
}

// ---- packed curves (MODE_BISECT, MODE_TABLE, MODE_UNIFORM) ------------------------------
// Per staged curve: interval j's Cub {1/h, y0, dy, e1} (common.cuh; 16 B fp32: ONE 16-byte
// shared-memory load) and its e2 (one 4-byte load), and -- for the modes that check a bracket --
// the plain knot array XK.  Slots have stride n per curve (slot n-1 unused).
//   MODE_BISECT : branch-free bisection over the knots in Eytzinger order (eytz_descend):
//                 L2 = ceil(log2(n-1)) uniform steps, no divergence, conflict-free; x_lo is
//                 the last key the descent went right of (no extra load).
//   MODE_TABLE  : bucket table over nb = 2n equal-width buckets of [x_0, x_{n-1}]:
//                   bucket(v) = min(nb, (int)((v - x_0) * s)),   s = nb / (x_{n-1} - x_0)
//                   Tb[b]     = max{ j in [0, n-2] : bucket(x_j) < b }   (Tb[0] = 0).
//                 bucket() is monotone in v, so for an in-range query q in bucket b the
//                 answer j* = max{ j : x_j <= q } satisfies Tb[b] <= j* <= Tb[b+1]: the
//                 table only brackets the search (long curves, many queries per knot).
//   MODE_UNIFORM: direct index (q - x_0)(n-1)/(x_{n-1} - x_0) on the hinted uniform grid.
// Every search ends in comparisons x_j <= q, so idx is exact on any grid.
// Per staged curve: range and scale (one vector load per group of V queries).
template <typename T> struct CurveHdr { T x0, xn, s, pad; };

constexpr int kBucketsPerKnot = 2;

template <typename T> __device__ __forceinline__ int bucket_of(T v, T x0, T s, int nb) {
  const T f = r_mul(r_sub(v, x0), s);
  return (f >= T(0)) ? min((int)f, nb) : 0;  // (int) truncates; f >= 0 here
}

// MODE_BISECT search structure: the keys x_1 .. x_{n-2} (padded with +inf to 2^L2 - 1 keys,
// 2^L2 >= n-1) in Eytzinger (breadth-first) order, E[1 .. 2^L2 - 1], E[i]'s children at 2i,
// 2i+1.  A branch-free descent i <- 2i + (E[i] <= q) of exactly L2 steps ends at
// i = 2^L2 + c with c = #{keys <= q}: for x_0 <= q <= x_{n-1} that is the locate rule's
// answer, the largest j in [0, n-2] with x_j <= q (x_{n-1} is deliberately not a key).
// Level t of the tree is 2^t consecutive words, so the probes of a warp hit distinct banks.
__host__ __device__ constexpr int eytz_levels(int n) {
  int l = 2;
  while ((1 << l) < n - 1) ++l;
  return l;
}
__device__ __forceinline__ float lds_f(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f(uint32_t a, double) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// The descent on shared-memory byte addresses a = ebase + s i: a <- 2a - ebase (+ s when
// E[i] <= q), one load, one compare and two integer adds per level (+ one select tracking the
// last key <= q, which is x_c).  Returns the final a, = ebase + s (2^L2 + c); xl = x_c, or the
// caller's x_0 when c = 0.
template <typename T, int L2> __device__ __forceinline__ uint32_t eytz_descend(uint32_t ebase, T q, T &xl) {
  uint32_t a = ebase + (uint32_t)sizeof(T);
#pragma unroll
  for (int t = 0; t < L2; ++t) {
    T v;
    if constexpr (sizeof(T) == 4) v = lds_f(a);
    else v = lds_f(a, 0.0);
    a = 2u * a - ebase;
    if (v <= q) {
      a += (uint32_t)sizeof(T);
      xl = v;
    }
  }
  return a;
}

// in-order rank (0-based) of breadth-first node i (1-based) in a complete tree of depth L2
__device__ __forceinline__ int eytz_rank(int i, int L2) {
  int d = 31 - __clz(i);  // depth
  return ((2 * (i - (1 << d)) + 1) << (L2 - 1 - d)) - 1;
}

// Locate + evaluate one query against a packed curve (cubics Pc + Ec2, knots Xc (not for
// MODE_BISECT), Eytzinger keys at shared address ebase).  Branch-light: out-of-range / NaN
// queries run the same path on a clamped stand-in (qc = x_0) and are masked at the end.
template <typename T, int MODE, int L2>
__device__ __forceinline__ void eval_packed(const Cub<T> *Pc, const T *Ec2, const T *Xc, uint32_t ebase,
                                            const uint16_t *Tb, const CurveHdr<T> &hd, int n, int nb, T q, T &val,
                                            int &j) {
  const T qc = fmin(fmax(q, hd.x0), hd.xn);  // NaN -> x_0 (fmax returns the number)
  const bool in = (qc == q);                 // false for NaN and for q outside [x_0, x_{n-1}]
  int lo;
  T xl;
  if (MODE == MODE_BISECT) {
    xl = hd.x0;
    const uint32_t a = eytz_descend<T, L2>(ebase, qc, xl);
    // (the clamp only matters for invalid knots, e.g. x_{n-1} = +inf: memory safety)
    lo = min((int)((a - ebase) / (uint32_t)sizeof(T)) - (1 << L2), n - 2);
  } else if (MODE == MODE_UNIFORM) {
    // direct index on the hinted grid; accepted only if x_g <= q < x_{g+1} (or g = n-2, i.e.
    // x_{g+1} = x_{n-1}), so rounding or a wrong hint costs a (rare) bisection, never a wrong idx
    lo = max(0, min((int)r_mul(r_sub(qc, hd.x0), hd.s), n - 2));
    xl = Xc[lo];
    const T xb = Xc[lo + 1];
    const bool miss = !(xl <= qc && (qc < xb || xb == hd.xn));
    if (__any_sync(__activemask(), miss) && miss) {  // warp-uniform test: no divergence bookkeeping
      int l = 0, h = n - 1;
      while (h - l > 1) {
        const int mid = (l + h) >> 1;
        if (Xc[mid] <= qc) l = mid;
        else h = mid;
      }
      lo = l;
      xl = Xc[lo];
    }
  } else {  // MODE_TABLE
    const int bk = bucket_of(qc, hd.x0, hd.s, nb);
    lo = min((int)Tb[bk], n - 2);  // clamps keep invalid (non-monotone) knots memory-safe
    int hi = max(lo, min((int)Tb[bk + 1], n - 2));
    if (hi - lo > 2) {  // wide bracket (clustered knots): bisect it down
      do {
        const int mid = (lo + hi + 1) >> 1;
        if (Xc[mid] <= qc) lo = mid;
        else hi = mid - 1;
      } while (hi - lo > 2);
    }
    while (lo < hi && Xc[lo + 1] <= qc) ++lo;  // largest j in [lo, hi] with x_j <= q
    xl = Xc[lo];
  }
  const T v = cub_eval<T>(Pc[lo], Ec2[lo], xl, qc);
  j = in ? lo : -1;
  val = in ? v : qnan<T>();
}

constexpr int kEvalThreads = 256;
constexpr int kStageHeader = 32;  // two mbarriers + two counters, ahead of the staged arrays

__host__ __device__ constexpr size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

// Shared-memory layout of one CTA: two stages, each holding an item's raw x, y, y2 (cpb
// curves) and -- when queries are staged too -- its up to qmax queries, all filled by TMA bulk
// copies; plus the packed knots / headers / Eytzinger keys / bucket table of the item being
// evaluated.
template <typename T> struct StageLayout {
  size_t raw0, rawstep, qoff, knots, e2, xk, hdr, xs, table, total;
  int P;  // Eytzinger array stride per curve (MODE_BISECT): 2^L2 >= n - 1
  __host__ __device__ StageLayout(int cpb, int n, int mode, int qmax) {
    const bool packed = mode != MODE_BSEARCH;
    P = 1 << eytz_levels(n);
    const size_t rawb = 3 * sizeof(T) * (size_t)cpb * n;
    raw0 = kStageHeader;
    qoff = align16(rawb);
    rawstep = align16(qoff + sizeof(T) * (size_t)qmax);
    size_t off = raw0 + 2 * rawstep;
    knots = off;
    if (packed) off = align16(off + sizeof(Cub<T>) * (size_t)cpb * n);
    e2 = off;
    if (packed) off = align16(off + sizeof(T) * (size_t)cpb * n);
    xk = off;
    if (packed && mode != MODE_BISECT) off = align16(off + sizeof(T) * (size_t)cpb * n);
    hdr = off;
    if (packed) off = align16(off + sizeof(CurveHdr<T>) * (size_t)cpb);
    xs = off;
    if (mode == MODE_BISECT) off = align16(off + sizeof(T) * (size_t)cpb * P);
    table = off;
    if (mode == MODE_TABLE) off = align16(off + sizeof(uint16_t) * (size_t)cpb * (kBucketsPerKnot * n + 2));
    total = off;
  }
};

// Packing pass of one staged item: nc curves with raw knots X, Y (curve-major, stride n) and
// second derivatives Z (row stride zs) become {x, y, y2, 1/h} records K, headers Hd and the
// mode's search structure (Eytzinger keys Xs with stride P, or the bucket table Tb).
// Threads tid = 0 .. nt-1 of the caller's group share the work.
template <typename T, int MODE, int L2>
__device__ __forceinline__ void pack_item(const T *X, const T *Y, const T *Z, int zs, int nc, int n, int nb,
                                          FastDiv divn, Cub<T> *RP, T *RE, T *XK, CurveHdr<T> *Hd, T *Xs,
                                          uint16_t *Tb, int P, int tid, int nt) {
  const int tot = nc * n;
  for (int e = tid; e < tot; e += nt) {
    const int c = (int)divn.div((uint32_t)e);
    const int j = e - c * n;
    const T xj = X[e];
    if (MODE != MODE_BISECT) XK[e] = xj;
    if (j < n - 1) {
      const T *zc = Z + c * zs + j;
      RP[e] = make_cub<T>(xj, X[e + 1], Y[e], Y[e + 1], zc[0], zc[1], RE[e]);
    }
    if (j == 0 || (MODE == MODE_TABLE && j < n - 1)) {
      const T x0 = X[c * n], xn = X[c * n + n - 1];
      // (the scale only steers a guess that is always verified: any positive value is exact)
      const T sc = r_mul((MODE == MODE_TABLE) ? (T)nb : (T)(n - 1), nr_rcp(xn - x0));
      if (j == 0) Hd[c] = CurveHdr<T>{x0, xn, sc, T(0)};
      if (MODE == MODE_TABLE) {
        uint16_t *Tc = Tb + c * (nb + 2);
        if (j == 0) Tc[0] = 0;
        const int blo = bucket_of(xj, x0, sc, nb);
        const int bhi = (j == n - 2) ? nb + 1 : bucket_of(X[e + 1], x0, sc, nb);
        for (int b = blo + 1; b <= bhi; ++b) Tc[b] = (uint16_t)j;
      }
    }
  }
  if (MODE == MODE_BISECT) {  // Eytzinger keys x_1 .. x_{n-2}, +inf padded
    const int te = nc * P;
    for (int e = tid; e < te; e += nt) {
      const int c = e >> L2;
      const int i = e & (P - 1);
      if (i == 0) continue;
      const int r = eytz_rank(i, L2) + 1;  // knot index
      Xs[e] = (r <= n - 2) ? X[c * n + r] : (T)INFINITY;
    }
  }
}

// Locate + evaluate the cnt queries of one staged item (first query k0 of HBM; first curve
// c0; the queries staged at Qs when BULK, else read from q).  Warp w of nw owns a contiguous
// run of V-query groups; lane l takes groups wb+l, wb+l+32, ...  Returns "some query was
// out of range".
template <typename T, int MODE, int V, bool BULK, int L2, int NW>
__device__ __forceinline__ bool eval_item_queries(const T *Qs, const T *__restrict__ q, int64_t k0, int64_t c0,
                                                  int m, int cnt, int cpb, FastDiv divm, const Cub<T> *RP,
                                                  const T *RE, const T *XK,
                                                  const CurveHdr<T> *Hd, const T *Xs, const uint16_t *Tb,
                                                  const T *X, const T *Y, const T *Z, int n, int nb, int P,
                                                  T *__restrict__ out, int32_t *__restrict__ idx, int w, int nw,
                                                  int lane) {
  constexpr bool PACKED = (MODE != MODE_BSEARCH);
  bool oor = false;
  const int ng = cnt / V;
  const int per = (ng + NW - 1) / NW;  // NW (= nw) a compile-time warp count: a shift
  const int wb = w * per, we = min(ng, wb + per);
  const int kbase = (int)(k0 - c0 * m);  // item's first query, relative to its first curve
  T *const ob = out + k0;
  int32_t *const ib = idx ? idx + k0 : nullptr;
  const T *const qb = q + k0;
  for (int g = wb + lane; g < we; g += 32) {
    T qv[V], val[V];
    int jj[V];
    if (BULK) {
      VecIO<T, V>::load_shared(Qs + g * V, qv);
    } else {
      VecIO<T, V>::load(qb + g * V, qv);
    }
    const int cl = (cpb > 1) ? (int)divm.div((uint32_t)(kbase + g * V)) : 0;
    if (PACKED) {
      const CurveHdr<T> hd = Hd[cl];
      const Cub<T> *Pc = RP + cl * n;
      const T *Ec2 = RE + cl * n;
      const T *Xc = XK + cl * n;
      const uint32_t ebase = smem_u32(Xs + (size_t)cl * P);
      const uint16_t *Tc = Tb + cl * (nb + 2);
#pragma unroll
      for (int i = 0; i < V; ++i) eval_packed<T, MODE, L2>(Pc, Ec2, Xc, ebase, Tc, hd, n, nb, qv[i], val[i], jj[i]);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) eval_one<T>(X + cl * n, Y + cl * n, Z + cl * n, n, qv[i], val[i], jj[i]);
    }
#pragma unroll
    for (int i = 0; i < V; ++i) oor |= (jj[i] < 0);
    VecIO<T, V>::store(ob + g * V, val);
    if (ib) VecIO<T, V>::store_idx(ib + g * V, jj);
  }
  return oor;
}

// Persistent, double-buffered staged eval (unsorted queries).  Work item `it` = curves
// [it*cpb, +cpb) with all their queries (cpb > 1), or queries [ch*qchunk, +qchunk) of curve
// it/nchunks (cpb == 1); an item's queries are contiguous in HBM.  Grid = min(items,
// SMs x CTAs/SM); CTA b takes items b, b+G, ...
//   BULK (aligned inputs, V = 16/sizeof(T)): stage s receives item i's x, y, y2 AND its
//     queries through cp.async.bulk (mbarrier s); item i+1 is already in flight in stage s^1
//     while item i is evaluated; stage s is refilled (item i+2) once item i is done.  Every
//     input byte arrives asynchronously; outputs leave as 16-byte streaming stores.
//   !BULK (unaligned or ragged m): coalesced synchronous staging, queries from registers.
// A packing pass then builds {x, y, y2, 1/h} records (+ the mode's search structure).  Each
// warp owns a contiguous run of the item's queries; lane l takes groups of V consecutive
// queries (one curve per group: m % V == 0 when V > 1).
template <typename T, int MODE, int V, bool BULK, int L2>
__global__ void __launch_bounds__(kEvalThreads, 3)
    k_eval_staged(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, const T *__restrict__ y2, int n, int64_t batch,
                  const T *__restrict__ q, int m, T *__restrict__ out, int32_t *__restrict__ idx, int cpb,
                  int nchunks, int qchunk, int qmax, int64_t nitems, FastDiv divn, FastDiv divm) {
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch)
  constexpr bool PACKED = (MODE != MODE_BSEARCH);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const StageLayout<T> L(cpb, n, MODE, BULK ? qmax : 0);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);  // bar[0], bar[1]
  Cub<T> *KP = reinterpret_cast<Cub<T> *>(smem_raw + L.knots);
  T *KE = reinterpret_cast<T *>(smem_raw + L.e2);
  T *XK = reinterpret_cast<T *>(smem_raw + L.xk);
  CurveHdr<T> *Hd = reinterpret_cast<CurveHdr<T> *>(smem_raw + L.hdr);
  T *Xs = reinterpret_cast<T *>(smem_raw + L.xs);
  uint16_t *Tb = reinterpret_cast<uint16_t *>(smem_raw + L.table);
  const int P = L.P;
  const int nb = kBucketsPerKnot * n;
  const int64_t G = gridDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t cn = (size_t)cpb * n;

  auto stage = [&](int s) { return smem_raw + L.raw0 + (size_t)s * L.rawstep; };
  auto item_of = [&](int64_t it, int64_t &c0, int64_t &k0, int &nc, int &cnt) {
    if (cpb > 1) {
      c0 = it * cpb;
      nc = (int)min64(cpb, batch - c0);
      k0 = c0 * m;
      cnt = nc * m;
    } else {
      c0 = it / nchunks;
      const int ch = (int)(it - c0 * nchunks);
      nc = 1;
      k0 = c0 * m + (int64_t)ch * qchunk;
      cnt = (int)(min64(c0 * m + m, k0 + qchunk) - k0);
    }
  };
  auto issue = [&](int64_t it, int s) {  // thread 0 only
    if (!BULK || it >= nitems) return;
    int64_t c0, k0;
    int nc, cnt;
    item_of(it, c0, k0, nc, cnt);
    const uint32_t bytes = (uint32_t)((size_t)nc * n * sizeof(T));
    const uint32_t qbytes = (uint32_t)((size_t)cnt * sizeof(T));
    T *R = reinterpret_cast<T *>(stage(s));
    mbar_expect_tx(bar + s, 3 * bytes + qbytes);
    bulk_g2s(R, x + c0 * n, bytes, bar + s);
    bulk_g2s(R + cn, y + c0 * n, bytes, bar + s);
    bulk_g2s(R + 2 * cn, y2 + c0 * n, bytes, bar + s);
    bulk_g2s(stage(s) + L.qoff, q + k0, qbytes, bar + s);
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
  bool oor = false;
  uint32_t phases = 0u;  // bit s = parity to wait for on bar[s]
  int s = 0;

  for (; it < nitems; it += G) {
    int64_t c0, k0;
    int nc, cnt;
    item_of(it, c0, k0, nc, cnt);
    T *X = reinterpret_cast<T *>(stage(s));
    const T *Qs = reinterpret_cast<const T *>(stage(s) + L.qoff);
    if (BULK) {
      mbar_wait(bar + s, (phases >> s) & 1u);
      phases ^= 1u << s;
    } else {  // unaligned inputs: synchronous coalesced staging
      for (int e = threadIdx.x; e < nc * n; e += blockDim.x) {
        X[e] = x[c0 * n + e];
        X[cn + e] = y[c0 * n + e];
        X[2 * cn + e] = y2[c0 * n + e];
      }
      __syncthreads();
    }
    const T *Y = X + cn, *Z = X + 2 * cn;
    if (PACKED) {
      pack_item<T, MODE, L2>(X, Y, Z, n, nc, n, nb, divn, KP, KE, XK, Hd, Xs, Tb, P, threadIdx.x, blockDim.x);
      __syncthreads();  // packed data built
    }
    oor |= eval_item_queries<T, MODE, V, BULK, L2, kEvalThreads / 32>(Qs, q, k0, c0, m, cnt, cpb, divm, KP, KE, XK, Hd,
                                                                      Xs, Tb, X, Y, Z, n,
                                                   nb, P, out, idx, w, nw, lane);
    __syncthreads();  // everyone is done with this item's stage and packed data
    if (threadIdx.x == 0) issue(it + 2 * G, s);
    s ^= 1;
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(status, kOutOfRange);
}

// Persistent staged eval with per-warp curve ownership (cpb a multiple of the warp count, 16-
// byte aligned inputs): warp w of the CTA owns curves [w cpw, (w+1) cpw) of every item
// (cpw = cpb / 8), packs them and evaluates their queries, so there is no CTA-wide barrier in
// the loop.  Each warp waits on the stage's TMA mbarrier itself; the last warp to finish an
// item (a shared counter) issues the refill of that stage (item + 2), so warps drift freely
// by up to one item and the pack of one warp overlaps the evaluation of another.
template <typename T, int MODE, int L2>
__global__ void __launch_bounds__(kEvalThreads, 3)
    k_eval_warps(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, const T *__restrict__ y2, int n, int64_t batch,
                 const T *__restrict__ q, int m, T *__restrict__ out, int32_t *__restrict__ idx, int cpb,
                 int64_t nitems, FastDiv divn, FastDiv divm) {
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch)
  constexpr int V = 16 / sizeof(T);
  constexpr int NW = kEvalThreads / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const StageLayout<T> L(cpb, n, MODE, cpb * m);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);  // bar[0], bar[1]
  int *cnt = reinterpret_cast<int *>(smem_raw + 16);       // cnt[0], cnt[1]
  Cub<T> *KP = reinterpret_cast<Cub<T> *>(smem_raw + L.knots);
  T *KE = reinterpret_cast<T *>(smem_raw + L.e2);
  T *XK = reinterpret_cast<T *>(smem_raw + L.xk);
  CurveHdr<T> *Hd = reinterpret_cast<CurveHdr<T> *>(smem_raw + L.hdr);
  T *Xs = reinterpret_cast<T *>(smem_raw + L.xs);
  uint16_t *Tb = reinterpret_cast<uint16_t *>(smem_raw + L.table);
  const int P = L.P;
  const int nb = kBucketsPerKnot * n;
  const int64_t G = gridDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t cn = (size_t)cpb * n;
  const int cpw = cpb / NW;

  auto stage = [&](int s) { return smem_raw + L.raw0 + (size_t)s * L.rawstep; };
  auto issue = [&](int64_t it, int s) {  // one thread
    if (it >= nitems) return;
    const int64_t c0 = it * cpb;
    const int nc = (int)min64(cpb, batch - c0);
    const uint32_t bytes = (uint32_t)((size_t)nc * n * sizeof(T));
    const uint32_t qbytes = (uint32_t)((size_t)nc * m * sizeof(T));
    T *R = reinterpret_cast<T *>(stage(s));
    mbar_expect_tx(bar + s, 3 * bytes + qbytes);
    bulk_g2s(R, x + c0 * n, bytes, bar + s);
    bulk_g2s(R + cn, y + c0 * n, bytes, bar + s);
    bulk_g2s(R + 2 * cn, y2 + c0 * n, bytes, bar + s);
    bulk_g2s(stage(s) + L.qoff, q + c0 * m, qbytes, bar + s);
  };

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    cnt[0] = cnt[1] = 0;
  }
  __syncthreads();
  const int64_t first = blockIdx.x;
  const int nmine = first < nitems ? (int)((nitems - 1 - first) / G + 1) : 0;
  if (threadIdx.x == 0) {
    issue(first, 0);
    issue(first + G, 1);
  }
  bool oor = false;
  for (int k = 0; k < nmine; ++k) {
    const int s = k & 1;
    const int64_t it = first + (int64_t)k * G;
    const int64_t c0 = it * cpb;
    const int nc = (int)min64(cpb, batch - c0);
    mbar_wait(bar + s, (uint32_t)(k >> 1) & 1u);
    const int cw0 = w * cpw, nmy = min(cpw, nc - cw0);
    if (nmy > 0) {
      const T *X = reinterpret_cast<const T *>(stage(s)) + (size_t)cw0 * n;
      const T *Y = X + cn, *Z = X + 2 * cn;
      const T *Qs = reinterpret_cast<const T *>(stage(s) + L.qoff) + (size_t)cw0 * m;
      pack_item<T, MODE, L2>(X, Y, Z, n, nmy, n, nb, divn, KP + cw0 * n, KE + cw0 * n, XK + cw0 * n, Hd + cw0,
                             Xs + cw0 * P,
                             Tb + cw0 * (nb + 2), P, lane, 32);
      __syncwarp();
      oor |= eval_item_queries<T, MODE, V, true, L2, 1>(Qs, q, (c0 + cw0) * m, c0 + cw0, m, nmy * m, cpb, divm,
                                                     KP + cw0 * n, KE + cw0 * n, XK + cw0 * n, Hd + cw0,
                                                     Xs + cw0 * P,
                                                     Tb + cw0 * (nb + 2), X, Y, Z, n, nb, P, out, idx, 0, 1, lane);
    }
    __syncwarp();
    if (lane == 0 && last_warp_arrival(cnt + s, NW)) {
      fence_proxy_async();
      issue(it + 2 * G, s);
    }
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(status, kOutOfRange);
}

// ---- one warp per curve, no staging pass (n <= 64, unsorted queries: BASELINE cfg2) -----
// Each warp walks its own sequence of curves.  Per curve: lane l loads knots l and l+32 of x,
// y, y2 straight from HBM (coalesced; the next curve's are already in flight), builds the
// records of intervals l and l+32 into the warp's table, then the Eytzinger keys (the slot ->
// knot rank of a lane's slots is the same for every curve: computed once), and evaluates the
// curve's m queries as 16-byte vectors (lane l: vectors l, l+32, ...), with the same
// eval_packed descent and make_cub / cub_eval arithmetic as the staged kernels.  No TMA ring,
// no block barrier, no per-element division.
#ifndef FS_CW_UNROLL
#define FS_CW_UNROLL 2  // A/B cfg2: fused step 75.8 -> 73.8 us (curvewarp alone unchanged, 63.5 us)
#endif
constexpr int kCwMaxN = 64, kCwWarps = 8;
constexpr int kCwUnroll = FS_CW_UNROLL;  // query vectors of a lane interleaved (A/B)
template <typename T> struct CwTable {
  Cub<T> c[kCwMaxN];
  T e2[kCwMaxN];
  T xk[kCwMaxN];
  T ey[kCwMaxN];  // Eytzinger keys, slot 0 unused
};

// The Eytzinger slot of knot j (1 <= j < 2^L2): the node of in-order rank j-1 (the inverse of
// eytz_rank), so each lane's keys go to the table straight from registers.
template <int L2> __device__ __forceinline__ int cw_slot(int j) {
  const int sft = __ffs(j) - 1, d = L2 - 1 - sft;
  return (1 << d) + (((j >> sft) - 1) >> 1);
}

// One curve's table from its knots in registers (lane l holds knots l, l+32: kx, ky, kz): the
// records of intervals l, l+32 (x_{j+1}, y_{j+1}, y2_{j+1} from the neighbour lane) and the
// Eytzinger keys x_1 .. x_{n-2}, +inf padded (slots s0, s1 of cw_slot).  The caller syncs the warp.
template <typename T, int L2>
__device__ __forceinline__ void cw_build_table(CwTable<T> &tb, int s0, int s1, const T (&kx)[2], const T (&ky)[2],
                                               const T (&kz)[2], int n, int lane) {
  constexpr int P = 1 << L2;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 32 * h;
    const T xn1 = __shfl_down_sync(0xffffffffu, kx[h], 1), yn1 = __shfl_down_sync(0xffffffffu, ky[h], 1),
            zn1 = __shfl_down_sync(0xffffffffu, kz[h], 1);
    // lane 31's neighbour is lane 0 of the next half
    const T xh = __shfl_sync(0xffffffffu, kx[1], 0), yh = __shfl_sync(0xffffffffu, ky[1], 0),
            zh = __shfl_sync(0xffffffffu, kz[1], 0);
    const T xb = (lane == 31) ? xh : xn1, yb = (lane == 31) ? yh : yn1, zb = (lane == 31) ? zh : zn1;
    if (j < n) tb.xk[j] = kx[h];
    if (j < n - 1) tb.c[j] = make_cub<T>(kx[h], xb, ky[h], yb, kz[h], zb, tb.e2[j]);
  }
  if (lane > 0 && lane < P) tb.ey[s0] = (lane <= n - 2) ? kx[0] : (T)INFINITY;
  if (lane + 32 < P) tb.ey[s1] = (lane + 32 <= n - 2) ? kx[1] : (T)INFINITY;
}

// The curve's queries (nv 16-byte vectors at qc; the lane's first two already in qpf): lane l
// takes vectors l, l+32, ...  Returns "some query was out of range".
template <typename T, int L2>
__device__ __forceinline__ bool cw_eval_queries(const CwTable<T> &tb, uint32_t ebase, int n, const T *__restrict__ qc,
                                                int nv, T *__restrict__ oc, int32_t *__restrict__ ic,
                                                const typename Vec16<T>::V (&qpf)[2], int lane) {
  constexpr int VW = 16 / sizeof(T);
  using VT = typename Vec16<T>::V;
  const CurveHdr<T> hd{tb.xk[0], tb.xk[n - 1], T(0), T(0)};
  bool oor = false;
#pragma unroll kCwUnroll
  for (int v = lane, i = 0; v < nv; v += 32, ++i) {
    const VT a = (i == 0) ? qpf[0] : (i == 1) ? qpf[1] : __ldcs(reinterpret_cast<const VT *>(qc) + v);
    const T *qa = reinterpret_cast<const T *>(&a);
    T val[VW];
    int jj[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      eval_packed<T, MODE_BISECT, L2>(tb.c, tb.e2, tb.xk, ebase, nullptr, hd, n, 0, qa[e], val[e], jj[e]);
      oor |= jj[e] < 0;
    }
    VecIO<T, VW>::store(oc + (size_t)v * VW, val);
    if (ic) VecIO<T, VW>::store_idx(ic + (size_t)v * VW, jj);
  }
  return oor;
}

template <typename T, int L2>
__global__ void __launch_bounds__(kCwWarps * 32, 4) k_eval_curvewarp(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y,
                                                                     const T *__restrict__ y2, int n, int64_t batch,
                                                                     const T *__restrict__ q, int m,
                                                                     T *__restrict__ out, int32_t *__restrict__ idx) {
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch)
  constexpr int P = 1 << L2;  // <= 64
  using VT = typename Vec16<T>::V;
  constexpr int VW = 16 / sizeof(T);
  __shared__ CwTable<T> tabs[kCwWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  CwTable<T> &tb = tabs[w];
  const uint32_t ebase = smem_u32(tb.ey);
  const int s0 = (lane > 0 && lane < P) ? cw_slot<L2>(lane) : 0;
  const int s1 = (lane + 32 < P) ? cw_slot<L2>(lane + 32) : 0;
  const int nv = m / VW;  // query vectors per curve
  const int64_t G = (int64_t)gridDim.x * kCwWarps;
  int64_t c = (int64_t)blockIdx.x * kCwWarps + w;
  bool oor = false;
  // the current curve's knots (lane's two) in registers
  T kx[2], ky[2], kz[2];
  auto load_knots = [&](int64_t cc) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      if (cc < batch && j < n) {
        kx[h] = __ldcs(x + cc * n + j);
        ky[h] = __ldcs(y + cc * n + j);
        kz[h] = __ldcs(y2 + cc * n + j);
      }
    }
  };
  load_knots(c);
  for (; c < batch; c += G) {
    const T *qc = q + c * m;
    // the lane's first two query vectors of this curve: in flight during the table build
    VT qpf[2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
      if (lane + 32 * i < nv) qpf[i] = __ldcs(reinterpret_cast<const VT *>(qc) + lane + 32 * i);
    cw_build_table<T, L2>(tb, s0, s1, kx, ky, kz, n, lane);
    load_knots(c + G);  // the next curve's knots, in flight during this curve's queries
    __syncwarp();
    oor |= cw_eval_queries<T, L2>(tb, ebase, n, qc, nv, out + c * m, idx ? idx + c * m : nullptr, qpf, lane);
    __syncwarp();  // the table is rebuilt for the next curve
  }
  raise_status_warp(status, oor, kOutOfRange);
}

// ---- tiny problems (a few K1h-sized curves: BASELINE cfg1) -------------------------------
// One CTA per curve does the whole call: warp 0's lanes 0/1 run K1h's two-ended register sweep
// (k1h_solve: bitwise K1h's y2), the CTA builds the interval records and Eytzinger keys, and
// every thread evaluates its queries with eval_packed -- one launch, no TMA pipeline, no
// warp-specialised hand-off.  The queries' first vectors load at kernel entry.
template <typename T, int N, int L2>
__global__ void __launch_bounds__(256) k_build_eval_tiny(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y,
                                                         int64_t batch, int bc, const T *__restrict__ yp1,
                                                         const T *__restrict__ ypn, T *__restrict__ y2,
                                                         const T *__restrict__ q, int m, T *__restrict__ out,
                                                         int32_t *__restrict__ idx) {
  constexpr int VW = 16 / sizeof(T);
  constexpr int P = 1 << L2;
  using VT = typename Vec16<T>::V;
  __shared__ CwTable<T> tb;
  __shared__ __align__(16) T zs[N];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t c = blockIdx.x;
  const T *qc = q + c * m;
  const int nv = m / VW;
  VT q0;
  if (tid < nv) q0 = __ldcs(reinterpret_cast<const VT *>(qc) + tid);
  // y2 to HBM (when asked) and to shared memory, which the table build reads
  if (tid < 32) k1h_solve<T, N>(status, x, y, batch, bc, yp1, ypn, y2, (lane < 2) ? c : batch, (lane & 1) == 0, zs);
  __syncthreads();  // y2 of the curve is in shared memory
  const T *X = x + c * N, *Y = y + c * N, *Z = zs;
  if (tid < N) tb.xk[tid] = X[tid];
  if (tid < N - 1) tb.c[tid] = make_cub<T>(X[tid], X[tid + 1], Y[tid], Y[tid + 1], Z[tid], Z[tid + 1], tb.e2[tid]);
  if (tid > 0 && tid < P) {
    const int r = eytz_rank(tid, L2) + 1;
    tb.ey[tid] = (r <= N - 2) ? X[r] : (T)INFINITY;
  }
  __syncthreads();
  const CurveHdr<T> hd{tb.xk[0], tb.xk[N - 1], T(0), T(0)};
  const uint32_t ebase = smem_u32(tb.ey);
  bool oor = false;
  for (int v = tid; v < nv; v += 256) {
    const VT a = (v == tid) ? q0 : __ldcs(reinterpret_cast<const VT *>(qc) + v);
    const T *qa = reinterpret_cast<const T *>(&a);
    T val[VW];
    int jj[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
      eval_packed<T, MODE_BISECT, L2>(tb.c, tb.e2, tb.xk, ebase, nullptr, hd, N, 0, qa[e], val[e], jj[e]);
      oor |= jj[e] < 0;
    }
    VecIO<T, VW>::store(out + c * m + (size_t)v * VW, val);
    if (idx) VecIO<T, VW>::store_idx(idx + c * m + (size_t)v * VW, jj);
  }
  raise_status_warp(status, oor, kOutOfRange);
}

// ---- many K1h-sized curves, unsorted queries: build + evaluate per warp (BASELINE cfg2) ------
// spline_build_eval's fused path for n in {16, 32, 64}.  Each warp owns
// a contiguous range of curves and walks it in groups of 16: the group is solved by K1h's
// two-ended register sweep (k1h_solve, lane pair 2t/2t+1 on curve t: bitwise K1h's y2), which
// leaves the y2 rows in the warp's shared-memory stage (and in HBM when the caller asked for y2);
// then each curve of the group goes through k_eval_curvewarp's body (cw_build_table,
// cw_eval_queries) with x, y re-read from L1/L2 (the solve just loaded them) and y2 from the
// stage.  Against K1h + k_eval_curvewarp, HBM sees y2 written at most once and never read back,
// and there is one launch.  The next group's x, y are prefetched to L2 during this group's queries.
constexpr int kBwWarps = 8, kBwGroup = 16;
template <typename T, int N> __host__ __device__ constexpr int bw_stride() { return N + 16 / (int)sizeof(T); }
template <typename T, int N> struct BwStage {
  CwTable<T> tb;
  alignas(16) T z[kBwGroup * bw_stride<T, N>()];  // y2 rows of the group, padded: lane pairs hit distinct banks
};
#ifndef FS_BW_MINB
#define FS_BW_MINB 2  // A/B on cfg2 (us, y2 written): 2 -> 74.2, 3 -> 79.9 (spills), 4 -> 88.1; split path 74.8
#endif
template <typename T, int N, int L2>
__global__ void __launch_bounds__(kBwWarps * 32, FS_BW_MINB)
    k_build_eval_warp(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int64_t batch,
                      int bc, const T *__restrict__ yp1, const T *__restrict__ ypn, T *__restrict__ y2,
                      const T *__restrict__ q, int m, T *__restrict__ out, int32_t *__restrict__ idx) {
  constexpr int P = 1 << L2, S = bw_stride<T, N>();
  constexpr int VW = 16 / sizeof(T);
  using VT = typename Vec16<T>::V;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  BwStage<T, N> &st = reinterpret_cast<BwStage<T, N> *>(smem_raw)[w];
  const uint32_t ebase = smem_u32(st.tb.ey);
  const int s0 = (lane > 0 && lane < P) ? cw_slot<L2>(lane) : 0;
  const int s1 = (lane + 32 < P) ? cw_slot<L2>(lane + 32) : 0;
  const int nv = m / VW;
  const int64_t GW = (int64_t)gridDim.x * kBwWarps, gw = (int64_t)blockIdx.x * kBwWarps + w;
  const int64_t cb = batch * gw / GW, ce = batch * (gw + 1) / GW;  // this warp's curves
  const int t = lane >> 1;
  const bool top = (lane & 1) == 0;
  bool oor = false;
  for (int64_t g0 = cb; g0 < ce; g0 += kBwGroup) {
    const int ng = (int)min64(kBwGroup, ce - g0);
    if (g0 + kBwGroup < ce) {  // the next group's x, y rows to L2 (one 128-byte line per lane)
      const int64_t nb = min64(kBwGroup, ce - g0 - kBwGroup) * N * (int64_t)sizeof(T);
      const char *px = reinterpret_cast<const char *>(x + (g0 + kBwGroup) * N);
      const char *py = reinterpret_cast<const char *>(y + (g0 + kBwGroup) * N);
      for (int64_t o = (int64_t)lane * 128; o < nb; o += 32 * 128) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(px + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(py + o));
      }
    }
    k1h_solve<T, N>(status, x, y, batch, bc, yp1, ypn, y2, t < ng ? g0 + t : batch, top, st.z + t * S);
    __syncwarp();
    T kx[2], ky[2], kz[2];
    auto load_knots = [&](int k) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j < N) {
          kx[h] = __ldg(x + (g0 + k) * N + j);
          ky[h] = __ldg(y + (g0 + k) * N + j);
          kz[h] = st.z[k * S + j];
        }
      }
    };
    load_knots(0);
    for (int k = 0; k < ng; ++k) {
      const int64_t c = g0 + k;
      const T *qc = q + c * m;
      VT qpf[2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
        if (lane + 32 * i < nv) qpf[i] = __ldcs(reinterpret_cast<const VT *>(qc) + lane + 32 * i);
      cw_build_table<T, L2>(st.tb, s0, s1, kx, ky, kz, N, lane);
      if (k + 1 < ng) load_knots(k + 1);
      __syncwarp();
      oor |= cw_eval_queries<T, L2>(st.tb, ebase, N, qc, nv, out + c * m, idx ? idx + c * m : nullptr, qpf, lane);
      __syncwarp();
    }
  }
  raise_status_warp(status, oor, kOutOfRange);
}

// ---- very short curves, few queries (fp32, n <= 8, m <= 32: BASELINE cfg3) -----------------
// One warp per tile of 32 curves, no block-level synchronisation and no staging pass: lane l
// builds the records of curve c0+l in registers straight from HBM (16-byte loads) into its
// own slot of the warp's shared-memory table; the tile's m*32 queries (contiguous in HBM) are
// then loaded as 16-byte vectors, lane l holding vectors l, l+32, ... (one curve each,
// m % 4 == 0), all in flight at once.  A query is located by branch-free
// binary lifting over its curve's n-1 left knots (3 steps for n <= 8; exact on any grid, so
// the uniform-grid hint needs no separate path) and evaluated with the same make_cub /
// cub_eval arithmetic as every other kernel.  Per query: ~35 instructions, no pack loop, no
// division to find the curve.
constexpr int kSmallN = 8, kSmallM = 32, kSmallWarps = 4;
struct alignas(16) SmallCurve {  // 208 B: 52 words, so the 4 curves of a warp access hit distinct banks
  Cub<float> c[kSmallN - 1];
  float e2[kSmallN - 1];
  float xk[kSmallN];
  float x0, xn;
  float pad[7];
};

// SOLVE (k_fused_small path of spline_build_eval): lane l also solves its curve -- K1r's
// thomas_regs on the same registers, so y2 is bitwise K1r's -- stores y2 (when y2w is
// non-null) and builds the records from registers: x, y are read once and y2 is never read back.
template <bool SOLVE>
__global__ void __launch_bounds__(kSmallWarps * 32, SOLVE ? 4 : 6) k_eval_small(unsigned *__restrict__ status, const float *__restrict__ x,
                                                                 const float *__restrict__ y,
                                                                 const float *__restrict__ y2, int n, int64_t batch,
                                                                 const float *__restrict__ q, int m,
                                                                 float *__restrict__ out, int32_t *__restrict__ idx,
                                                                 int vecn, int bc = 0,
                                                                 const float *__restrict__ yp1 = nullptr,
                                                                 const float *__restrict__ ypn = nullptr,
                                                                 float *__restrict__ y2w = nullptr,
                                                                 int64_t xs = -1) {
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch; SOLVE too: its
              // launch carries the attribute, and its outputs must not race the predecessor)
  constexpr int MV = kSmallM;  // at most m vectors per lane (32 curves x m queries / (32 lanes x 4))
  __shared__ SmallCurve tab[kSmallWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SmallCurve *T = tab[w];
  const int64_t ntiles = (batch + 31) >> 5;
  bool oor = false;
  for (int64_t tile = (int64_t)blockIdx.x * kSmallWarps + w; tile < ntiles; tile += (int64_t)gridDim.x * kSmallWarps) {
    const int64_t c0 = tile << 5;
    const int nc = (int)min64(32, batch - c0);
    const int nq = nc * m;          // the tile's queries, contiguous from q + c0 m
    const int nv = nq >> 2;         // 16-byte vectors
    const float *qt = q + c0 * m;
    // records of curve c0 + lane (xs: the knot row stride -- n, or 0 when the batch shares x)
    if (lane < nc) {
      const int64_t c = c0 + lane;
      const float *xr = x + c * (xs < 0 ? (int64_t)n : xs);
      float xv[kSmallN], yv[kSmallN], zv[kSmallN];
      if (vecn) {  // n == 8 with 16-byte aligned rows
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float4 a = __ldg(reinterpret_cast<const float4 *>(xr) + h);
          const float4 b = __ldg(reinterpret_cast<const float4 *>(y + c * 8) + h);
          xv[4 * h] = a.x; xv[4 * h + 1] = a.y; xv[4 * h + 2] = a.z; xv[4 * h + 3] = a.w;
          yv[4 * h] = b.x; yv[4 * h + 1] = b.y; yv[4 * h + 2] = b.z; yv[4 * h + 3] = b.w;
          if constexpr (!SOLVE) {
            const float4 d = __ldg(reinterpret_cast<const float4 *>(y2 + c * 8) + h);
            zv[4 * h] = d.x; zv[4 * h + 1] = d.y; zv[4 * h + 2] = d.z; zv[4 * h + 3] = d.w;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < kSmallN; ++j) {
          const int jj = min(j, n - 1);
          xv[j] = __ldg(xr + jj);
          yv[j] = __ldg(y + c * n + jj);
          if constexpr (!SOLVE) zv[j] = __ldg(y2 + c * n + jj);
        }
      }
      if constexpr (SOLVE) {  // K1r's sweep (build_thomas.cuh thomas_regs), then y2 out
        const bool ok = thomas_regs<float, kSmallN>(xv, yv, n, bc, (bc & 1) ? yp1[c] : 0.f, (bc & 2) ? ypn[c] : 0.f, zv);
        if (!ok) raise_status(status, kBadKnots);
        if (y2w) {
          if (vecn) {
            reinterpret_cast<float4 *>(y2w + c * 8)[0] = make_float4(zv[0], zv[1], zv[2], zv[3]);
            reinterpret_cast<float4 *>(y2w + c * 8)[1] = make_float4(zv[4], zv[5], zv[6], zv[7]);
          } else {
#pragma unroll
            for (int j = 0; j < kSmallN; ++j)
              if (j < n) y2w[c * n + j] = zv[j];
          }
        }
      }
      SmallCurve &S = T[lane];
#pragma unroll
      for (int j = 0; j < kSmallN - 1; ++j) {
        if (j < n - 1) {
          float e2;
          S.c[j] = make_cub<float>(xv[j], xv[j + 1], yv[j], yv[j + 1], zv[j], zv[j + 1], e2);
          S.e2[j] = e2;
        }
      }
#pragma unroll
      for (int j = 0; j < kSmallN; ++j) S.xk[j] = xv[j];  // (entries past n-1 repeat x_{n-1})
      S.x0 = xv[0];
      S.xn = xv[kSmallN - 1];  // = x_{n-1} (clamped index above)
    }
    float4 qv[MV / 4];  // (loaded after the record build: registers)
#pragma unroll
    for (int i = 0; i < MV / 4; ++i) {
      const int v = lane + 32 * i;
      if (v < nv) qv[i] = __ldcs(reinterpret_cast<const float4 *>(qt) + v);
    }
    __syncwarp();
    // evaluate: vector v = lane + 32 i holds queries 4v .. 4v+3 of curve (4v) / m
    const int top = n - 2;
#pragma unroll
    for (int i = 0; i < MV / 4; ++i) {
      const int v = lane + 32 * i;
      if (v < nv) {
        const int cl = (4 * v) / m;
        const SmallCurve &S = T[cl];
        const float x0 = S.x0, xn = S.xn;
        const float qq[4] = {qv[i].x, qv[i].y, qv[i].z, qv[i].w};
        float r[4];
        int jj[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = (qq[e] >= x0) && (qq[e] <= xn);
          const float qc = in ? qq[e] : x0;
          int j = 0;
#pragma unroll
          for (int d = kSmallN / 2; d >= 1; d >>= 1) {  // largest j <= n-2 with x_j <= q
            const int p = min(j + d, top);
            j = (S.xk[p] <= qc) ? p : j;
          }
          const float val = cub_eval<float>(S.c[j], S.e2[j], S.xk[j], qc);
          r[e] = in ? val : qnan<float>();
          jj[e] = in ? j : -1;
          oor |= !in;
        }
        __stcs(reinterpret_cast<float4 *>(out + c0 * m) + v, make_float4(r[0], r[1], r[2], r[3]));
        if (idx) __stcs(reinterpret_cast<int4 *>(idx + c0 * m) + v, make_int4(jj[0], jj[1], jj[2], jj[3]));
      }
    }
    __syncwarp();  // the table is rebuilt for the next tile
  }
  raise_status_warp(status, oor, kOutOfRange);
}

// ---- sorted query runs ------------------------------------------------------------------

// Warp-cooperative 32-ary search (all lanes hold the same q, X[0] <= q <= X[n-1]):
// 32 probes per round, a ballot keeps the last probe with X[p] <= q.  ~log_33(n) rounds of
// one parallel load each (3 rounds for n = 4096) instead of log2(n) dependent loads.
template <typename T> __device__ __forceinline__ int warp_locate(const T *X, int n, T q, int lane) {
  int lo = 0, hi = n - 1;  // invariant: X[lo] <= q, and hi == n-1 or X[hi] > q
  while (hi - lo > 1) {
    const int span = hi - lo;
    const int p = lo + (int)(((int64_t)span * (lane + 1)) / 33);
    const bool le = (p > lo) && (__ldg(X + p) <= q);
    const unsigned ball = __ballot_sync(0xffffffffu, le);
    const int k = ball ? 31 - __clz(ball) : -1;  // X[p] <= q is monotone in the lane index
    const int nlo = (k >= 0) ? __shfl_sync(0xffffffffu, p, k) : lo;
    const int nhi = (k < 31) ? __shfl_sync(0xffffffffu, p, k + 1) : hi;
    lo = nlo;
    hi = max(nhi, lo + 1);
  }
  return min(lo, n - 2);
}

// SPLINE_Q_SORTED: one warp per run of `qrun` consecutive queries of one curve.  Lane l
// takes groups of V consecutive queries, 32V per warp step; every lane starts from the
// warp's carried bracket jc (the largest interval found in the previous step) and moves
// forward -- generalising the paper's "while x[i+1] < q: i += 1" sweep to 32
// lanes.  FORM_RECORD (spline_eval): the warp keeps a window of kSortWin interval records
// in shared memory, built cooperatively (one make_cub per lane) at the carry and rebuilt when
// the carry passes its middle; a query in the window is located by a short verified lift
// from the carry (first query of the lane) or from the lane's previous query, so a step costs
// a few shared-memory loads per query and no per-query record build.  Queries outside the
// window, and the ablation FORMs, take the general path: a scan from the carry through L1
// (bisection below the carry -- a wrong hint --, galloping for long jumps).  The host takes
// the window (WIN) only for dense queries (at least kSortWinDensity per interval): for sparse
// ones a rebuild would serve too few queries.
// FORM (common.cuh interp_form) selects the evaluation variant: FORM_RECORD for spline_eval,
// the others for spline_eval_ablation (the paper's division variants and no-op loop).
// A warp's window of kSortWin interval records (FORM_RECORD): built cooperatively, one
// interval per lane, at the carried bracket and reused while the carry stays in its first half.
constexpr int kSortWin = 32;
#ifndef FS_SORTED_FAST
#define FS_SORTED_FAST 1  // round 1 (3-level first lift, a range pre-check): 1497 vs 1112 us on cfg4; now the default
#endif
constexpr bool kSortedFast = FS_SORTED_FAST != 0;  // the warp-uniform fast path of sorted_run (WIN)
#ifndef FS_SORTED_L1PF
#define FS_SORTED_L1PF 1
#endif
constexpr bool kSortedL1Prefetch = FS_SORTED_L1PF != 0;  // L1 prefetch of the next window's knots
#ifndef FS_SORTED_OUTLINE
#define FS_SORTED_OUTLINE 0  // A/B: 1224 vs 1100 us on cfg4 (the call and its stack cost more than the registers saved)
#endif
constexpr bool kSortedOutlineGeneral = FS_SORTED_OUTLINE != 0;  // the window miss path out of line
constexpr int kSortWinDensity = 8;  // queries per interval from which the window pays
// One window record: the interval's left knot and its cubic (Cub + e2), 16-byte aligned so that
// a lookup is 2 (fp32) or 3 (fp64) vector loads.
// fp64: 48 B -- a stride of 12 banks, so the 8 lanes of a quarter-warp phase reading 8 different
// records hit disjoint banks (a 64 B record measured 22% slower on cfg4: 4-way conflicts).
template <typename T> struct alignas(16) WRec {
  T x0, ih, y0, dy, e1, e2;  // the interval's left knot, then its cubic (Cub + e2)
};
template <typename T> __device__ __forceinline__ WRec<T> ld_wrec(const WRec<T> *p) {
  using VT = typename Vec16<T>::V;
  constexpr int NV = (int)(sizeof(WRec<T>) / 16);
  WRec<T> r;
#pragma unroll
  for (int i = 0; i < NV; ++i) reinterpret_cast<VT *>(&r)[i] = reinterpret_cast<const VT *>(p)[i];
  return r;
}
template <typename T> struct SortWin {
  WRec<T> r[kSortWin];
  T x[kSortWin + 1];  // x[i] = x_{wb+i} (+inf past x_{n-2}); x[kSortWin] = x_{wb+kSortWin} or +inf
};

// Where a sorted run reads the second derivatives from: global memory (spline_eval) or the
// shared-memory y2 a fused build just produced (k_tile_eval: padded rows, pad(j) = j + j/R).
template <typename T> struct ZGlobal {
  const T *Z;
  __device__ __forceinline__ T operator()(int j) const { return __ldg(Z + j); }
  __device__ __forceinline__ const T *prefetch_ptr() const { return Z; }
};
template <typename T, int R> struct ZShared {
  const T *Zs;
  __device__ __forceinline__ T operator()(int j) const { return Zs[j + j / R]; }
  __device__ __forceinline__ const T *prefetch_ptr() const { return nullptr; }
};

// One warp's run of queries [k0, k1) of one curve (X, Y in global memory, Z through ZA).
// Shared by k_eval_sorted and the fused long-curve kernel, so both give the same bits.
// The general path of a sorted run as an out-of-line call (rare: queries outside the window).
template <typename T> struct GQ { T v; int j; };
template <typename T, int FORM, typename ZA>
__device__ __noinline__ GQ<T> general_query_ni(const T *__restrict__ X, const T *__restrict__ Y, ZA Z, int n, T qc,
                                                int j) {
  if (__ldg(X + j) > qc) {
    j = bisect(X, n, qc);
  } else {
    int steps = 0;
    while (j < n - 2 && __ldg(X + j + 1) <= qc) {
      ++j;
      if (++steps == 8) {
        j = gallop_up(X, n, j, qc);
        break;
      }
    }
  }
  const T xa = __ldg(X + j), xb = __ldg(X + j + 1);
  return GQ<T>{interp_form<T, FORM>(qc, xa, xb, __ldg(Y + j), __ldg(Y + j + 1), Z(j), Z(j + 1)), j};
}

template <typename T, int V, int FORM, bool WIN, int PF, typename ZA>
__device__ __forceinline__ bool sorted_run(const T *__restrict__ X, const T *__restrict__ Y, const ZA &Z, int n,
                                           const T *__restrict__ qb, T *__restrict__ ob, int32_t *__restrict__ ib,
                                           int64_t k0, int64_t k1, SortWin<T> &sw, int lane) {
  const T x0 = __ldg(X), xn = __ldg(X + n - 1);
  // initial bracket from the run's first query (clamped into range)
  T qf = __ldg(qb + k0);
  qf = (qf >= x0 && qf <= xn) ? qf : x0;
  int jc = warp_locate(X, n, qf, lane);
  bool oor = false;
  int wb = -(1 << 30);            // window base: none yet

  // the queries of the next PF warp steps are in flight (a register ring, rotated each step):
  // the run is bound by the bytes in flight per warp, not by its arithmetic
  T qr[PF + 1][V];
#pragma unroll
  for (int d = 0; d < PF; ++d) {
    const int64_t kd = k0 + (int64_t)(d * 32 + lane) * V;
    if (kd < k1) VecIO<T, V>::load(qb + kd, qr[d]);
  }
  for (int64_t base = k0; base < k1; base += 32 * V) {
    const int64_t k = base + (int64_t)lane * V;
    const int64_t kn = k + (int64_t)PF * 32 * V;
    if (kn < k1) VecIO<T, V>::load(qb + kn, qr[PF]);  // PF steps ahead
    T qa[V];
#pragma unroll
    for (int i = 0; i < V; ++i) qa[i] = qr[0][i];
    if constexpr (!WIN) {
      const T *zp = Z.prefetch_ptr();
      if (lane < 2 || (lane == 2 && zp)) prefetch_l1((lane == 0 ? X : lane == 1 ? Y : zp) + min(jc + 32, n - 1));
    } else {
      if (jc < wb || jc - wb > kSortWin / 2) {  // warp-uniform: rebuild the window at the carry
        __syncwarp();
        wb = jc;
        const int jw = wb + lane;
        if (jw <= n - 2) {
          const T xa = __ldg(X + jw), xb = __ldg(X + jw + 1);
          T e2;
          const Cub<T> cb = make_cub<T>(xa, xb, __ldg(Y + jw), __ldg(Y + jw + 1), Z(jw), Z(jw + 1), e2);
          sw.r[lane] = WRec<T>{xa, cb.ih, cb.y0, cb.dy, cb.e1, e2};
          sw.x[lane] = xa;
          if (lane == kSortWin - 1) sw.x[kSortWin] = xb;
        } else {
          sw.x[lane] = inf_of<T>();
          if (lane == kSortWin - 1) sw.x[kSortWin] = inf_of<T>();
        }
        __syncwarp();
        if constexpr (kSortedL1Prefetch) {
          // the next rebuild starts in (wb + 16, wb + 32] and reads up to 32 intervals on: pull
          // those knots into L1 now (3 lines of x, y, y2 each), so its loads hit L1 instead of
          // waiting on L2 (ncu r02: the rebuild's x/y loads were 28% of the stall samples)
          if (lane < 9) {
            const int a = lane / 3, part = lane % 3;
            const T *base = a == 0 ? X : a == 1 ? Y : Z.prefetch_ptr();
            const int j = min(wb + kSortWin + part * (128 / (int)sizeof(T)), n - 1);
            if (base) prefetch_l1(base + j);
          }
        }
      }
    }
    int jl = -1;
    if constexpr (WIN && kSortedFast) {
      // warp-uniform fast path, no per-query branches: a lane's first query lifts 5 levels from
      // the carry (any slot of the window), each next one 2 levels from the previous slot (a
      // sorted run rarely passes more than 3 knots between two consecutive queries); every slot
      // is VERIFIED against the window's knots (x_{wb+l} <= q < x_{wb+l+1}), which also rejects
      // NaN, queries below the window and a run that is not sorted.  A query in a verified slot
      // is in range unless the window reaches the curve's end (wtail: then q <= x_{n-1} is
      // tested).  Any miss anywhere in the warp redoes the step on the general path below (the
      // same make_cub / cub_eval arithmetic, so the same bits).
      const int l0 = jc - wb;
      const bool wtail = !(sw.x[kSortWin] <= xn);
      T val[V];
      int jj[V];
      bool ok = true, soor = false;
      int l = l0, sjl = -1;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const T qc = qa[i];
#pragma unroll
        for (int d = (i == 0) ? kSortWin / 2 : 2; d >= 1; d >>= 1) {
          const int p = min(l + d, kSortWin - 1);
          l = (sw.x[p] <= qc) ? p : l;
        }
        const WRec<T> wr = ld_wrec(&sw.r[l]);
        const T xr = sw.x[l + 1];
        ok &= (qc >= wr.x0) & (qc < xr);
        const bool in = !wtail || qc <= xn;
        const T v = cub_eval<T>(Cub<T>{wr.ih, wr.y0, wr.dy, wr.e1}, wr.e2, wr.x0, qc);
        val[i] = in ? v : qnan<T>();
        jj[i] = in ? wb + l : -1;
        soor |= !in;
        sjl = in ? wb + l : sjl;
      }
      if (__all_sync(0xffffffffu, ok || k >= k1)) {
        if (k < k1) {
          VecIO<T, V>::store(ob + k, val);
          if (ib) VecIO<T, V>::store_idx(ib + k, jj);
          jl = sjl;
          oor |= soor;
        }
        const int jm = __reduce_max_sync(0xffffffffu, jl);
        if (jm >= 0) jc = jm;
#pragma unroll
        for (int d = 0; d < PF; ++d)
#pragma unroll
          for (int i = 0; i < V; ++i) qr[d][i] = qr[d + 1][i];
        continue;
      }
    }
    if (k < k1) {
      T val[V];
      int jj[V];
      int j = jc;
      int lp = 0;  // this lane's previous window slot (FORM_RECORD)
      // the window's bounds for this step (warp-uniform; read once, not per query)
      const int l0 = WIN ? jc - wb : 0;
      T wlo = T(0), whi = T(0);
      if constexpr (WIN) {
        wlo = sw.x[l0];
        whi = sw.x[kSortWin];
      }
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const T qq = qa[i];
        const bool in = (qq >= x0) && (qq <= xn);
        const T qc = in ? qq : x0;
        if constexpr (WIN) {
          // in the window at or after the carry: branch-free lifting over the window's knots
          // (largest l < kSortWin with x_{wb+l} <= q; +inf past x_{n-2} keeps it <= n-2-wb)
          if (qc >= wlo && qc < whi) {
            int l;
            if (i == 0) {
              // the lane's first query: a full 5-level lift from the carry (the lanes' first
              // queries spread over the whole window: a short lift would miss for the upper lanes)
              l = l0;
#pragma unroll
              for (int d = kSortWin / 2; d >= 1; d >>= 1) {
                const int p = min(l + d, kSortWin - 1);
                l = (sw.x[p] <= qc) ? p : l;
              }
            } else {
              // the next query of the lane (sorted: the same or the next interval, as a rule):
              // one step from the previous slot, verified; a longer jump lifts from there
              l = lp;
              {
                const int p = min(l + 1, kSortWin - 1);
                l = (sw.x[p] <= qc) ? p : l;
              }
              if (sw.x[l + 1] <= qc && l < kSortWin - 1) {  // clustered knots: a longer jump
#pragma unroll
                for (int d = kSortWin / 2; d >= 1; d >>= 1) {
                  const int p = min(l + d, kSortWin - 1);
                  l = (sw.x[p] <= qc) ? p : l;
                }
              }
            }
            const WRec<T> wr = ld_wrec(&sw.r[l]);
            if (qc >= wr.x0) {  // always for i = 0; for i > 0 it guards a run that is not sorted
              lp = l;
              const T v = cub_eval<T>(Cub<T>{wr.ih, wr.y0, wr.dy, wr.e1}, wr.e2, wr.x0, qc);
              j = wb + l;
              val[i] = in ? v : qnan<T>();
              jj[i] = in ? j : -1;
              oor |= !in;
              if (in) jl = j;
              continue;
            }
          }
        }  // outside the window: the general path, from this lane's previous interval
        if constexpr (WIN && kSortedOutlineGeneral) {  // out of line: the hot window path keeps its registers
          const GQ<T> g = general_query_ni<T, FORM_RECORD, ZA>(X, Y, Z, n, qc, j);
          j = g.j;
          val[i] = in ? g.v : qnan<T>();
          jj[i] = in ? j : -1;
          oor |= !in;
          if (in) jl = j;
          continue;
        }
        if (__ldg(X + j) > qc) {
          j = bisect(X, n, qc);  // below the carry: unsorted input despite the hint
        } else {
          int steps = 0;
          while (j < n - 2 && __ldg(X + j + 1) <= qc) {
            ++j;
            if (++steps == 8) {  // sparse queries: gallop the rest of the way
              j = gallop_up(X, n, j, qc);
              break;
            }
          }
        }
        const T xa = __ldg(X + j), xb = __ldg(X + j + 1);
        T v;
        if constexpr (FORM == FORM_NOOP) v = __ldg(Y + j);
        else v = interp_form<T, FORM>(qc, xa, xb, __ldg(Y + j), __ldg(Y + j + 1), Z(j), Z(j + 1));
        val[i] = in ? v : qnan<T>();
        jj[i] = in ? j : -1;
        oor |= !in;
        if (in) jl = j;
      }
      VecIO<T, V>::store(ob + k, val);
      if (ib) VecIO<T, V>::store_idx(ib + k, jj);
    }
    const int jm = __reduce_max_sync(0xffffffffu, jl);
    if (jm >= 0) jc = jm;
#pragma unroll
    for (int d = 0; d < PF; ++d)
#pragma unroll
      for (int i = 0; i < V; ++i) qr[d][i] = qr[d + 1][i];
  }
  return oor;
}

// The dense-run form (FORM_RECORD with the window): every lane takes V consecutive queries per
// warp step; its first query is located by a branch-free 5-level search over the window's knots,
// the following ones by two branch-free advance steps from the previous slot (sorted: rarely more
// than one interval apart), and every hit is VERIFIED against the record's own [x0, x1] -- a
// miss (below / beyond the window, or a wrong sorted hint) takes the general path, so idx is the
// locate rule's on any input.  The window (32 records) is rebuilt at the carry when the carry
// leaves it or the step's last query passes its end.  Bitwise the other forms' out (make_cub +
// cub_eval on the same interval).
template <typename T, int FORM, typename ZA>
__device__ __forceinline__ T general_query(const T *__restrict__ X, const T *__restrict__ Y, const ZA &Z, int n, T qc,
                                           int &j) {
  if (__ldg(X + j) > qc) {
    j = bisect(X, n, qc);  // below the carry: unsorted input despite the hint
  } else {
    int steps = 0;
    while (j < n - 2 && __ldg(X + j + 1) <= qc) {
      ++j;
      if (++steps == 8) {  // sparse queries: gallop the rest of the way
        j = gallop_up(X, n, j, qc);
        break;
      }
    }
  }
  const T xa = __ldg(X + j), xb = __ldg(X + j + 1);
  if constexpr (FORM == FORM_NOOP) return __ldg(Y + j);
  else return interp_form<T, FORM>(qc, xa, xb, __ldg(Y + j), __ldg(Y + j + 1), Z(j), Z(j + 1));
}

template <typename T, int V, int PF, typename ZA>
__device__ __forceinline__ bool sorted_run_win(const T *__restrict__ X, const T *__restrict__ Y, const ZA &Z, int n,
                                               const T *__restrict__ qb, T *__restrict__ ob, int32_t *__restrict__ ib,
                                               int64_t k0, int64_t k1, SortWin<T> &sw, int lane) {
  const T x0 = __ldg(X), xn = __ldg(X + n - 1);
  T qf = __ldg(qb + k0);
  qf = (qf >= x0 && qf <= xn) ? qf : x0;
  int jc = warp_locate(X, n, qf, lane);
  bool oor = false;
  int wb = -(1 << 30);
  T xwhi = -inf_of<T>();  // x_{wb+32} (or +inf past the curve): the window's end, in a register
  T qr[PF + 1][V];
#pragma unroll
  for (int d = 0; d <= PF; ++d)
#pragma unroll
    for (int i = 0; i < V; ++i) qr[d][i] = x0;  // lanes past the run's end keep a harmless value
#pragma unroll
  for (int d = 0; d < PF; ++d) {
    const int64_t kd = k0 + (int64_t)(d * 32 + lane) * V;
    if (kd < k1) VecIO<T, V>::load(qb + kd, qr[d]);
  }
  for (int64_t base = k0; base < k1; base += 32 * V) {
    const int64_t k = base + (int64_t)lane * V;
    const int64_t kn = k + (int64_t)PF * 32 * V;
    if (kn < k1) VecIO<T, V>::load(qb + kn, qr[PF]);  // PF steps ahead
    // warp-uniform rebuild: the carry left the window, or the step's last query passes its end
    // (the last lane's query is only a hint: a miss is caught by the verification below)
    const T ql = __shfl_sync(0xffffffffu, qr[0][V - 1], 31);
    if (jc < wb || jc >= wb + kSortWin || !(ql < xwhi)) {
      __syncwarp();
      wb = jc;
      const int jw = wb + lane;
      if (jw <= n - 2) {
        const T xa = __ldg(X + jw), xb = __ldg(X + jw + 1);
        T e2;
        const Cub<T> cb = make_cub<T>(xa, xb, __ldg(Y + jw), __ldg(Y + jw + 1), Z(jw), Z(jw + 1), e2);
        sw.r[lane] = WRec<T>{xa, cb.ih, cb.y0, cb.dy, cb.e1, e2};
        sw.x[lane] = xa;
        if (lane == kSortWin - 1) sw.x[kSortWin] = xb;
      } else {
        sw.x[lane] = inf_of<T>();
        if (lane == kSortWin - 1) sw.x[kSortWin] = inf_of<T>();
      }
      __syncwarp();
      xwhi = sw.x[kSortWin];
    }
    int jl = -1;
    if (k < k1) {
      T val[V];
      int jj[V];
      int l = 0, j = jc;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const T qq = qr[0][i];
        const bool in = (qq >= x0) && (qq <= xn);
        const T qc = in ? qq : x0;
        if (i == 0) {  // largest slot l <= 31 with x_{wb+l} <= qc (x_{wb} <= qc assumed; verified below)
          l = 0;
#pragma unroll
          for (int d = kSortWin / 2; d >= 1; d >>= 1) l = (sw.x[l + d] <= qc) ? l + d : l;
        } else {       // sorted: the previous query's slot, at most two intervals back
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const int p = min(l + 1, kSortWin - 1);
            l = (sw.x[p] <= qc) ? p : l;
          }
        }
        const WRec<T> r = ld_wrec(&sw.r[l]);
        const T rx1 = sw.x[l + 1];
        T v;
        if (qc >= r.x0 && (qc < rx1 || wb + l == n - 2)) {
          j = wb + l;
          v = cub_eval<T>(Cub<T>{r.ih, r.y0, r.dy, r.e1}, r.e2, r.x0, qc);
        } else {  // outside the window or a wrong hint: the general path from the last interval
          v = general_query<T, FORM_RECORD>(X, Y, Z, n, qc, j);
        }
        val[i] = in ? v : qnan<T>();
        jj[i] = in ? j : -1;
        oor |= !in;
        if (in) jl = j;
      }
      VecIO<T, V>::store(ob + k, val);
      if (ib) VecIO<T, V>::store_idx(ib + k, jj);
    }
    const int jm = __reduce_max_sync(0xffffffffu, jl);
    if (jm >= 0) jc = jm;
#pragma unroll
    for (int d = 0; d < PF; ++d)
#pragma unroll
      for (int i = 0; i < V; ++i) qr[d][i] = qr[d + 1][i];
  }
  return oor;
}

#ifndef FS_SORTED_PF
#define FS_SORTED_PF 1
#endif
constexpr int kSortedPF = FS_SORTED_PF;  // query prefetch depth of k_eval_sorted (warp steps)
#ifndef FS_SORTED_SEARCH
#define FS_SORTED_SEARCH 0
#endif
// 1: sorted_run_win (branch-free search + advance + verify); 0: the window lift of sorted_run
// (measured faster on cfg4: 1113 vs 1266 us -- DESIGN.md)
constexpr bool kSortedSearchForm = FS_SORTED_SEARCH != 0;
#ifndef FS_SORTED_MINB
#define FS_SORTED_MINB 4
#endif
template <typename T, int V, int FORM = FORM_RECORD, bool WIN = false>
__global__ void __launch_bounds__(256, FS_SORTED_MINB) k_eval_sorted(unsigned *__restrict__ status, const T *__restrict__ x,
                                                       const T *__restrict__ y, const T *__restrict__ y2, int n,
                                                       const T *__restrict__ q, int64_t m, T *__restrict__ out,
                                                       int32_t *__restrict__ idx, int64_t qrun,
                                                       int64_t runs_per_curve, int64_t ntasks) {
  static_assert(!WIN || FORM == FORM_RECORD, "the record window serves the product form");
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch)
  const int lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (task >= ntasks) return;  // whole warp; no block-level synchronisation below
  const int64_t c = task / runs_per_curve;
  const int64_t k0 = (task - c * runs_per_curve) * qrun;
  const int64_t k1 = min64(m, k0 + qrun);
  __shared__ SortWin<T> wins[8];  // one per warp of the 256-thread CTA
  bool oor;
  if constexpr (WIN && kSortedSearchForm)
    oor = sorted_run_win<T, V, kSortedPF>(x + c * n, y + c * n, ZGlobal<T>{y2 + c * n}, n, q + c * m, out + c * m,
                                          idx ? idx + c * m : nullptr, k0, k1, wins[threadIdx.x >> 5], lane);
  else
    oor = sorted_run<T, V, FORM, WIN, kSortedPF>(x + c * n, y + c * n, ZGlobal<T>{y2 + c * n}, n, q + c * m,
                                                   out + c * m, idx ? idx + c * m : nullptr, k0, k1,
                                                   wins[threadIdx.x >> 5], lane);
  raise_status_warp(status, oor, kOutOfRange);
}

// ---- dense sorted runs: each lane walks its own contiguous queries (k_eval_walk) -----------
// A warp takes its run in supersteps of kWalkQ = 256 queries.  The superstep's queries are
// loaded coalesced (256-bit accesses: 1 KB per warp instruction) and transposed through a padded
// shared-memory stage so that lane l owns queries [8l, 8l+8) -- consecutive, hence (sorted) in the
// same or the next interval.  Lane l locates its first query in the warp's window of 32 interval
// records (built at the carry, as in sorted_run) by a 5-level branch-free search, keeps that
// interval's record in REGISTERS and walks: each next query advances the slot by one when it
// passes the record's right knot (predicated: no branch), and is verified against the record's
// [x0, x1); a query that jumps further, falls outside the window or arrives out of order (a wrong
// sorted hint) takes the general path.  Results go back through the stage and out with 256-bit
// stores.  Per query: one shared-memory load, a compare, the 7-operation cubic and two stores --
// against the window lift + record load of sorted_run.  Bitwise the other forms (make_cub +
// cub_eval on the same interval).
constexpr int kWalkQ = 256, kWalkPer = kWalkQ / 32, kWalkPad = kWalkPer + 1;
#ifndef FS_WALK_REBUILD
#define FS_WALK_REBUILD 4
#endif
constexpr int kWalkRebuild = FS_WALK_REBUILD;
template <typename T> struct WalkStage {
  T q[32 * kWalkPad];        // queries, then the results in place (row l = lane l's 8, padded)
  int32_t j[32 * kWalkPad];  // interval indices
};

template <typename T, typename ZA>
__device__ __forceinline__ bool walk_run(const T *__restrict__ X, const T *__restrict__ Y, const ZA &Z, int n,
                                         const T *__restrict__ qb, T *__restrict__ ob, int32_t *__restrict__ ib,
                                         int64_t k0, int64_t k1, SortWin<T> &sw, WalkStage<T> &st, int lane) {
  constexpr int VE = 32 / sizeof(T);  // elements per 256-bit access
  constexpr int NI = kWalkQ / (32 * VE);  // 256-bit loads per lane per superstep
  const T x0 = __ldg(X), xn = __ldg(X + n - 1);
  T qf = __ldg(qb + k0);
  qf = (qf >= x0 && qf <= xn) ? qf : x0;
  int jc = warp_locate(X, n, qf, lane);
  bool oor = false;
  int wb = -(1 << 30);
  // this superstep's queries in registers (coalesced), the next superstep's in flight
  T qn[NI][VE];
#pragma unroll
  for (int a = 0; a < NI; ++a) {
    const int64_t k = k0 + (int64_t)(a * 32 + lane) * VE;
    if (k < k1) ld_cs_256(qb + k, qn[a]);
  }
  for (int64_t base = k0; base < k1; base += kWalkQ) {
    // stage: 256-bit group g = a*32 + lane holds queries [g VE, g VE + VE) -> row (g VE) / 8
    __syncwarp();
#pragma unroll
    for (int a = 0; a < NI; ++a) {
      const int g = (a * 32 + lane) * VE;
#pragma unroll
      for (int e = 0; e < VE; ++e) st.q[(g + e) / kWalkPer * kWalkPad + (g + e) % kWalkPer] = qn[a][e];
    }
#pragma unroll
    for (int a = 0; a < NI; ++a) {
      const int64_t k = base + kWalkQ + (int64_t)(a * 32 + lane) * VE;
      if (k < k1) ld_cs_256(qb + k, qn[a]);  // next superstep in flight
    }
    // the window at the carry (warp-uniform): a superstep spans ~kWalkQ / density intervals
    // (16 on cfg4) beyond the carry, so the window moves on as soon as the carry is 4 past its base
    if (jc < wb || jc - wb > kWalkRebuild) {
      wb = jc;
      const int jw = wb + lane;
      if (jw <= n - 2) {
        const T xa = __ldg(X + jw), xb = __ldg(X + jw + 1);
        T e2;
        const Cub<T> cb = make_cub<T>(xa, xb, __ldg(Y + jw), __ldg(Y + jw + 1), Z(jw), Z(jw + 1), e2);
        sw.r[lane] = WRec<T>{xa, cb.ih, cb.y0, cb.dy, cb.e1, e2};
        sw.x[lane] = xa;
        if (lane == kSortWin - 1) sw.x[kSortWin] = xb;
      } else {
        sw.x[lane] = inf_of<T>();
        if (lane == kSortWin - 1) sw.x[kSortWin] = inf_of<T>();
      }
      if constexpr (kSortedL1Prefetch) {
        if (lane < 9) {
          const int a = lane / 3, part = lane % 3;
          const T *pb = a == 0 ? X : a == 1 ? Y : Z.prefetch_ptr();
          if (pb) prefetch_l1(pb + min(wb + kSortWin + part * (128 / (int)sizeof(T)), n - 1));
        }
      }
    }
    __syncwarp();
    // lane l: queries [8l, 8l+8) of the superstep
    const int nq = (int)min64(kWalkPer, k1 - base - (int64_t)lane * kWalkPer);
    T *rq = st.q + lane * kWalkPad;
    int32_t *rj = st.j + lane * kWalkPad;
    int jl = -1;
    if (nq > 0) {
      const T q0 = rq[0];
      const T qs = (q0 >= x0 && q0 <= xn) ? q0 : x0;
      int l = 0;
#pragma unroll
      for (int d = kSortWin / 2; d >= 1; d >>= 1) l = (sw.x[l + d] <= qs) ? l + d : l;
      WRec<T> r = ld_wrec(&sw.r[l]);
      T xr = sw.x[l + 1];
      int j = wb + l;
#pragma unroll
      for (int i = 0; i < kWalkPer; ++i) {
        if (i < nq) {
          const T qq = rq[i];
          const bool in = (qq >= x0) && (qq <= xn);
          const T qc = in ? qq : x0;
          if (qc >= xr && l < kSortWin - 1) {  // the next interval (predicated reload)
            ++l;
            r = ld_wrec(&sw.r[l]);
            xr = sw.x[l + 1];
          }
          T v;
          if (qc >= r.x0 && (qc < xr || wb + l == n - 2)) {
            j = wb + l;
            v = cub_eval<T>(Cub<T>{r.ih, r.y0, r.dy, r.e1}, r.e2, r.x0, qc);
          } else {  // a longer jump, past the window, or out of order: the general path
            j = max(0, min(j, n - 2));
            v = general_query<T, FORM_RECORD>(X, Y, Z, n, qc, j);
            if (j - wb >= 0 && j - wb < kSortWin) {  // resynchronise the walk at the found interval
              l = j - wb;
              r = ld_wrec(&sw.r[l]);
              xr = sw.x[l + 1];
            }
          }
          rq[i] = in ? v : qnan<T>();
          rj[i] = in ? j : -1;
          oor |= !in;
          if (in) jl = j;
        }
      }
    }
    __syncwarp();
    // results out: the same 256-bit groups the queries came in
#pragma unroll
    for (int a = 0; a < NI; ++a) {
      const int g = (a * 32 + lane) * VE;
      const int64_t k = base + g;
      if (k < k1) {
        T v[VE];
        int jv[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          v[e] = st.q[(g + e) / kWalkPer * kWalkPad + (g + e) % kWalkPer];
          jv[e] = st.j[(g + e) / kWalkPer * kWalkPad + (g + e) % kWalkPer];
        }
        st_cs_256(ob + k, v);
        if (ib) VecIO<int32_t, VE>::store_idx(ib + k, jv);
      }
    }
    const int jm = __reduce_max_sync(0xffffffffu, jl);
    if (jm >= 0) jc = jm;
  }
  return oor;
}

template <typename T>
__global__ void __launch_bounds__(256, FS_SORTED_MINB) k_eval_walk(unsigned *__restrict__ status, const T *__restrict__ x,
                                                                   const T *__restrict__ y, const T *__restrict__ y2,
                                                                   int n, const T *__restrict__ q, int64_t m,
                                                                   T *__restrict__ out, int32_t *__restrict__ idx,
                                                                   int64_t qrun, int64_t runs_per_curve,
                                                                   int64_t ntasks) {
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (task >= ntasks) return;
  const int64_t c = task / runs_per_curve;
  const int64_t k0 = (task - c * runs_per_curve) * qrun;
  const int64_t k1 = min64(m, k0 + qrun);
  __shared__ SortWin<T> wins[8];
  __shared__ WalkStage<T> stages[8];
  const bool oor = walk_run<T>(x + c * n, y + c * n, ZGlobal<T>{y2 + c * n}, n, q + c * m, out + c * m,
                               idx ? idx + c * m : nullptr, k0, k1, wins[w], stages[w], lane);
  raise_status_warp(status, oor, kOutOfRange);
}

// ---- long curves through interval records in HBM ---------------------------------------
// k_pack_records writes, per curve c, the interval records R[c n + j] (j < n-1; the full
// common.cuh Ival, 32 B fp32 / 64 B fp64, one aligned DRAM burst) and a header
// {x_0, x_{n-1}, (n-1)/(x_{n-1} - x_0)}; k_eval_records then needs ONE gather round trip per
// query on near-uniform grids (the interpolation guess g, checked against the record's own
// x_g, x_{g+1}) instead of the two dependent trips and 4-5 scattered sectors of x, y, y2.
// Algorithmic cost of the pack: read 3 s B and write sizeof(Ival) B per knot (workspace).
// 256-bit global accesses (LDG.256 / STG.256 on sm_100a): one instruction per full 32-byte
// sector, so a record is requested from L2 exactly once per sector.
__device__ __forceinline__ void ld256(const void *p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld256(const void *p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void st256(void *p, const double (&v)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}
__device__ __forceinline__ void st256(void *p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

template <typename T> __device__ __forceinline__ Ival<T> ld_ival(const Ival<T> *p) {
  constexpr int W = 32 / sizeof(T);  // elements per 256-bit access
  Ival<T> r;
  T *d = reinterpret_cast<T *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Ival<T>) / 32); ++i) {
    T v[W];
    ld256(reinterpret_cast<const char *>(p) + 32 * i, v);
#pragma unroll
    for (int k = 0; k < W; ++k) d[i * W + k] = v[k];
  }
  return r;
}
template <typename T> __device__ __forceinline__ void st_ival(Ival<T> *p, const Ival<T> &r) {
  constexpr int W = 32 / sizeof(T);
  const T *d = reinterpret_cast<const T *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Ival<T>) / 32); ++i) {
    T v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) v[k] = d[i * W + k];
    st256(reinterpret_cast<char *>(p) + 32 * i, v);
  }
}

// KP consecutive knots per thread (one curve-aligned run), each loaded once: the run's x, y,
// y2 plus the first knot of the next run, then KP records stored with 256-bit stores.
template <typename T>
__global__ void __launch_bounds__(256) k_pack_records(const T *__restrict__ x, const T *__restrict__ y,
                                                      const T *__restrict__ y2, int n, int64_t batch,
                                                      Ival<T> *__restrict__ R, CurveHdr<T> *__restrict__ H) {
  pdl_wait();  // x, y, y2 may come from the preceding kernel (programmatic launch)
  constexpr int KP = 4;
  const int runs = (n + KP - 1) / KP;  // runs per curve
  const int64_t total = batch * runs;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = (batch == 1) ? 0 : e / runs;
    const int j0 = (int)(e - c * runs) * KP;
    const int64_t b = c * n + j0;
    const int cnt = min(KP + 1, n - j0);  // knots of the run, + the next run's first
    T xv[KP + 1], yv[KP + 1], zv[KP + 1];
#pragma unroll
    for (int i = 0; i < KP + 1; ++i) {
      if (i < cnt) {
        xv[i] = __ldg(x + b + i);
        yv[i] = __ldg(y + b + i);
        zv[i] = __ldg(y2 + b + i);
      }
    }
#pragma unroll
    for (int i = 0; i < KP; ++i)
      if (i + 1 < cnt) st_ival(R + b + i, make_ival<T>(xv[i], xv[i + 1], yv[i], yv[i + 1], zv[i], zv[i + 1]));
    if (j0 + cnt == n) {  // the run holding the curve's last knot writes the header
      const T x0 = __ldg(x + c * n), xn = xv[cnt - 1];
      H[c] = CurveHdr<T>{x0, xn, (T)(n - 1) / (xn - x0), T(0)};
    }
  }
}

// U independent queries per thread; per query: the guess g = (q - x_0)(n-1)/(x_{n-1} - x_0),
// one record; if x_g <= q < x_{g+1} fails (jitter, or a non-uniform grid) the neighbour on the
// indicated side, then a bisection over the records' x_j (any grid: never a wrong idx).
template <typename T>
__global__ void __launch_bounds__(256) k_eval_records(unsigned *__restrict__ status, const Ival<T> *__restrict__ R, const CurveHdr<T> *__restrict__ H,
                                                      int n, int64_t batch, const T *__restrict__ q, int64_t m,
                                                      T *__restrict__ out, int32_t *__restrict__ idx) {
  constexpr int U = 4;
  const int64_t total = batch * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool oor = false;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += U * stride) {
    T qc[U];
    int g[U];
    int64_t off[U];
    bool act[U], in[U];
    Ival<T> r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = base + u * stride;
      act[u] = k < total;
      const T qq = act[u] ? ld_stream(q + k) : T(0);
      const int64_t c = (batch == 1) ? 0 : (act[u] ? k / m : 0);
      off[u] = c * n;
      const CurveHdr<T> hd = H[c];
      qc[u] = fmin(fmax(qq, hd.x0), hd.xn);
      in[u] = act[u] && (qc[u] == qq);
      g[u] = max(0, min((int)r_mul(r_sub(qc[u], hd.x0), hd.s), n - 2));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld_ival(R + off[u] + g[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool below = qc[u] < r[u].x0;
      const bool above = !(qc[u] < r[u].x1) && g[u] < n - 2;
      if (below || above) {
        const Ival<T> *Rc = R + off[u];
        int j = below ? g[u] - 1 : g[u] + 1;
        Ival<T> t = ld_ival(Rc + j);
        if (!(t.x0 <= qc[u] && (qc[u] < t.x1 || j == n - 2))) {
          int lo = 0, hi = n - 1;  // bisection on x_j = R[j].x0
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(&Rc[mid].x0) <= qc[u]) lo = mid;
            else hi = mid;
          }
          j = lo;
          t = ld_ival(Rc + j);
        }
        g[u] = j;
        r[u] = t;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!act[u]) continue;
      const int64_t k = base + u * stride;
      const T v = ival_interp<T>(r[u], qc[u]);
      st_stream(out + k, in[u] ? v : qnan<T>());
      if (idx) st_stream(idx + k, in[u] ? (int32_t)g[u] : -1);
      oor |= !in[u];
    }
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(status, kOutOfRange);
}

// ---- diagnostics: the random-gather ceiling of the long-curve evaluation ---
// The access pattern alone, with the interval already known (idx_in, e.g. from spline_eval):
//   k_probe_raw : q, then x_j, x_{j+1}, y_j, y_{j+1}, y2_j, y2_{j+1} from the three arrays
//                 (the pattern of an evaluation without records), out = the cubic, idx copied;
//   k_probe_rec : q, then the one record of interval j (the pattern of k_eval_records).
// They do no search: their time is what the gathers themselves cost on this memory system.
template <typename T>
__global__ void __launch_bounds__(256) k_probe_raw(const T *__restrict__ x, const T *__restrict__ y,
                                                   const T *__restrict__ y2, int n, int64_t batch,
                                                   const T *__restrict__ q, int64_t m,
                                                   const int32_t *__restrict__ idx_in, T *__restrict__ out,
                                                   int32_t *__restrict__ idx) {
  const int64_t total = batch * m;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int j = __ldcs(idx_in + k);
    const int64_t off = (batch == 1) ? 0 : (k / m) * n;
    const int jj = max(j, 0);
    const T *X = x + off + jj, *Y = y + off + jj, *Z = y2 + off + jj;
    const T v = nr_interp(ld_stream(q + k), __ldg(X), __ldg(X + 1), __ldg(Y), __ldg(Y + 1), __ldg(Z), __ldg(Z + 1));
    st_stream(out + k, j >= 0 ? v : qnan<T>());
    st_stream(idx + k, j);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_probe_rec(const Ival<T> *__restrict__ R, int n, int64_t batch,
                                                   const T *__restrict__ q, int64_t m,
                                                   const int32_t *__restrict__ idx_in, T *__restrict__ out,
                                                   int32_t *__restrict__ idx);

template <typename T>
__global__ void __launch_bounds__(256) k_probe_rec(const Ival<T> *__restrict__ R, int n, int64_t batch,
                                                   const T *__restrict__ q, int64_t m,
                                                   const int32_t *__restrict__ idx_in, T *__restrict__ out,
                                                   int32_t *__restrict__ idx) {
  const int64_t total = batch * m;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int j = __ldcs(idx_in + k);
    const int64_t off = (batch == 1) ? 0 : (k / m) * n;
    const Ival<T> r = ld_ival(R + off + max(j, 0));
    const T v = ival_interp<T>(r, ld_stream(q + k));
    st_stream(out + k, j >= 0 ? v : qnan<T>());
    st_stream(idx + k, j);
  }
}

}  // namespace fs
