// fused.cuh -- spline_build_eval: construction (y2) and evaluation in ONE persistent kernel.
//
// evaluating right after the build (the paper's sweeps)
// without the round trip of y2 through HBM and without re-reading x, y.  Per work item
// (cpb curves with all their queries, or one chunk of one curve's queries):
//
//   TMA (cp.async.bulk)  x, y of item i -> knot stage i % 3, q of item i -> query stage i % 2
//                        [one mbarrier per stage]; a knot stage is refilled as soon as its
//                        item is packed, a query stage once its item is evaluated
//   solver warp(s)       raw x, y -> tridiagonal solve -> y2 tile i % 3 (+ y2 to HBM)
//                           n <= 8 : the paper's sweep in registers, one lane per curve
//                           n >  8 : two lanes per curve, the sweep from both ends meeting in
//                                    the middle (build_thomas.cuh babe_tile), on an
//                                    odd-stride transposed copy (conflict-free)
//   8 evaluator warps    pack the interval cubics + search keys, locate + Eq. nr_formula for the
//                        item's queries, 16-byte streaming stores of out / idx
//
// Warp specialisation: two solver warps take alternate items and work up to two items ahead of
// the evaluator warps;
// hand-offs are named barriers (bar.arrive / bar.sync): TFULL[s] "y2 tile s is ready",
// TEMPTY[s] "y2 tile s has been packed, the solver may overwrite it".  The solve
// (a serial chain of ~n/2 dependent steps per curve) is latency-bound; overlapping it with
// the issue-bound evaluation of the previous item hides it.
//
// Arithmetic is the same as the separate kernels: the solver runs babe_tile / thomas_regs
// of K1 / K1r, the evaluators run pack_item + eval_item_queries of k_eval_staged, so
// spline_build_eval gives bitwise the y2, out and idx of spline_build followed by
// spline_eval (tested).
#pragma once
#include "build_thomas.cuh"
#include "eval.cuh"

namespace fs {

__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

enum { SOLVE_REGS = 0, SOLVE_BABE = 1 };
constexpr int kFusedEvalWarps = 8;
constexpr int kFusedEvalThreads = 32 * kFusedEvalWarps;
constexpr int kRegsNMax = 8;     // SOLVE_REGS for n <= 8
constexpr int kBabeCurves = 16;  // curves per solver-warp pass (2 lanes each)
constexpr int kKnotStages = 3;   // x, y (+ y2 tile) stages
constexpr int kQueryStages = 2;
// solver warps per CTA, each solving whole items in turn: 4 with per-warp ownership (the
// hand-offs are mbarriers, see the solver's tempty wait); 1 otherwise -- several solvers
// would share a named barrier id for different items.
__host__ __device__ constexpr int fused_solver_warps(bool wown) { return wown ? 4 : 1; }
__host__ __device__ constexpr int fused_threads(bool wown) { return kFusedEvalThreads + 32 * fused_solver_warps(wown); }
// named barrier ids (0 is __syncthreads)
enum { BAR_EVAL = 1, BAR_TFULL = 2, BAR_TEMPTY = 2 + kKnotStages };

template <typename T> struct FusedLayout {
  size_t kst0, kststep, qst0, qststep, ytile, ytstep, scratch, scrstep, knots, e2, xk, hdr, xs, total;
  int P, S2;
  __host__ __device__ FusedLayout(int cpb, int n, int qmax, int solve, int mode, bool wown) {
    P = 1 << eytz_levels(n);
    S2 = (solve == SOLVE_BABE) ? babe_stride(n) : n;
    size_t off = 128;  // mbarriers (knot stages, query stages, tile full, tile empty) + counters
    kst0 = off;
    kststep = align16(2 * sizeof(T) * (size_t)cpb * n);
    off += kKnotStages * kststep;
    qst0 = off;
    qststep = align16(sizeof(T) * (size_t)qmax);
    off += kQueryStages * qststep;
    ytile = off;
    ytstep = align16(sizeof(T) * (size_t)cpb * S2);
    off += kKnotStages * ytstep;
    scratch = off;  // per solver warp: c' rows of one babe pass + 2 rows for inactive pairs
    scrstep = (solve == SOLVE_BABE) ? align16(sizeof(T) * (size_t)(kBabeCurves + 2) * S2) : 0;
    off += fused_solver_warps(wown) * scrstep;
    knots = off;
    off = align16(off + sizeof(Cub<T>) * (size_t)cpb * n);
    e2 = off;
    off = align16(off + sizeof(T) * (size_t)cpb * n);
    xk = off;
    if (mode != MODE_BISECT) off = align16(off + sizeof(T) * (size_t)cpb * n);
    hdr = off;
    off = align16(off + sizeof(CurveHdr<T>) * (size_t)cpb);
    xs = off;
    if (mode == MODE_BISECT) off = align16(off + sizeof(T) * (size_t)cpb * P);
    total = off;
  }
};

// Solver warp, SOLVE_BABE: curves [0, nc) of the item in passes of 16 (2 lanes each).
template <typename T>
__device__ __forceinline__ void fused_solve_babe(unsigned *__restrict__ status, const T *Xr, const T *Yr, T *Yt, T *scr, int S, int n, int nc,
                                                 int64_t c0, int bc, const T *__restrict__ yp1,
                                                 const T *__restrict__ ypn, T *__restrict__ y2, FastDiv divn,
                                                 int lane, int sw, int nsw) {
  constexpr int VW = 16 / sizeof(T);
  using VT = typename Vec16<T>::V;
  T *Xs = scr, *dummy = scr + kBabeCurves * S;
  for (int p0 = sw * kBabeCurves; p0 < nc; p0 += nsw * kBabeCurves) {
    const int np = min(kBabeCurves, nc - p0);
    T *Yp = Yt + (size_t)p0 * S;
    const T sl = babe_slope(c0 + p0, np, bc, yp1, ypn, lane);  // in flight during the transposition
    // transpose x, y of the pass into the tiles (16-byte reads of the raw stage)
    const int tot = np * n;
    for (int e = lane * VW; e < tot; e += 32 * VW) {
      const int c = (int)divn.div((uint32_t)e);
      const int j = e - c * n;
      const VT a = *reinterpret_cast<const VT *>(Xr + (size_t)p0 * n + e);
      const VT b = *reinterpret_cast<const VT *>(Yr + (size_t)p0 * n + e);
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        Xs[c * S + j + i] = reinterpret_cast<const T *>(&a)[i];
        Yp[c * S + j + i] = reinterpret_cast<const T *>(&b)[i];
      }
    }
    __syncwarp();
    babe_tile(status, Xs, Yp, S, n, np, bc, sl, dummy, lane);
    __syncwarp();
    if (y2) {
      T *yb = y2 + (c0 + p0) * n;
      for (int e = lane * VW; e < tot; e += 32 * VW) {
        const int c = (int)divn.div((uint32_t)e);
        const int j = e - c * n;
        VT a;
#pragma unroll
        for (int i = 0; i < VW; ++i) reinterpret_cast<T *>(&a)[i] = Yp[c * S + j + i];
        __stcs(reinterpret_cast<VT *>(yb + e), a);
      }
    }
    __syncwarp();  // scratch rows are reused by the next pass
  }
}

// Solver warp, SOLVE_REGS (n <= 8, n * sizeof(T) % 16 == 0): one lane per curve, the
// paper's sweep in registers (thomas_regs).
template <typename T>
__device__ __forceinline__ void fused_solve_regs(unsigned *__restrict__ status, const T *Xr, const T *Yr, T *Yt, int n, int nc, int64_t c0, int bc,
                                                 const T *__restrict__ yp1, const T *__restrict__ ypn,
                                                 T *__restrict__ y2, int lane, int sw, int nsw) {
  constexpr int VW = 16 / sizeof(T);
  constexpr int NM = kRegsNMax;
  using VT = typename Vec16<T>::V;
  for (int p0 = sw * 32; p0 < nc; p0 += nsw * 32) {
    const int c = p0 + lane;
    bool ok = true;
    if (c < nc) {
      T xv[NM], yv[NM], z[NM];
#pragma unroll
      for (int j = 0; j < NM; j += VW) {
        if (j < n) {
          const VT a = *reinterpret_cast<const VT *>(Xr + (size_t)c * n + j);
          const VT b = *reinterpret_cast<const VT *>(Yr + (size_t)c * n + j);
#pragma unroll
          for (int i = 0; i < VW; ++i) {
            xv[j + i] = reinterpret_cast<const T *>(&a)[i];
            yv[j + i] = reinterpret_cast<const T *>(&b)[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < VW; ++i) xv[j + i] = yv[j + i] = T(0);
        }
      }
      const int64_t cg = c0 + c;
      ok = thomas_regs<T, NM>(xv, yv, n, bc, (bc & 1) ? yp1[cg] : T(0), (bc & 2) ? ypn[cg] : T(0), z);
#pragma unroll
      for (int j = 0; j < NM; j += VW) {
        if (j < n) {
          VT a;
#pragma unroll
          for (int i = 0; i < VW; ++i) reinterpret_cast<T *>(&a)[i] = z[j + i];
          *reinterpret_cast<VT *>(Yt + (size_t)c * n + j) = a;
          if (y2) __stcs(reinterpret_cast<VT *>(y2 + cg * n + j), a);
        }
      }
    }
    raise_status_warp(status, !ok, kBadKnots);
  }
}

// Requirements (checked by the host): x, y, q, out 16-byte aligned, idx 4V-byte aligned,
// n * sizeof(T) % 16 == 0, m % V == 0 (V = 16 / sizeof(T)), 3 <= n <= 128.
// WOWN (cpb a multiple of 8): evaluator warp w owns curves [w cpb/8, (w+1) cpb/8) of every item
// -- it packs and evaluates them with no CTA-wide barrier; hand-offs are mbarriers (tile full:
// solver -> warps; tile empty: 8 warp arrivals -> solver) and the last warp done with a stage
// (shared counter) refills it.  Otherwise (chunked single curves) the CTA packs together and
// the hand-offs are named barriers.
template <typename T, int MODE, int L2, int SOLVE, bool WOWN>
__global__ void __launch_bounds__(fused_threads(WOWN), WOWN ? 2 : 3)
    k_fused_staged(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int n, int64_t batch, int bc,
                   const T *__restrict__ yp1, const T *__restrict__ ypn, T *__restrict__ y2, const T *__restrict__ q,
                   int m, T *__restrict__ out, int32_t *__restrict__ idx, int cpb, int nchunks, int qchunk, int qmax,
                   int64_t nitems, FastDiv divn, FastDiv divm) {
  constexpr int V = 16 / sizeof(T);
  constexpr int NSW = fused_solver_warps(WOWN);
  constexpr int NB = kFusedEvalThreads + 32;  // named-barrier participants: evaluators + one solver warp
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const FusedLayout<T> L(cpb, n, qmax, SOLVE, MODE, WOWN);
  uint64_t *kbar = reinterpret_cast<uint64_t *>(smem_raw);  // [kKnotStages]
  uint64_t *qbar = kbar + kKnotStages;                       // [kQueryStages]
  uint64_t *tfull = qbar + kQueryStages;                     // [kKnotStages]  (WOWN)
  uint64_t *tempty = tfull + kKnotStages;                    // [kKnotStages]  (WOWN)
  int *kcnt = reinterpret_cast<int *>(tempty + kKnotStages);  // [kKnotStages]  (WOWN)
  int *qcnt = kcnt + kKnotStages;                            // [kQueryStages] (WOWN)
  Cub<T> *KP = reinterpret_cast<Cub<T> *>(smem_raw + L.knots);
  T *KE = reinterpret_cast<T *>(smem_raw + L.e2);
  T *XK = reinterpret_cast<T *>(smem_raw + L.xk);
  CurveHdr<T> *Hd = reinterpret_cast<CurveHdr<T> *>(smem_raw + L.hdr);
  T *Xs = reinterpret_cast<T *>(smem_raw + L.xs);
  const int P = L.P, S2 = L.S2;
  const int64_t G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t cn = (size_t)cpb * n;

  auto kstage = [&](int s) { return reinterpret_cast<T *>(smem_raw + L.kst0 + (size_t)s * L.kststep); };
  auto qstage = [&](int s) { return reinterpret_cast<T *>(smem_raw + L.qst0 + (size_t)s * L.qststep); };
  auto ytile = [&](int s) { return reinterpret_cast<T *>(smem_raw + L.ytile + (size_t)s * L.ytstep); };
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
  auto issue_knots = [&](int64_t it, int s) {  // one thread
    if (it >= nitems) return;
    int64_t c0, k0;
    int nc, cnt;
    item_of(it, c0, k0, nc, cnt);
    const uint32_t bytes = (uint32_t)((size_t)nc * n * sizeof(T));
    mbar_expect_tx(kbar + s, 2 * bytes);
    bulk_g2s(kstage(s), x + c0 * n, bytes, kbar + s);
    bulk_g2s(kstage(s) + cn, y + c0 * n, bytes, kbar + s);
  };
  auto issue_queries = [&](int64_t it, int s) {  // one thread
    if (it >= nitems) return;
    int64_t c0, k0;
    int nc, cnt;
    item_of(it, c0, k0, nc, cnt);
    const uint32_t qbytes = (uint32_t)((size_t)cnt * sizeof(T));
    mbar_expect_tx(qbar + s, qbytes);
    bulk_g2s(qstage(s), q + k0, qbytes, qbar + s);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKnotStages; ++s) {
      mbar_init(kbar + s, 1);
      mbar_init(tfull + s, 1);
      mbar_init(tempty + s, kFusedEvalWarps);
      kcnt[s] = 0;
    }
    for (int s = 0; s < kQueryStages; ++s) {
      mbar_init(qbar + s, 1);
      qcnt[s] = 0;
    }
  }
  __syncthreads();
  const int64_t first = blockIdx.x;
  const int nmine = first < nitems ? (int)((nitems - 1 - first) / G + 1) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kKnotStages; ++s) issue_knots(first + s * G, s);
    for (int s = 0; s < kQueryStages; ++s) issue_queries(first + s * G, s);
  }
  bool oor = false;

  if (warp >= kFusedEvalWarps) {
    // ---------------- solver warps: warp sw takes the items k = sw, sw + NSW, ... whole, so
    // NSW solves (latency-bound dependency chains) are in flight at once
    const int sw = warp - kFusedEvalWarps;
    for (int k = sw; k < nmine; k += NSW) {
      const int ks = k % kKnotStages;
      const int64_t it = first + (int64_t)k * G;
      int64_t c0, k0;
      int nc, cnt;
      item_of(it, c0, k0, nc, cnt);
      if constexpr (WOWN) {
        // item k-3 packed.  A solver reaching item k has finished item k-NSW, so stage ks may be
        // up to ceil(NSW/3) completions behind; a parity wait only tells phases one apart, so
        // wait for each of them in order (one wait for NSW <= 2).
#pragma unroll
        for (int back = (NSW + kKnotStages - 1) / kKnotStages; back >= 1; --back)
          if (k / kKnotStages - back >= 0) mbar_wait(tempty + ks, (uint32_t)(k / kKnotStages - back) & 1u);
        mbar_wait(kbar + ks, (uint32_t)(k / kKnotStages) & 1u);
      } else {
        mbar_wait(kbar + ks, (uint32_t)(k / kKnotStages) & 1u);
        if (k >= kKnotStages) nbar_sync(BAR_TEMPTY + ks, NB);  // tile ks packed (item k-3)
      }
      const T *Xr = kstage(ks);
      const T *Yr = Xr + cn;
      T *y2o = (y2 && (cpb > 1 || it % nchunks == 0)) ? y2 : nullptr;  // chunk 0 writes y2
      if constexpr (SOLVE == SOLVE_BABE)
        fused_solve_babe<T>(status, Xr, Yr, ytile(ks), reinterpret_cast<T *>(smem_raw + L.scratch + sw * L.scrstep), S2, n,
                            nc, c0, bc, yp1, ypn, y2o, divn, lane, 0, 1);
      else
        fused_solve_regs<T>(status, Xr, Yr, ytile(ks), n, nc, c0, bc, yp1, ypn, y2o, lane, 0, 1);
      __syncwarp();
      if constexpr (WOWN) {
        if (lane == 0) mbar_arrive(tfull + ks);
      } else {
        nbar_arrive(BAR_TFULL + ks, NB);
      }
    }
  } else if constexpr (WOWN) {
    // ---------------- evaluator warps, per-warp curve ownership
    const int cpw = cpb / kFusedEvalWarps;
    for (int k = 0; k < nmine; ++k) {
      const int ks = k % kKnotStages, qs = k % kQueryStages;
      const int64_t it = first + (int64_t)k * G;
      const int64_t c0 = it * cpb;
      const int nc = (int)min64(cpb, batch - c0);
      mbar_wait(tfull + ks, (uint32_t)(k / kKnotStages) & 1u);  // y2 tile ks ready (so the stage landed)
      mbar_wait(kbar + ks, (uint32_t)(k / kKnotStages) & 1u);   // completes at once; orders the TMA writes
      const int cw0 = warp * cpw, nmy = min(cpw, nc - cw0);
      const T *X = kstage(ks) + (size_t)cw0 * n;
      const T *Y = X + cn;
      const T *Z = ytile(ks) + (size_t)cw0 * S2;
      if (nmy > 0)
        pack_item<T, MODE, L2>(X, Y, Z, S2, nmy, n, 0, divn, KP + cw0 * n, KE + cw0 * n, XK + cw0 * n, Hd + cw0,
                               Xs + cw0 * P, nullptr, P, lane, 32);
      __syncwarp();
      if (lane == 0) {
        if (k + kKnotStages < nmine) mbar_arrive(tempty + ks);  // this warp is done with tile ks
        if (last_warp_arrival(kcnt + ks, kFusedEvalWarps)) {     // every warp is: refill knot stage ks
          fence_proxy_async();
          issue_knots(it + kKnotStages * G, ks);
        }
      }
      mbar_wait(qbar + qs, (uint32_t)(k / kQueryStages) & 1u);
      if (nmy > 0)
        oor |= eval_item_queries<T, MODE, V, true, L2, 1>(qstage(qs) + (size_t)cw0 * m, q, (c0 + cw0) * m, c0 + cw0, m,
                                                       nmy * m, cpb, divm, KP + cw0 * n, KE + cw0 * n, XK + cw0 * n,
                                                       Hd + cw0, Xs + cw0 * P, nullptr, X, Y, Z, n, 0, P, out, idx,
                                                       0, 1, lane);
      __syncwarp();
      if (lane == 0 && last_warp_arrival(qcnt + qs, kFusedEvalWarps)) {
        fence_proxy_async();
        issue_queries(it + kQueryStages * G, qs);
      }
    }
  } else {
    // ---------------- evaluator warps
    for (int k = 0; k < nmine; ++k) {
      const int ks = k % kKnotStages, qs = k % kQueryStages;
      const int64_t it = first + (int64_t)k * G;
      int64_t c0, k0;
      int nc, cnt;
      item_of(it, c0, k0, nc, cnt);
      nbar_sync(BAR_TFULL + ks, NB);                           // y2 tile ks ready (so the stage landed)
      mbar_wait(kbar + ks, (uint32_t)(k / kKnotStages) & 1u);  // completes at once; orders the TMA writes
      const T *X = kstage(ks);
      const T *Y = X + cn;
      pack_item<T, MODE, L2>(X, Y, ytile(ks), S2, nc, n, 0, divn, KP, KE, XK, Hd, Xs, nullptr, P, threadIdx.x,
                             kFusedEvalThreads);
      if (k + kKnotStages < nmine) nbar_arrive(BAR_TEMPTY + ks, NB);  // this thread is done with tile ks
      nbar_sync(BAR_EVAL, kFusedEvalThreads);                          // packed data built; stage ks free
      if (threadIdx.x == 0) issue_knots(it + kKnotStages * G, ks);
      mbar_wait(qbar + qs, (uint32_t)(k / kQueryStages) & 1u);
      oor |= eval_item_queries<T, MODE, V, true, L2, kFusedEvalWarps>(qstage(qs), q, k0, c0, m, cnt, cpb, divm, KP, KE, XK,
                                                                      Hd, Xs, nullptr,
                                                     X, Y, ytile(ks), n, 0, P, out, idx, warp, kFusedEvalWarps,
                                                     lane);
      nbar_sync(BAR_EVAL, kFusedEvalThreads);  // done with query stage qs and the packed data
      if (threadIdx.x == 0) issue_queries(it + kQueryStages * G, qs);
    }
  }
  if (__syncthreads_or(oor) && threadIdx.x == 0) raise_status(status, kOutOfRange);
}

}  // namespace fs
