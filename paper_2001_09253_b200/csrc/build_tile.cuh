// build_tile.cuh -- K2..K5: partitioned tridiagonal solve (mid-length curves and long curves).
//
// The system is the one of Eq. init_val with natural (P:1062-1064,
// P:1096-1098) or clamped end rows.  It is strictly diagonally
// dominant and symmetric positive definite, so every elimination below is
// pivot-free (the paper's justification for Thomas), and the GPU remark of
// P:815-821 (fewer serial steps via the parallel tridiagonal literature) is what this
// file implements.
//
// Block record.  For a contiguous block of rows [p, q] whose couplings to the outside
// unknowns L = y_{p-1} and R = y_{q+1} are moved to the right-hand side, the block's
// solution is affine in (L, R).  Only its two tips are kept:
//     y_p = Gp - Vp L - Wp R,        y_q = Gq - Vq L - Wq R          (6 scalars)
// (SURVEY.md Appendix A's spike tips g, v, w).  Records of adjacent blocks merge
// associatively (a 2x2 solve for the two rows at the seam, determinant 1 - A.Wq B.Vp > 0
// by diagonal dominance), and the merge is reversed top-down once the outer L, R are
// known.  One machinery serves three levels:
//   leaf   : one thread, R consecutive rows -- a Thomas forward sweep with
//            three right-hand sides (d, a_p e_1, c_q e_q) and a backward Horner pass;
//   tile   : one CTA, 256 leaves -- merge tree in registers (warp shuffles; tile_tree_up/down);
//   curve  : tiles of one long curve (and ranks of a multi-GPU curve) -- k4_top.
// The final per-row solve is the paper's back-substitution:
// y_i = g'_i - v'_i L - c'_i y_{i+1}.
#pragma once
#include "common.cuh"

namespace fs {

template <typename T> struct Rec { T Gp, Vp, Wp, Gq, Vq, Wq; };

// Merge adjacent block records A = [p, m], B = [m+1, q] into [p, q].
template <typename T> __device__ __forceinline__ Rec<T> merge_rec(const Rec<T> &A, const Rec<T> &B) {
  const T iD = nr_rcp(T(1) - A.Wq * B.Vp);
  const T Gm = (A.Gq - A.Wq * B.Gp) * iD, Vm = A.Vq * iD, Wm = -(A.Wq * B.Wp) * iD;    // y_m
  const T Gm1 = (B.Gp - B.Vp * A.Gq) * iD, Vm1 = -(B.Vp * A.Vq) * iD, Wm1 = B.Wp * iD;  // y_{m+1}
  Rec<T> o;
  o.Gp = A.Gp - A.Wp * Gm1;
  o.Vp = A.Vp - A.Wp * Vm1;
  o.Wp = -(A.Wp * Wm1);
  o.Gq = B.Gq - B.Vq * Gm;
  o.Vq = -(B.Vq * Vm);
  o.Wq = B.Wq - B.Vq * Wm;
  return o;
}

// Given the outer unknowns (L, R) of a merged block, recover the two seam rows
// y_m (last row of A) and y_{m+1} (first row of B) from A's q-tip and B's p-tip.
template <typename T>
__device__ __forceinline__ void split_seam(T AGq, T AVq, T AWq, T BGp, T BVp, T BWp, T L, T R, T &ym, T &ym1) {
  const T alpha = AGq - AVq * L;
  const T beta = BGp - BWp * R;
  ym = (alpha - AWq * beta) * nr_rcp(T(1) - AWq * BVp);
  ym1 = beta - BVp * ym;
}

// Block-level merge tree over nleaf <= blockDim.x records held in shared memory.  Level s
// (1, 2, 4..) merges rec[i] and rec[i+s] for i a multiple of 2s into rec[i], done by thread i;
// the six seam values of every merge are saved in mi[] for the top-down pass.  The levels
// with 2s <= 32 stay inside one warp (both children and the next level's reader are lanes of
// the same warp), so they need only __syncwarp; a CTA barrier separates the wider levels.
// Ends with __syncthreads().
template <typename T> __device__ void tree_up(Rec<T> *rec, T *mi, int nleaf) {
  const int t = threadIdx.x;
  int off = 0;
  for (int lg = 0; (1 << lg) < nleaf; ++lg) {  // s = 2^lg (shifts: the level sizes are powers of 2)
    const int s = 1 << lg;
    const int nn = (nleaf + 2 * s - 1) >> (lg + 1);
    if ((t & (2 * s - 1)) == 0 && t + s < nleaf) {
      const Rec<T> A = rec[t], B = rec[t + s];
      T *o = mi + 6 * (off + (t >> (lg + 1)));
      o[0] = A.Gq; o[1] = A.Vq; o[2] = A.Wq; o[3] = B.Gp; o[4] = B.Vp; o[5] = B.Wp;
      rec[t] = merge_rec(A, B);
    }
    off += nn;
    if (4 * s <= 32) __syncwarp();  // the next level (children 2s apart) is warp-local too
    else __syncthreads();
  }
  __syncthreads();
}

// Top-down: ext[i] = (L, R) of leaf i, given the root's (L, R); thread i splits the merges it
// made on the way up.  Ends with __syncthreads().
template <typename T> __device__ void tree_down(const T *mi, T *ext, int nleaf, T L, T R) {
  const int t = threadIdx.x;
  if (t == 0) { ext[0] = L; ext[1] = R; }
  int lgmax = 0, total = 0;
  for (int lg = 0; (1 << lg) < nleaf; ++lg) {
    lgmax = lg;
    total += (nleaf + (2 << lg) - 1) >> (lg + 1);
  }
  __syncthreads();
  if (nleaf == 1) return;
  int off = total;
  for (int lg = lgmax; lg >= 0; --lg) {
    const int s = 1 << lg;
    const int nn = (nleaf + 2 * s - 1) >> (lg + 1);
    off -= nn;
    if ((t & (2 * s - 1)) == 0 && t + s < nleaf) {
      const int j = t + s;
      const T *o = mi + 6 * (off + (t >> (lg + 1)));
      const T Li = ext[2 * t], Ri = ext[2 * t + 1];
      T ym, ym1;
      split_seam(o[0], o[1], o[2], o[3], o[4], o[5], Li, Ri, ym, ym1);
      ext[2 * t + 1] = ym1;
      ext[2 * j] = ym;
      ext[2 * j + 1] = Ri;
    }
    if (2 * s <= 32) __syncwarp();  // the next level's readers were written by their own warp
    else __syncthreads();
  }
  __syncthreads();
}

enum { TILE_FULL = 0, TILE_REDUCE = 1, TILE_FINISH = 2 };
// Diagnostic build only (-DFS_TILE_PHASES=1): thread 0 of every tile adds the SM cycles of each
// phase of tile_solve to g_tile_phase[] (read by spline_debug_tile_phases).  Off in the product.
#ifndef FS_TILE_PHASES
#define FS_TILE_PHASES 0
#endif
#if FS_TILE_PHASES
__device__ unsigned long long g_tile_phase[8];
#define TILE_MARK(k)                                              \
  do {                                                            \
    if (threadIdx.x == 0) {                                       \
      const long long t_ = clock64();                             \
      atomicAdd(&g_tile_phase[k], (unsigned long long)(t_ - tp_)); \
      tp_ = t_;                                                   \
    }                                                             \
  } while (0)
#else
#define TILE_MARK(k) \
  do {               \
  } while (0)
#endif
constexpr int kTileThreads = 256;
#ifndef FS_TILE_PREFETCH
#define FS_TILE_PREFETCH 1  // A/B at 3 CTAs/SM: cfg4 build 125.4 vs 133.1 us, cfg5 757 vs 840 us
#endif
constexpr int kTilePrefetchAhead = FS_TILE_PREFETCH;
#ifndef FS_TILE_WARP_STAGE
#define FS_TILE_WARP_STAGE 1
#endif
constexpr bool kTileWarpStage = FS_TILE_WARP_STAGE != 0;  // full tiles staged and stored per warp (no CTA barrier)
#ifndef FS_TILE_FINISH_REVERSE
#define FS_TILE_FINISH_REVERSE 1
#endif
constexpr bool kTileFinishReverse = FS_TILE_FINISH_REVERSE != 0;
#ifndef FS_TILE_PF_LATE
#define FS_TILE_PF_LATE 0  // A/B: cfg4 124.9 vs 125.0 us, cfg5 788 vs 755 us (prefetch at entry kept)
#endif
constexpr bool kTilePrefetchLate = FS_TILE_PF_LATE != 0;  // prefetch after the tile's own staging
#ifndef FS_TILE_STAGE_UNROLL
#define FS_TILE_STAGE_UNROLL 4
#endif
constexpr int kTileStageUnroll = FS_TILE_STAGE_UNROLL;
#ifndef FS_TILE_MINB
#define FS_TILE_MINB 3  // 3 tiles of 4096 fp64 rows per SM (76 KB each): cfg4 build 133.1 vs 138.2 us at 2
#endif  // staging loop unroll: vector loads per array in flight per thread  // waves ahead whose x, y a tile prefetches to L2

// Merge A, B like merge_rec, and also return the seam SOLVED for the outer unknowns:
//   y_m = Gm - Vm L - Wm R,   y_{m+1} = Gm1 - Vm1 L - Wm1 R      (sm = {Gm, Vm, Wm, Gm1, Vm1, Wm1})
// -- the intermediate values merge_rec computes anyway, so the top-down pass needs no
// reciprocal: each seam row is two fused multiply-adds from the block's (L, R).
template <typename T> __device__ __forceinline__ Rec<T> merge_rec_seam(const Rec<T> &A, const Rec<T> &B, T (&sm)[6]) {
  const T iD = nr_rcp(T(1) - A.Wq * B.Vp);
  const T Gm = (A.Gq - A.Wq * B.Gp) * iD, Vm = A.Vq * iD, Wm = -(A.Wq * B.Wp) * iD;    // y_m
  const T Gm1 = (B.Gp - B.Vp * A.Gq) * iD, Vm1 = -(B.Vp * A.Vq) * iD, Wm1 = B.Wp * iD;  // y_{m+1}
  sm[0] = Gm; sm[1] = Vm; sm[2] = Wm; sm[3] = Gm1; sm[4] = Vm1; sm[5] = Wm1;
  Rec<T> o;
  o.Gp = A.Gp - A.Wp * Gm1;
  o.Vp = A.Vp - A.Wp * Vm1;
  o.Wp = -(A.Wp * Wm1);
  o.Gq = B.Gq - B.Vq * Gm;
  o.Vq = -(B.Vq * Vm);
  o.Wq = B.Wq - B.Vq * Wm;
  return o;
}
// g - v L - w R
template <typename T> __device__ __forceinline__ T seam_row(T g, T v, T w, T L, T R) {
  return __fma_rn(-w, R, __fma_rn(-v, L, g));
}

// The tile's merge tree (tile_solve): the merges of tree_up over the tile's nleaf <= 256 leaves,
// in the same order and on the same operands (so the tile record is bitwise tree_up's), with the
// records in registers.  Levels 0-4 (blocks of up to 32 leaves) are inside a warp: the right
// child's record comes by shuffle from lane t+s; levels 5-7 merge the 8 warp records in warp 0,
// lanes 0-7.  Each merge's SOLVED seam (merge_rec_seam) goes to shared memory (TileTree::mi),
// except at level 0, where lane t keeps the half its own leaf needs on the way down in registers
// (k0: even t the y_{m+1} row -- its right neighbour --, odd t the y_m row -- its left one).
// Shared memory: 127 seams + 8 warp records -- 6.6 KB against the 24 KB of a record and a seam
// per leaf, which lets three 4096-row fp64 tiles share an SM.
__host__ __device__ constexpr int tile_levels() { return kTileThreads == 256 ? 8 : 0; }
static_assert(kTileThreads == 256, "the tile tree is written for 8 warps of leaves");
template <typename T> struct TileTree {
  T mi[6 * (kTileThreads / 2 - 1)];  // seams of levels 1..7: level lg at mi_off(lg) + (t >> (lg + 1))
  Rec<T> wrec[kTileThreads / 32];    // the warps' records (level 5's leaves)
  T wext[2 * (kTileThreads / 32)];   // the warps' (L, R)
};
__device__ __forceinline__ int mi_off(int lg) { return kTileThreads / 2 - (kTileThreads >> lg); }  // lg >= 1

template <typename T> __device__ __forceinline__ Rec<T> shfl_down_rec(const Rec<T> &r, int s) {
  Rec<T> o;
  o.Gp = __shfl_down_sync(0xffffffffu, r.Gp, s);
  o.Vp = __shfl_down_sync(0xffffffffu, r.Vp, s);
  o.Wp = __shfl_down_sync(0xffffffffu, r.Wp, s);
  o.Gq = __shfl_down_sync(0xffffffffu, r.Gq, s);
  o.Vq = __shfl_down_sync(0xffffffffu, r.Vq, s);
  o.Wq = __shfl_down_sync(0xffffffffu, r.Wq, s);
  return o;
}
template <typename T> __device__ __forceinline__ void put6(T *o, const T (&v)[6]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) o[i] = v[i];
}

// Bottom-up.  r: this thread's leaf record (any value when t >= nleaf).  Returns the tile's
// record in thread 0.  Every thread of the CTA must call it; ends with the warp-0 levels (no
// trailing barrier: tile_tree_down starts with one).
// notok: this thread's leaf saw bad knots; bad (out): any leaf of the tile did (the CTA barrier
// between the warp levels and warp 0's levels carries the OR).
template <typename T>
__device__ __forceinline__ Rec<T> tile_tree_up(Rec<T> r, int nleaf, TileTree<T> &tt, T (&k0)[3], bool notok, bool &bad) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  T km[3] = {T(0), T(0), T(0)};
#pragma unroll
  for (int lg = 0; lg < 5; ++lg) {
    const int s = 1 << lg;
    const Rec<T> B = shfl_down_rec(r, s);
    if ((t & (2 * s - 1)) == 0 && t + s < nleaf) {
      T sm[6];
      r = merge_rec_seam(r, B, sm);
      if (lg > 0) {
        put6(tt.mi + 6 * (mi_off(lg) + (t >> (lg + 1))), sm);
      } else {
        km[0] = sm[0]; km[1] = sm[1]; km[2] = sm[2];  // y_m's row: the odd neighbour's
        k0[0] = sm[3]; k0[1] = sm[4]; k0[2] = sm[5];  // y_{m+1}'s row: this lane's
      }
    }
    if (lg == 0) {
      const T a0 = __shfl_up_sync(0xffffffffu, km[0], 1), a1 = __shfl_up_sync(0xffffffffu, km[1], 1),
              a2 = __shfl_up_sync(0xffffffffu, km[2], 1);
      if (lane & 1) { k0[0] = a0; k0[1] = a1; k0[2] = a2; }
    }
  }
  if (lane == 0 && t < nleaf) tt.wrec[w] = r;
  bad = __syncthreads_or(notok);
  if (w == 0) {
    const int nw = (nleaf + 31) >> 5;
    r = tt.wrec[lane < nw ? lane : 0];
#pragma unroll
    for (int lg = 5; lg < tile_levels(); ++lg) {
      const int s = 1 << (lg - 5);  // in warps
      const Rec<T> B = shfl_down_rec(r, s);
      if ((lane & (2 * s - 1)) == 0 && lane + s < nw) {
        T sm[6];
        r = merge_rec_seam(r, B, sm);
        put6(tt.mi + 6 * (mi_off(lg) + ((32 * lane) >> (lg + 1))), sm);
      }
    }
  }
  return r;
}

// Top-down from the tile's outer (L, R): every leaf t < nleaf gets its own (L, R) in (Lo, Ro).
// A merged block's (L, R) sit with its left child's thread; the right child's thread gets them
// by shuffle, and each child evaluates ITS half of the solved seam: the left child its new
// R = y_{m+1}, the right child its new L = y_m (two FMAs each, no reciprocal).  Every thread of
// the CTA must call it.
template <typename T>
__device__ __forceinline__ void tile_tree_down(int nleaf, TileTree<T> &tt, const T (&k0)[3], T L, T R, T &Lo, T &Ro) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  __syncthreads();  // the seams of tile_tree_up are visible
  if (w == 0) {
    const int nw = (nleaf + 31) >> 5;
    T Li = L, Ri = R;  // lane 0's; lanes 1..nw-1 receive theirs below
#pragma unroll
    for (int lg = tile_levels() - 1; lg >= 5; --lg) {
      const int s = 1 << (lg - 5);
      const T pL = __shfl_up_sync(0xffffffffu, Li, s), pR = __shfl_up_sync(0xffffffffu, Ri, s);
      const bool left = (lane & (2 * s - 1)) == 0 && lane + s < nw;
      const bool right = (lane & (2 * s - 1)) == s && lane < nw;
      const T *o = tt.mi + 6 * (mi_off(lg) + ((32 * lane) >> (lg + 1)));
      if (left) Ri = seam_row(o[3], o[4], o[5], Li, Ri);
      if (right) { Li = seam_row(o[0], o[1], o[2], pL, pR); Ri = pR; }
    }
    if (lane < nw) { tt.wext[2 * lane] = Li; tt.wext[2 * lane + 1] = Ri; }
  }
  __syncthreads();
  T Li = tt.wext[2 * w], Ri = tt.wext[2 * w + 1];  // lane 0's; the others receive theirs below
#pragma unroll
  for (int lg = 4; lg >= 0; --lg) {
    const int s = 1 << lg;
    const T pL = __shfl_up_sync(0xffffffffu, Li, s), pR = __shfl_up_sync(0xffffffffu, Ri, s);
    const bool left = (t & (2 * s - 1)) == 0 && t + s < nleaf;
    const bool right = (t & (2 * s - 1)) == s && t < nleaf;
    if (lg > 0) {
      const T *o = tt.mi + 6 * (mi_off(lg) + (t >> (lg + 1)));
      if (left) Ri = seam_row(o[3], o[4], o[5], Li, Ri);
      if (right) { Li = seam_row(o[0], o[1], o[2], pL, pR); Ri = pR; }
    } else {
      if (left) Ri = seam_row(k0[0], k0[1], k0[2], Li, Ri);
      if (right) { Li = seam_row(k0[0], k0[1], k0[2], pL, pR); Ri = pR; }
    }
  }
  Lo = Li;
  Ro = Ri;
}

// X, Y: 256 leaves x R rows each, one pad element per leaf (pad(i) = i + i/R: a warp's 32 leaves
// read their k-th rows from distinct banks); then the tree.
template <typename T, int R> __host__ __device__ constexpr size_t tile_xy_bytes() {
  return sizeof(T) * 2 * (size_t)kTileThreads * (R + 1);
}
template <typename T, int R> __host__ __device__ constexpr size_t tile_smem_bytes() {
  return tile_xy_bytes<T, R>() + sizeof(TileTree<T>);
}

// One leaf (thread l): rows [p, p + rows) of the tile (global P + p ...), the Thomas sweep with three
// right-hand sides (d, a_p e_1, c_q e_q) storing c' in X and g' in Y (their pads) and
// v' in registers, then the backward Horner pass -> the leaf's block record.
// RAG = false: a full leaf (rows == R) -- the curve's first / last row can only be its row 0 /
// R-1, so those two rows take the end-row coefficients by selects and no row carries a bounds
// test; RAG = true: the ragged last leaf of a tile (the general code).  The same operations on
// every row either way, so the same bits.
template <typename T, int R, bool RAG>
__device__ __forceinline__ Rec<T> leaf_sweep(T *X, T *Y, T (&v)[R], int p, int rows, int64_t P, int64_t n, int bc,
                                             T s0, T s1, T xm1, T ym1, T xq1, T yq1, bool &ok) {
  auto pad = [](int i) { return i + i / R; };
  T xi = X[pad(p)], yi = Y[pad(p)];
  T hprev = T(0), ddprev = T(0);
  if (P + p > 0) {
    hprev = xi - xm1;
    ddprev = (yi - ym1) * nr_rcp(hprev);
  }
  T cprev = T(0), gprev = T(0), vprev = T(0);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (!RAG || k < rows) {
      const int i = p + k;
      const int64_t gi = P + i;
      T xn = T(0), yn = T(0), h = T(0), dd = T(0);
      ok = ok && finite(xi) && finite(yi);
      const bool has_next = (RAG || k == R - 1) ? (gi < n - 1) : true;  // rows before R-1 always have one
      if (has_next) {
        if (RAG ? (k < rows - 1) : (k < R - 1)) { xn = X[pad(i + 1)]; yn = Y[pad(i + 1)]; }
        else { xn = xq1; yn = yq1; }
        ok = ok && (xn > xi);
        h = xn - xi;
        dd = (yn - yi) * nr_rcp(h);
      }
      T a, b, cc, d;
      const bool first = (RAG || k == 0) && gi == 0;           // only row 0 of a full leaf can be
      const bool last = (RAG || k == R - 1) && gi == n - 1;    // only row R-1 of a full leaf can be
      if (first) {
        a = T(0);
        if (bc & 1) { b = T(2) * h; cc = h; d = T(6) * (dd - s0); }
        else { b = T(1); cc = T(0); d = T(0); }                       // y2_0 = 0
      } else if (last) {
        cc = T(0);
        if (bc & 2) { a = hprev; b = T(2) * hprev; d = T(6) * (s1 - ddprev); }
        else { a = T(0); b = T(1); d = T(0); }                                   // y2_{n-1} = 0
      } else {  // Eq. init_val
        a = hprev; b = T(2) * (hprev + h); cc = h; d = T(6) * (dd - ddprev);
      }
      const T inv = nr_rcp(k == 0 ? b : b - a * cprev);
      const T cp = cc * inv;
      const T gp = (k == 0 ? d : d - a * gprev) * inv;
      const T vp = (k == 0 ? a : -(a * vprev)) * inv;
      X[pad(i)] = cp;
      Y[pad(i)] = gp;
      v[k] = vp;
      cprev = cp; gprev = gp; vprev = vp;
      xi = xn; yi = yn; hprev = h; ddprev = dd;
    }
  }
  Rec<T> r;
  r.Gq = gprev; r.Vq = vprev; r.Wq = cprev;
  T G = T(0), V = T(0), W = T(-1);  // y_{q+1} = R
#pragma unroll
  for (int k = R - 1; k >= 0; --k) {
    if (!RAG || k < rows) {
      const T ck = X[pad(p + k)], gk = Y[pad(p + k)];
      G = gk - ck * G;
      V = v[k] - ck * V;
      W = -(ck * W);
    }
  }
  r.Gp = G; r.Vp = V; r.Wp = W;
  return r;
}

// The tile this SM slot will most likely run a wave from now (block nb): its x, y into L2, so
// that tile's staging loads (the kernel's largest stall, ncu r02) are L2 hits.  One thread.
template <typename T, int R>
__device__ __forceinline__ void tile_prefetch_l2(const T *x, const T *y, int64_t n, int64_t row_begin, int64_t row_end,
                                                 int ntiles, int64_t nb, int64_t nblocks) {
  if (nb >= nblocks) return;
  const int64_t c2 = nb / ntiles, t2 = nb - c2 * ntiles;
  const int64_t P2 = row_begin + t2 * (int64_t)kTileThreads * R;
  const int64_t r2 = min64((int64_t)kTileThreads * R, row_end - P2);
  constexpr int64_t A = 16 / sizeof(T);
  const int64_t e0 = (c2 * n + P2) & ~(A - 1), e1 = (c2 * n + P2 + r2) & ~(A - 1);
  if (e1 > e0) {
    prefetch_l2_bulk(x + e0, (uint32_t)((e1 - e0) * sizeof(T)));
    prefetch_l2_bulk(y + e0, (uint32_t)((e1 - e0) * sizeof(T)));
  }
}

// One CTA solves rows [P, Q] of one curve: the linear block index is curve c times ntiles plus
// tile t (a 1-D grid, so the batch is not capped at 65535), P = row_begin + t * 256R.
//  FULL   : the tile is the whole curve (row_begin = 0, row_end = n <= 256R); writes y2.
//  REDUCE : writes the tile's block record to tile_rec[(c*ntiles + t)*6].
//  FINISH : reads the tile's outer (L, R) from tile_ext[(c*ntiles + t)*2]; writes y2 rows
//           [P, Q] to y2 + c*(row_end-row_begin) + (P - row_begin).
// tile_solve is the body; on return (FULL / FINISH) the tile's y2 is ALSO in shared memory at
// X[pad(i)] (pad(i) = i + i/R; a warp-staged tile may return per warp: the caller syncs before
// reading other warps' rows), which the fused build+eval kernel
// evaluates from; y2 == nullptr skips the global store (FULL only).
template <typename T, int R, int MODE>
__device__ __forceinline__ void tile_solve(unsigned *__restrict__ status, const T *__restrict__ x,
                                           const T *__restrict__ y, int64_t n, int64_t row_begin, int64_t row_end,
                                           int bc, const T *__restrict__ yp1, const T *__restrict__ ypn,
                                           T *__restrict__ y2, T *__restrict__ tile_rec, const T *__restrict__ tile_ext,
                                           int *__restrict__ badflag, int ntiles, int64_t blk, unsigned char *smem_raw,
                                           int pf_blocks = 0, int64_t nblocks = 0) {
  constexpr int NT = kTileThreads;
  constexpr int TR = NT * R;
  T *X = reinterpret_cast<T *>(smem_raw);
  T *Y = X + NT * (R + 1);
#if FS_TILE_PHASES
  long long tp_ = clock64();
#endif
  TileTree<T> &tt = *reinterpret_cast<TileTree<T> *>(smem_raw + tile_xy_bytes<T, R>());

  const int64_t c = blk / ntiles;
  const int tile = (int)(blk - c * ntiles);
  const int64_t P = row_begin + (int64_t)tile * TR;
  const int nrows = (int)min64(TR, row_end - P);
  const int nleaf = (nrows + R - 1) / R;
  const T *xc = x + c * n;
  const T *yc = y + c * n;
  auto pad = [](int i) { return i + i / R; };

  // coalesced staging with all of a thread's loads in flight before its first store;
  // 16-byte vectors when the tile's rows are 16-byte aligned.  A full, aligned tile is staged
  // PER WARP (kTileWarpStage): warp w loads the rows of its own 32 leaves and goes on to their
  // sweeps after a __syncwarp -- no CTA barrier until the merge tree, so the warps of a tile
  // overlap their loads with one another's arithmetic.
  constexpr int VW = 16 / sizeof(T);
  using VT = typename Vec16<T>::V;
  const bool vec = ((((uintptr_t)(xc + P)) | ((uintptr_t)(yc + P))) & 15) == 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool wstage = kTileWarpStage && vec && nrows == TR;
  if (wstage) {
    constexpr int WR = 32 * R;  // rows of a warp's leaves
    const int r0 = wid * WR;
#pragma unroll kTileStageUnroll
    for (int v = lane; v < WR / VW; v += 32) {
      const VT a = __ldcs(reinterpret_cast<const VT *>(xc + P + r0) + v);
      const VT b = __ldcs(reinterpret_cast<const VT *>(yc + P + r0) + v);
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        X[pad(r0 + v * VW + i)] = reinterpret_cast<const T *>(&a)[i];
        Y[pad(r0 + v * VW + i)] = reinterpret_cast<const T *>(&b)[i];
      }
    }
    __syncwarp();
  } else {
    const int nvec = vec ? nrows / VW : 0;
#pragma unroll kTileStageUnroll
    for (int v = threadIdx.x; v < nvec; v += NT) {
      const VT a = __ldcs(reinterpret_cast<const VT *>(xc + P) + v);
      const VT b = __ldcs(reinterpret_cast<const VT *>(yc + P) + v);
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        X[pad(v * VW + i)] = reinterpret_cast<const T *>(&a)[i];
        Y[pad(v * VW + i)] = reinterpret_cast<const T *>(&b)[i];
      }
    }
#pragma unroll 8
    for (int e = nvec * VW + threadIdx.x; e < nrows; e += NT) {
      X[pad(e)] = ld_stream(xc + P + e);
      Y[pad(e)] = ld_stream(yc + P + e);
    }
    __syncthreads();
  }
  TILE_MARK(0);
  // (FS_TILE_PF_LATE) the next wave's tile is prefetched once this tile's own loads are done, so
  // the two do not compete for DRAM at the start of a wave
  if (pf_blocks > 0 && threadIdx.x == 0) tile_prefetch_l2<T, R>(x, y, n, row_begin, row_end, ntiles, blk + pf_blocks, nblocks);

  const int l = threadIdx.x;
  const int p = l * R;
  const int rows = min(R, nrows - p);
  T v[R];
  bool ok = true;
  T xm1 = T(0), ym1 = T(0), xq1 = T(0), yq1 = T(0);
  if (l < nleaf) {
    if (l == 0) {
      if (P > 0) { xm1 = xc[P - 1]; ym1 = yc[P - 1]; }
    } else if (wstage && lane == 0) {  // the previous warp's last row: from global memory (L2)
      xm1 = xc[P + p - 1];
      ym1 = yc[P + p - 1];
    } else {
      xm1 = X[pad(p - 1)];
      ym1 = Y[pad(p - 1)];
    }
    const int q = p + rows - 1;
    if (l == nleaf - 1) {
      if (P + q + 1 < n) { xq1 = xc[P + q + 1]; yq1 = yc[P + q + 1]; }
    } else if (wstage && lane == 31) {  // the next warp's first row
      xq1 = xc[P + q + 1];
      yq1 = yc[P + q + 1];
    } else {
      xq1 = X[pad(q + 1)];
      yq1 = Y[pad(q + 1)];
    }
  }
  // every neighbour value is in registers before the sweeps overwrite X/Y (per warp: a warp's
  // sweeps touch only its own rows when it staged them itself)
  if (wstage) __syncwarp();
  else __syncthreads();
  TILE_MARK(1);

  Rec<T> r{T(0), T(0), T(0), T(0), T(0), T(0)};
  if (l < nleaf) {
    const T s0 = (bc & 1) ? yp1[c] : T(0);
    const T s1 = (bc & 2) ? ypn[c] : T(0);
    if (bc & 1) ok = ok && finite(s0);
    if (bc & 2) ok = ok && finite(s1);
    // full leaves (all but a ragged last one) run without per-row bounds tests (leaf_sweep)
    r = rows == R ? leaf_sweep<T, R, false>(X, Y, v, p, rows, P, n, bc, s0, s1, xm1, ym1, xq1, yq1, ok)
                  : leaf_sweep<T, R, true>(X, Y, v, p, rows, P, n, bc, s0, s1, xm1, ym1, xq1, yq1, ok);
  }
  TILE_MARK(2);
  T k0[3];
  bool bad;
  r = tile_tree_up(r, nleaf, tt, k0, !ok, bad);
  TILE_MARK(3);

  if (MODE == TILE_REDUCE) {
    if (threadIdx.x == 0) {
      T *o = tile_rec + (c * ntiles + tile) * 6;
      o[0] = r.Gp; o[1] = r.Vp; o[2] = r.Wp; o[3] = r.Gq; o[4] = r.Vq; o[5] = r.Wq;
      if (bad) {  // a NaN record: every merge and every finish that uses it is NaN (the whole curve)
        for (int k = 0; k < 6; ++k) o[k] = qnan<T>();
        atomicOr(badflag + c, 1);
        raise_status(status, kBadKnots);
      }
    }
    return;
  }

  T *y2o = !y2 ? nullptr : (MODE == TILE_FULL) ? y2 + c * n + P : y2 + c * (row_end - row_begin) + (P - row_begin);
  const bool curve_bad = (MODE == TILE_FULL) ? bad : (badflag[c] != 0);
  if (curve_bad) {
    if (MODE == TILE_FULL && threadIdx.x == 0) raise_status(status, kBadKnots);
    for (int e = threadIdx.x; e < nrows; e += NT) {
      X[pad(e)] = qnan<T>();
      if (y2o) y2o[e] = qnan<T>();
    }
    __syncthreads();
    return;
  }
  T Lr = T(0), Rr = T(0);
  if (MODE == TILE_FINISH) {
    Lr = tile_ext[(c * ntiles + tile) * 2];
    Rr = tile_ext[(c * ntiles + tile) * 2 + 1];
  }
  T L, ynext;
  tile_tree_down(nleaf, tt, k0, Lr, Rr, L, ynext);
  TILE_MARK(4);
  if (l < nleaf) {
    if (rows == R) {
#pragma unroll
      for (int k = R - 1; k >= 0; --k) {
        const int i = p + k;
        const T yv = Y[pad(i)] - v[k] * L - X[pad(i)] * ynext;  // y_i = g'_i - v'_i L - c'_i y_{i+1}
        X[pad(i)] = yv;
        ynext = yv;
      }
    } else {
#pragma unroll
      for (int k = R - 1; k >= 0; --k) {
        if (k < rows) {
          const int i = p + k;
          const T yv = Y[pad(i)] - v[k] * L - X[pad(i)] * ynext;
          X[pad(i)] = yv;
          ynext = yv;
        }
      }
    }
  }
  const bool vo = y2o && (((uintptr_t)y2o) & 15) == 0;
  if (wstage && vo) {  // each warp stores its own leaves' rows (no CTA barrier)
    __syncwarp();
    TILE_MARK(5);
    constexpr int WR = 32 * R;
    const int r0 = wid * WR;
    for (int v = lane; v < WR / VW; v += 32) {
      VT a;
#pragma unroll
      for (int i = 0; i < VW; ++i) reinterpret_cast<T *>(&a)[i] = X[pad(r0 + v * VW + i)];
      __stcs(reinterpret_cast<VT *>(y2o + r0) + v, a);
    }
    TILE_MARK(6);
    return;  // (the tile's y2 is in X; a caller that reads other warps' rows syncs first)
  }
  __syncthreads();
  TILE_MARK(5);
  if (!y2o) return;
  const int novec = vo ? nrows / VW : 0;
  for (int v = threadIdx.x; v < novec; v += NT) {
    VT a;
#pragma unroll
    for (int i = 0; i < VW; ++i) reinterpret_cast<T *>(&a)[i] = X[pad(v * VW + i)];
    __stcs(reinterpret_cast<VT *>(y2o) + v, a);
  }
  for (int e = novec * VW + threadIdx.x; e < nrows; e += NT) y2o[e] = X[pad(e)];
  TILE_MARK(6);
}

template <typename T, int R, int MODE>
__global__ void __launch_bounds__(kTileThreads, FS_TILE_MINB) k_tile(unsigned *__restrict__ status, const T *__restrict__ x,
                                                      const T *__restrict__ y, int64_t n, int64_t row_begin,
                                                      int64_t row_end, int bc, const T *__restrict__ yp1,
                                                      const T *__restrict__ ypn, T *__restrict__ y2,
                                                      T *__restrict__ tile_rec, const T *__restrict__ tile_ext,
                                                      int *__restrict__ badflag, int ntiles, int pf_blocks) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  pdl_wait();  // (programmatic launch after K4: its (L, R) per tile; x, y from any earlier kernel)
  // K5 (FINISH) walks the tiles last to first: K3 just read them first to last, so the L2 still
  // holds the last tiles' x, y when K5 starts
  const int64_t nbk = gridDim.x;
  auto logical = [&](int64_t b) { return (MODE == TILE_FINISH && kTileFinishReverse) ? nbk - 1 - b : b; };
  if (!kTilePrefetchLate && pf_blocks > 0 && threadIdx.x == 0 && (int64_t)blockIdx.x + pf_blocks < nbk)
    tile_prefetch_l2<T, R>(x, y, n, row_begin, row_end, ntiles, logical((int64_t)blockIdx.x + pf_blocks), nbk);
  tile_solve<T, R, MODE>(status, x, y, n, row_begin, row_end, bc, yp1, ypn, y2, tile_rec, tile_ext, badflag, ntiles,
                         logical((int64_t)blockIdx.x), smem_raw, kTilePrefetchLate ? pf_blocks : 0, nbk);
}

// K4: merge the per-tile records of each curve (grid = batch, one CTA per curve) and,
// unless up_only, push the root's outer (L, R) back down to per-tile (L, R).
// Each of the kTopThreads threads folds a contiguous chunk of tiles sequentially
// (saving the running q-tips in foldq for the way down), then a shared-memory tree
// merges the chunk records.
constexpr int kTopThreads = 512;
template <typename T> __host__ __device__ constexpr size_t top_smem_bytes() {
  return sizeof(T) * (6 * kTopThreads + 6 * kTopThreads);
}

// Group c of the launch covers records [c ntiles, min((c+1) ntiles, ntot)) of the arrays (ntot <= 0:
// every group has ntiles records -- one group per curve); so one long curve's tile records can
// be merged by many CTAs (groups), their group records by one, and pushed back down by many.
template <typename T>
__global__ void __launch_bounds__(kTopThreads) k4_top(const T *__restrict__ recs, int ntiles, int up_only,
                                                      const T *__restrict__ root_ext, T *__restrict__ tile_ext,
                                                      T *__restrict__ root_out, T *__restrict__ foldq,
                                                      int64_t ntot) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  pdl_trigger();  // the next kernel (K4's next phase, K5) may be launched now; it waits for this one
  pdl_wait();     // the records of the previous kernel (programmatic launch)
  Rec<T> *rec = reinterpret_cast<Rec<T> *>(smem_raw);
  T *mi = reinterpret_cast<T *>(rec + kTopThreads);
  T *ext = reinterpret_cast<T *>(rec);
  const int64_t c = blockIdx.x;
  const T *rc = recs + c * ntiles * 6;
  T *fq = foldq + c * ntiles * 3;
  T *te = tile_ext + c * ntiles * 2;
  if (ntot > 0) ntiles = (int)min64(ntiles, ntot - c * ntiles);
  const int chunk = (ntiles + kTopThreads - 1) / kTopThreads;
  const int nleaf = (ntiles + chunk - 1) / chunk;
  const int th = threadIdx.x;
  const int first = th * chunk;
  const int last = min(ntiles, first + chunk) - 1;
  auto load = [&](int t) {
    Rec<T> r;
    r.Gp = rc[6 * t]; r.Vp = rc[6 * t + 1]; r.Wp = rc[6 * t + 2];
    r.Gq = rc[6 * t + 3]; r.Vq = rc[6 * t + 4]; r.Wq = rc[6 * t + 5];
    return r;
  };
  if (th < nleaf) {
    Rec<T> acc = load(first);
    for (int t = first + 1; t <= last; ++t) {
      fq[3 * t] = acc.Gq; fq[3 * t + 1] = acc.Vq; fq[3 * t + 2] = acc.Wq;
      acc = merge_rec(acc, load(t));
    }
    rec[th] = acc;
  }
  __syncthreads();
  tree_up(rec, mi, nleaf);
  if (up_only) {
    if (th == 0) {
      const Rec<T> r = rec[0];
      T *o = root_out + c * 6;
      o[0] = r.Gp; o[1] = r.Vp; o[2] = r.Wp; o[3] = r.Gq; o[4] = r.Vq; o[5] = r.Wq;
    }
    return;
  }
  const T L0 = root_ext ? root_ext[2 * c] : T(0);
  const T R0 = root_ext ? root_ext[2 * c + 1] : T(0);
  tree_down(mi, ext, nleaf, L0, R0);
  if (th < nleaf) {
    const T L = ext[2 * th];
    T Rv = ext[2 * th + 1];
    for (int t = last; t > first; --t) {
      const Rec<T> B = load(t);
      T ym, ym1;
      split_seam(fq[3 * t], fq[3 * t + 1], fq[3 * t + 2], B.Gp, B.Vp, B.Wp, L, Rv, ym, ym1);
      te[2 * t] = ym;
      te[2 * t + 1] = Rv;
      Rv = ym1;
    }
    te[2 * first] = L;
    te[2 * first + 1] = Rv;
  }
}

}  // namespace fs
