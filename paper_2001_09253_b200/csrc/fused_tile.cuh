// fused_tile.cuh -- spline_build_eval for mid-length curves with sorted queries (BASELINE cfg4):
// the curve's build and its evaluation in ONE kernel, the second derivatives never leaving the chip
// on their way from the solve to the evaluation (the paper evaluates right
// after the build).
//
// k_tile_eval: CTA (c, chunk) first solves curve c exactly as K2 does (tile_solve<FULL>: leaf
// Thomas sweeps, merged by the block-record tree; the paper's back-substitution,
// P:1116-1122), which leaves y2 in shared memory; chunk 0 also stores it to HBM when the caller
// asked for y2.  Its 8 warps then walk the chunk's queries as sorted runs (sorted_run: the
// carried bracket of P:1505-1509 and the per-warp record window), reading x, y through L1/L2
// (just staged by the solve: L2-hot) and y2 from shared memory.  So per curve HBM sees x and y
// read once, y2 written once and the queries streamed -- against the split path's x, y read
// twice and y2 written then read back -- and the latency-bound solve of one CTA overlaps the
// streaming evaluation of the other CTA on its SM.  Results are bitwise the split path's: the
// same tile_solve arithmetic and the same sorted_run.
#pragma once
#include "build_tile.cuh"
#include "eval.cuh"

namespace fs {

constexpr int kTileEvalWarps = kTileThreads / 32;
#ifndef FS_TILE_EVAL_PF
#define FS_TILE_EVAL_PF 1
#endif
constexpr int kTileEvalPF = FS_TILE_EVAL_PF;  // query prefetch depth (warp steps) of the eval phase

// The warps' record windows reuse the solve's Y rows (the g' values, dead once tile_solve has
// returned: it ends with a barrier after the back-substitution), so the fused kernel needs no
// more shared memory than the solve.
template <typename T, int R> __host__ __device__ constexpr size_t tile_eval_win_offset() {
  return sizeof(T) * (size_t)kTileThreads * (R + 1);
}
template <typename T, int R> __host__ __device__ constexpr size_t tile_eval_smem_bytes() {
  return tile_smem_bytes<T, R>() > tile_eval_win_offset<T, R>() + kTileEvalWarps * sizeof(SortWin<T>)
             ? tile_smem_bytes<T, R>()
             : tile_eval_win_offset<T, R>() + kTileEvalWarps * sizeof(SortWin<T>);
}

#ifndef FS_TILE_EVAL_MINB
#define FS_TILE_EVAL_MINB 3  // cfg4 PATH_FUSED: 1374 vs 1614 us at 2 (the split path: 1225-1233 us)
#endif
template <typename T, int R, int V, bool WIN>
__global__ void __launch_bounds__(kTileThreads, FS_TILE_EVAL_MINB)
    k_tile_eval(unsigned *__restrict__ status, const T *__restrict__ x, const T *__restrict__ y, int n, int bc,
                const T *__restrict__ yp1, const T *__restrict__ ypn, T *__restrict__ y2, const T *__restrict__ q,
                int64_t m, T *__restrict__ out, int32_t *__restrict__ idx, int nchunks, int64_t qchunk) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t c = blockIdx.x / nchunks;
  const int chunk = (int)(blockIdx.x - c * nchunks);
  // the solve (chunk 0 writes y2 when asked; every chunk keeps its own copy on chip)
  tile_solve<T, R, TILE_FULL>(status, x, y, n, 0, n, bc, yp1, ypn, chunk == 0 ? y2 : nullptr, nullptr, nullptr,
                              nullptr, 1, c, smem_raw);
  __syncthreads();  // every warp's rows of y2 are in shared memory (tile_solve may end per warp)
  const T *Zs = reinterpret_cast<const T *>(smem_raw);  // y2, padded rows (tile_solve)
  SortWin<T> *wins = reinterpret_cast<SortWin<T> *>(smem_raw + tile_eval_win_offset<T, R>());
  // the chunk's queries, one contiguous run per warp (whole 32V steps)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q0 = chunk * qchunk, q1 = min64(m, q0 + qchunk);
  int64_t per = (q1 - q0 + kTileEvalWarps - 1) / kTileEvalWarps;
  per = (per + 32 * V - 1) / (32 * V) * (32 * V);
  const int64_t k0 = q0 + w * per, k1 = min64(q1, k0 + per);
  bool oor = false;
  if (k0 < k1) {
    if constexpr (WIN && kSortedSearchForm)
      oor = sorted_run_win<T, V, kTileEvalPF>(x + c * n, y + c * n, ZShared<T, R>{Zs}, n, q + c * m, out + c * m,
                                              idx ? idx + c * m : nullptr, k0, k1, wins[w], lane);
    else
      oor = sorted_run<T, V, FORM_RECORD, WIN, kTileEvalPF>(x + c * n, y + c * n, ZShared<T, R>{Zs}, n, q + c * m,
                                                              out + c * m, idx ? idx + c * m : nullptr, k0, k1,
                                                              wins[w], lane);
  }
  raise_status_warp(status, oor, kOutOfRange);
}

}  // namespace fs
