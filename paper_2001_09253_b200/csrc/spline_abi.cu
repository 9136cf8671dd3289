// spline_abi.cu -- the C ABI of include/spline.h: argument checks, kernel dispatch, launches.
//
// Dispatch (build, by n and dtype):
//   n <= 8                        K1r k1_thomas_regs     one thread per curve, registers
//   n = 16 (f32: 32, 64)          K1h k1_thomas_half     two threads per curve, half curves in registers
//   n <= 128                      K1 k1_thomas_pipe      two threads per curve, sweep from both ends
//   n <= 256*RMAX (4096 f64,      K2 k_tile<FULL>        one CTA per curve: 256 leaves x R rows,
//                  8192 f32)                              merge tree in shared memory
//   longer                        K3 k_tile<REDUCE> -> K4 k4_top -> K5 k_tile<FINISH>   (tiled SPIKE)
// Dispatch (eval):
//   SPLINE_Q_SORTED               k_eval_sorted          carried bracket + per-warp record window
//   fp32 n <= 8, m <= 32          k_eval_small           a warp per 32 curves, records in registers
//   n <= 64, many curves          k_eval_curvewarp       a warp per curve, Eytzinger keys
//   fits shared memory            k_eval_warps / k_eval_staged   TMA-staged curves (BISECT, TABLE,
//                                                          UNIFORM, BSEARCH)
//   one curve >> L2, many queries k_bucket_*             queries bucketed by L2-sized chunks
//   otherwise                     k_pack_records + k_eval_records   one record gather per query
// spline_build_eval: k_build_eval_tiny (few curves) | k_eval_small<true> | k_build_eval_warp
// (many K1h-sized curves) | k_fused_staged | k_tile_eval (on SPLINE_PATH_FUSED) | the two above
// back to back.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "../../include/spline.h"
#include "build_thomas.cuh"
#include "build_tile.cuh"
#include "common.cuh"
#include "eval.cuh"
#include "eval_bucket.cuh"
#include "fused.cuh"
#include "fused_tile.cuh"

using namespace fs;

namespace {

constexpr int kK1MaxN = 128;
// spline_build_eval's automatic choice: the fused warp-specialised kernel only for
// launch-latency-sized problems (measured with spline_build_eval on scaled configs, round 1: K1h + curvewarp win from ~2^18)
constexpr int64_t kFuseMaxWork = int64_t(1) << 17;
#ifndef FS_BUILD_EVAL_WARP
#define FS_BUILD_EVAL_WARP 1
#endif
constexpr bool kBuildEvalWarp = FS_BUILD_EVAL_WARP != 0;  // spline_build_eval: k_build_eval_warp for many K1h-sized curves
constexpr int kNoFusedStaged = 1 << 30;  // internal: automatic path, but not k_fused_staged
constexpr int kEvalNoBucket = SPLINE_NO_BUCKET;  // spline_eval: the record-gather path for long curves
#ifndef FS_TOP_PDL
#define FS_TOP_PDL 1
#endif
constexpr bool kTopPdl = FS_TOP_PDL != 0;  // K4's phases and K5 launched programmatically (launch latency hidden)
#ifndef FS_BK_BAND
#define FS_BK_BAND 1
#endif
constexpr bool kBkBand = FS_BK_BAND != 0;  // bucketed eval: the neighbour knot only near a cell boundary
#ifndef FS_SPLIT_OVERLAP
#define FS_SPLIT_OVERLAP 0  // A/B: 1358 vs 1283 us on cfg4 -- the concurrent build slows the evaluation more
#endif
constexpr bool kSplitOverlap = FS_SPLIT_OVERLAP != 0;  // build half B while half A is evaluated

template <typename T> constexpr int rmax() { return sizeof(T) == 8 ? 16 : 32; }

inline int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return SPLINE_OK;
  if (e == cudaErrorMemoryAllocation) return SPLINE_ENOMEM;
  return SPLINE_ECUDA;
}

template <typename K> int set_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return SPLINE_OK;
  return cuda_rc(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

inline int launch_rc() { return cuda_rc(cudaGetLastError()); }

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while the
// previous kernel of the stream is finishing; it must pdl_wait() before reading its inputs.
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_rc(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// Stream-ordered scratch (SPIKE tile records; y2 for an unfused spline_build_eval without y2)
// from a library-owned pool per device that keeps its memory between calls (release
// threshold = max), so repeated calls do not map and unmap device memory.
inline int ws_alloc(void **p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[128] = {};
  int dev = 0;
  if (int rc = cuda_rc(cudaGetDevice(&dev))) return rc;
  if (dev < 0 || dev >= 128) return SPLINE_ECUDA;
  {
    std::lock_guard<std::mutex> g(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      if (int rc = cuda_rc(cudaMemPoolCreate(&pools[dev], &props))) return rc;
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return cuda_rc(cudaMallocFromPoolAsync(p, bytes, pools[dev], st));
}
// Per-stream data-error words (spline_status).  Each device has a slab of kStatusSlots words;
// a stream handle is given its own slot the first time it is seen (slot 0 is the shared
// overflow slot once all are taken).  Every kernel receives its launching call's word, so bits
// raised on one stream are read and cleared by spline_status on that stream only.
constexpr int kStatusSlots = 4096;
struct StatusSlab {
  unsigned *words = nullptr;
  std::unordered_map<uintptr_t, int> slot;
  int next = 1;
};
inline unsigned *status_word(cudaStream_t st) {
  static std::mutex mu;
  static StatusSlab slabs[128];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 128) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  StatusSlab &s = slabs[dev];
  if (!s.words) {
    unsigned *w = nullptr;
    if (cudaMalloc(&w, sizeof(unsigned) * kStatusSlots) != cudaSuccess) return nullptr;
    if (cudaMemset(w, 0, sizeof(unsigned) * kStatusSlots) != cudaSuccess) return nullptr;
    s.words = w;
  }
  const uintptr_t key = (uintptr_t)st;
  auto it = s.slot.find(key);
  int k = 0;
  if (it != s.slot.end()) k = it->second;
  else if (s.next < kStatusSlots) s.slot.emplace(key, k = s.next++);
  return s.words + k;
}
// The word of the API call being enqueued on this host thread (set by StatusScope in every
// entry point; the launch helpers below pass it to their kernels).
thread_local unsigned *tl_status = nullptr;
struct StatusScope {
  unsigned *prev;
  explicit StatusScope(cudaStream_t st) : prev(tl_status) { tl_status = status_word(st); }
  ~StatusScope() { tl_status = prev; }
  bool ok() const { return tl_status != nullptr; }
};

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }
inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}



// Shared-knot mode (SPLINE_X_SHARED): kernels without a native knot-row stride get the knot
// vector broadcast into stream-ordered scratch ([batch][n]) first; results are bitwise the
// per-curve-x call's (the kernels see the same values).
template <typename T> int broadcast_x(const T *x, int64_t n, int64_t batch, cudaStream_t st, T **out) {
  if (int rc = ws_alloc((void **)out, sizeof(T) * (size_t)n * batch, st)) return rc;
  const int64_t total = n * batch;
  const int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  k_broadcast_rows<T><<<(unsigned)grid, 256, 0, st>>>(x, n, total, *out);
  return launch_rc();
}

// Internal streams and per-call events (the host path; the overlapped split path)
constexpr int kHostStreams = 3;
constexpr size_t kHostChunkBytes = 32u << 20;  // target copy traffic per chunk

struct HostStreams {
  cudaStream_t s[kHostStreams];
};
inline int host_streams(HostStreams **out) {
  static std::mutex mu;
  static HostStreams *per_dev[128] = {};
  int dev = 0;
  if (int rc = cuda_rc(cudaGetDevice(&dev))) return rc;
  if (dev < 0 || dev >= 128) return SPLINE_ECUDA;
  std::lock_guard<std::mutex> lk(mu);
  if (!per_dev[dev]) {
    auto *h = new HostStreams;
    for (int i = 0; i < kHostStreams; ++i)
      if (int rc = cuda_rc(cudaStreamCreateWithFlags(&h->s[i], cudaStreamNonBlocking))) return rc;
    per_dev[dev] = h;
  }
  *out = per_dev[dev];
  return SPLINE_OK;
}
// The events of ONE host call (never shared between calls, so concurrent calls from several
// threads cannot re-record each other's start/done points).  Destroyed at the end of the call:
// CUDA releases an event still pending on the device once it completes.
struct CallEvents {
  cudaEvent_t start = nullptr, ready = nullptr, done[kHostStreams] = {};
  int init() {
    int rc = cuda_rc(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    if (!rc) rc = cuda_rc(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    for (int k = 0; !rc && k < kHostStreams; ++k) rc = cuda_rc(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
    return rc;
  }
  ~CallEvents() {
    if (start) cudaEventDestroy(start);
    if (ready) cudaEventDestroy(ready);
    for (int k = 0; k < kHostStreams; ++k)
      if (done[k]) cudaEventDestroy(done[k]);
  }
};
// Device bytes one chunk slot may take (3 slots in flight): caps the curves per chunk for very
// long curves / many queries, whatever the SM floor asks for.
constexpr size_t kMaxSlotBytes = size_t(4) << 30;

// ------------------------------------------------------------------------ build

// k_tile's L2 prefetch distance: the CTAs resident at once (one wave ahead), 0 = off
template <typename K> int tile_prefetch_blocks(K kern, size_t sm) {
  if (kTilePrefetchAhead <= 0) return 0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTileThreads, sm) != cudaSuccess || occ < 1) occ = 1;
  return kTilePrefetchAhead * occ * num_sms();
}

template <typename T, int R>
int launch_tile_full(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                     cudaStream_t st) {
  auto kern = k_tile<T, R, TILE_FULL>;
  const size_t sm = tile_smem_bytes<T, R>();
  if (int rc = set_smem(kern, sm)) return rc;
  kern<<<(unsigned)batch, kTileThreads, sm, st>>>(tl_status, x, y, n, 0, n, bc, yp1, ypn, y2, nullptr, nullptr, nullptr, 1,
                                                  tile_prefetch_blocks(kern, sm));
  return launch_rc();
}

template <typename T>
int build_mid(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
              cudaStream_t st) {
  if (n <= 256 * 1) return launch_tile_full<T, 1>(x, y, n, batch, bc, yp1, ypn, y2, st);
  if (n <= 256 * 2) return launch_tile_full<T, 2>(x, y, n, batch, bc, yp1, ypn, y2, st);
  if (n <= 256 * 4) return launch_tile_full<T, 4>(x, y, n, batch, bc, yp1, ypn, y2, st);
  if (n <= 256 * 8) return launch_tile_full<T, 8>(x, y, n, batch, bc, yp1, ypn, y2, st);
  if (n <= 256 * 16) return launch_tile_full<T, 16>(x, y, n, batch, bc, yp1, ypn, y2, st);
  if constexpr (rmax<T>() >= 32) {
    if (n <= 256 * 32) return launch_tile_full<T, 32>(x, y, n, batch, bc, yp1, ypn, y2, st);
  }
  return SPLINE_EINVAL;
}

struct SpikeWs {
  void *tile_rec, *tile_ext, *foldq, *badflag, *rank_ext, *rank_foldq, *grp_rec;
};
constexpr int kMaxRanks = 1024;

template <typename T> size_t spike_ws_layout(int64_t ntiles, int64_t batch, SpikeWs *ws, char *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void *p = base ? base + off : nullptr;
    off += (bytes + 255) & ~(size_t)255;
    return p;
  };
  SpikeWs w;
  w.tile_rec = take(sizeof(T) * 6 * ntiles * batch);
  w.tile_ext = take(sizeof(T) * 2 * ntiles * batch);
  w.foldq = take(sizeof(T) * 3 * ntiles * batch);
  w.badflag = take(sizeof(int) * batch);
  w.rank_ext = take(sizeof(T) * 2 * kMaxRanks);
  w.rank_foldq = take(sizeof(T) * 3 * kMaxRanks);
  w.grp_rec = take(sizeof(T) * 6 * kMaxRanks);
  if (ws) *ws = w;
  return off;
}

template <typename T> int launch_top(const T *recs, int ntiles, int64_t batch, int up_only, const T *root_ext,
                                     T *tile_ext, T *root_out, T *foldq, cudaStream_t st, int64_t ntot = 0) {
  auto kern = k4_top<T>;
  const size_t sm = top_smem_bytes<T>();
  if (int rc = set_smem(kern, sm)) return rc;
  if (kTopPdl) return launch_pdl(kern, dim3((unsigned)batch), dim3(kTopThreads), sm, st, recs, ntiles, up_only, root_ext,
                                 tile_ext, root_out, foldq, ntot);
  kern<<<(unsigned)batch, kTopThreads, sm, st>>>(recs, ntiles, up_only, root_ext, tile_ext, root_out, foldq, ntot);
  return launch_rc();
}

// K4 for ONE long curve with many tiles: groups of kGroupTiles tiles are merged by one CTA each
// (up), the group records by one CTA (up + down), and the outer values pushed back down the
// groups (down) -- instead of one CTA folding every tile record.
constexpr int kGroupTiles = 64;
template <typename T>
int launch_top_grouped(const T *recs, int ntiles, const SpikeWs &w, cudaStream_t st) {
  const int G = (ntiles + kGroupTiles - 1) / kGroupTiles;
  T *grp = (T *)w.grp_rec, *gext = (T *)w.rank_ext, *gfq = (T *)w.rank_foldq;
  int rc = launch_top<T>(recs, kGroupTiles, G, 1, nullptr, nullptr, grp, (T *)w.foldq, st, ntiles);
  if (!rc) rc = launch_top<T>(grp, G, 1, 0, nullptr, gext, nullptr, gfq, st);
  if (!rc) rc = launch_top<T>(recs, kGroupTiles, G, 0, gext, (T *)w.tile_ext, nullptr, (T *)w.foldq, st, ntiles);
  return rc;
}

template <typename T, int MODE>
int launch_tile_part(const T *x, const T *y, int64_t n, int64_t rb, int64_t re, int64_t batch, int bc, const T *yp1,
                     const T *ypn, T *y2, const SpikeWs &w, cudaStream_t st) {
  constexpr int R = rmax<T>();
  const int64_t ntiles = (re - rb + 256 * R - 1) / (256 * R);
  auto kern = k_tile<T, R, MODE>;
  const size_t sm = tile_smem_bytes<T, R>();
  if (int rc = set_smem(kern, sm)) return rc;
  if (ntiles * batch >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  if (kTopPdl && MODE == TILE_FINISH)  // K5 after K4 (which triggers at its start): programmatic launch
    return launch_pdl(kern, dim3((unsigned)(ntiles * batch)), dim3(kTileThreads), sm, st, tl_status, x, y, n, rb, re, bc,
                      yp1, ypn, y2, (T *)w.tile_rec, (const T *)w.tile_ext, (int *)w.badflag, (int)ntiles,
                      tile_prefetch_blocks(kern, sm));
  kern<<<(unsigned)(ntiles * batch), kTileThreads, sm, st>>>(tl_status, x, y, n, rb, re, bc, yp1, ypn, y2, (T *)w.tile_rec,
                                                             (const T *)w.tile_ext, (int *)w.badflag, (int)ntiles,
                                                             tile_prefetch_blocks(kern, sm));
  return launch_rc();
}

template <typename T>
int build_long(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
               cudaStream_t st) {
  constexpr int R = rmax<T>();
  const int64_t ntiles = (n + 256 * R - 1) / (256 * R);
  const size_t bytes = spike_ws_layout<T>(ntiles, batch, nullptr, nullptr);
  void *base = nullptr;
  if (int rc = ws_alloc(&base, bytes, st)) return rc;
  SpikeWs w;
  spike_ws_layout<T>(ntiles, batch, &w, (char *)base);
  int rc = cuda_rc(cudaMemsetAsync(w.badflag, 0, sizeof(int) * batch, st));
  if (!rc) rc = launch_tile_part<T, TILE_REDUCE>(x, y, n, 0, n, batch, bc, yp1, ypn, y2, w, st);
  if (!rc) {
    if (batch == 1 && ntiles > 2 * kGroupTiles && (ntiles + kGroupTiles - 1) / kGroupTiles <= kMaxRanks)
      rc = launch_top_grouped<T>((const T *)w.tile_rec, (int)ntiles, w, st);
    else
      rc = launch_top<T>((const T *)w.tile_rec, (int)ntiles, batch, 0, nullptr, (T *)w.tile_ext, nullptr,
                         (T *)w.foldq, st);
  }
  if (!rc) rc = launch_tile_part<T, TILE_FINISH>(x, y, n, 0, n, batch, bc, yp1, ypn, y2, w, st);
  cudaFreeAsync(base, st);
  return rc;
}

template <typename T>
int build_t(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
            cudaStream_t st, bool xshared = false) {
  if (n <= kRegsNMax) {  // K1r: registers only (the fused kernel's SOLVE_REGS takes the same n)
    constexpr int VW = 16 / sizeof(T);
    const int vec = (n % VW == 0) && aligned16(x) && aligned16(y) && aligned16(y2);
    const int64_t grid = (batch + 255) / 256;
    k1_thomas_regs<T, kRegsNMax><<<(unsigned)grid, 256, 0, st>>>(tl_status, x, y, (int)n, batch, bc, yp1, ypn, y2, vec,
                                                                 xshared ? (int64_t)0 : n);
    return launch_rc();
  }
  if (xshared && batch > 1) {  // no native knot-row stride: broadcast the knot vector first
    T *xb = nullptr;
    int rc = broadcast_x<T>(x, n, batch, st, &xb);
    if (!rc) rc = build_t<T>(xb, y, n, batch, bc, yp1, ypn, y2, st, false);
    if (xb) cudaFreeAsync(xb, st);
    return rc;
  }
  if (n <= kK1MaxN) {  // K1: two threads per curve, staged odd-stride tiles
    // K1h: the same sweep with each half curve in registers (16-byte-aligned rows)
    // (fp32 n = 16, 32, 64; fp64 n = 16: 2n values per thread stay within ~90 registers)
    if (aligned16(x) && aligned16(y) && aligned16(y2)) {
      const unsigned grid = (unsigned)((2 * batch + kK1hThreads - 1) / kK1hThreads);
      if constexpr (sizeof(T) == 4) {
        if (n == 64 || n == 32) {
          if (n == 64) k1_thomas_half<T, 64><<<grid, kK1hThreads, 0, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2);
          else k1_thomas_half<T, 32><<<grid, kK1hThreads, 0, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2);
          return launch_rc();
        }
      }
      if (n == 16) {
        k1_thomas_half<T, 16><<<grid, kK1hThreads, 0, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2);
        return launch_rc();
      }
    }
    const int S = babe_stride((int)n);
    if ((n * sizeof(T)) % 16 == 0 && aligned16(x) && aligned16(y)) {
      // persistent + TMA-pipelined; CPB curves per tile (2 threads each)
      int cpb = 64;
      const auto smem_of = [&](int c) {
        return 16 + ((2 * (size_t)c * n * sizeof(T) + 15) & ~(size_t)15) + 2 * (size_t)(c + 1) * S * sizeof(T);
      };
      while (cpb > 16 && smem_of(cpb) > 64 * 1024) cpb -= 16;
      const size_t sm = smem_of(cpb);
      auto kern = k1_thomas_pipe<T>;
      if (int rc = set_smem(kern, sm)) return rc;
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 2 * cpb, sm) != cudaSuccess || occ < 1) occ = 1;
      const int64_t ntiles = (batch + cpb - 1) / cpb;
      const int64_t grid = std::min<int64_t>(ntiles, (int64_t)occ * num_sms());
      kern<<<(unsigned)grid, 2 * cpb, sm, st>>>(tl_status, x, y, (int)n, batch, bc, yp1, ypn, y2, S, ntiles,
                                                 FastDiv((uint32_t)n));
      return launch_rc();
    }
    int cpb = 128;
    while (cpb > 16 && (size_t)2 * (cpb + 1) * S * sizeof(T) > 100 * 1024) cpb -= 16;
    const size_t sm = (size_t)2 * (cpb + 1) * S * sizeof(T);
    auto kern = k1_thomas_babe<T>;
    if (int rc = set_smem(kern, sm)) return rc;
    const int64_t grid = (batch + cpb - 1) / cpb;
    kern<<<(unsigned)grid, 2 * cpb, sm, st>>>(tl_status, x, y, (int)n, batch, bc, yp1, ypn, y2, S, FastDiv((uint32_t)n));
    return launch_rc();
  }
  if (n <= 256 * rmax<T>()) return build_mid<T>(x, y, n, batch, bc, yp1, ypn, y2, st);
  return build_long<T>(x, y, n, batch, bc, yp1, ypn, y2, st);
}

// ------------------------------------------------------------------------- eval

template <typename T, int MODE, int V, bool BULK, int L2 = 0>
int launch_staged_k(const T *x, const T *y, const T *y2, int n, int64_t batch, const T *q, int64_t m, T *out,
                    int32_t *idx, int cpb, int nchunks, int qchunk, int64_t nitems, cudaStream_t st) {
  static_assert(!BULK || V > 1, "query staging needs 16-byte query groups");
  if constexpr (MODE == MODE_BISECT && L2 == 0) {
    // the compile-time search depth: 2^L2 >= n - 1
    switch (eytz_levels(n)) {
      case 2: return launch_staged_k<T, MODE, V, BULK, 2>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 3: return launch_staged_k<T, MODE, V, BULK, 3>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 4: return launch_staged_k<T, MODE, V, BULK, 4>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 5: return launch_staged_k<T, MODE, V, BULK, 5>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 6: return launch_staged_k<T, MODE, V, BULK, 6>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 7: return launch_staged_k<T, MODE, V, BULK, 7>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 8: return launch_staged_k<T, MODE, V, BULK, 8>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      default: return launch_staged_k<T, MODE, V, BULK, 9>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
    }
  }
  const int qmax = (cpb > 1) ? cpb * (int)m : qchunk;
  const StageLayout<T> L(cpb, n, MODE, BULK ? qmax : 0);
  const size_t sm = L.total;
  auto kern = k_eval_staged<T, MODE, V, BULK, L2>;
  if (int rc = set_smem(kern, sm)) return rc;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kEvalThreads, sm) != cudaSuccess || occ < 1) occ = 1;
  const int64_t grid = std::min<int64_t>(nitems, (int64_t)occ * num_sms());
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kEvalThreads), sm, st, tl_status, x, y, y2, n, batch, q, (int)m, out, idx,
                    cpb, nchunks, qchunk, qmax, nitems, FastDiv((uint32_t)n), FastDiv((uint32_t)m));
}


template <typename T, int MODE, int L2 = 0>
int launch_warps_k(const T *x, const T *y, const T *y2, int n, int64_t batch, const T *q, int64_t m, T *out,
                   int32_t *idx, int cpb, int64_t nitems, cudaStream_t st) {
  if constexpr (MODE == MODE_BISECT && L2 == 0) {
    switch (eytz_levels(n)) {
      case 2: return launch_warps_k<T, MODE, 2>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      case 3: return launch_warps_k<T, MODE, 3>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      case 4: return launch_warps_k<T, MODE, 4>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      case 5: return launch_warps_k<T, MODE, 5>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      case 6: return launch_warps_k<T, MODE, 6>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      case 7: return launch_warps_k<T, MODE, 7>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      case 8: return launch_warps_k<T, MODE, 8>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
      default: return launch_warps_k<T, MODE, 9>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
    }
  } else {
    const StageLayout<T> L(cpb, n, MODE, cpb * (int)m);
    const size_t sm = L.total;
    auto kern = k_eval_warps<T, MODE, L2>;
    if (int rc = set_smem(kern, sm)) return rc;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kEvalThreads, sm) != cudaSuccess || occ < 1) occ = 1;
    const int64_t grid = std::min<int64_t>(nitems, (int64_t)occ * num_sms());
    return launch_pdl(kern, dim3((unsigned)grid), dim3(kEvalThreads), sm, st, tl_status, x, y, y2, n, batch, q, (int)m, out,
                      idx, cpb, nitems, FastDiv((uint32_t)n), FastDiv((uint32_t)m));
  }
}

constexpr size_t kSmemCap = 220 * 1024;   // per-CTA dynamic shared memory we allow ourselves
constexpr size_t kItemSmem = 72 * 1024;   // target per-CTA footprint for multi-curve items

constexpr int kQMax = 4096;  // queries per staged work item (BULK path)
template <typename T> size_t stage_total(int cpb, int n, int mode, int qmax = 0) {
  return StageLayout<T>(cpb, n, mode, qmax).total;
}

template <typename T, int MODE>
int launch_staged(const T *x, const T *y, const T *y2, int n, int64_t batch, const T *q, int64_t m, T *out,
                  int32_t *idx, cudaStream_t st) {
  constexpr int VW = 16 / sizeof(T);
  int cpb = 1, nchunks = 1, qchunk = (int)m;
  int64_t nitems;
  if (m >= 2048 || batch == 1) {
    // One curve per item; split a curve's queries into chunks of <= kQMax (and enough items
    // to fill the GPU when there are few curves).
    const int64_t want = (4 * 148 + batch - 1) / batch;
    nchunks = (int)std::max<int64_t>({(int64_t)1, std::min<int64_t>(want, (m + 1023) / 1024),
                                      (m + kQMax - 1) / kQMax});
    qchunk = (int)((m + nchunks - 1) / nchunks);
    qchunk = (qchunk + VW - 1) / VW * VW;
    nchunks = (int)((m + qchunk - 1) / qchunk);
    nitems = batch * nchunks;
  } else {
    int64_t c = std::max<int64_t>(1, kQMax / m);
    c = std::min<int64_t>(c, batch);
    while (c > 1 && stage_total<T>((int)c, n, MODE, (int)(c * m)) > kItemSmem) c >>= 1;
    while (c > 1 && (uint64_t)c * m * m >= (1ull << 32)) c >>= 1;  // FastDiv range
    cpb = (int)std::max<int64_t>(1, c);
    nitems = (batch + cpb - 1) / cpb;
  }
  // 16-byte vector query I/O when every curve's query run is whole vectors and aligned;
  // TMA bulk staging of knots + queries when, in addition, curve blocks are whole 16-byte units.
  const bool vec = (m % VW == 0) && aligned16(q) && aligned16(out) && (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0));
  const bool bulk = vec && ((n * sizeof(T)) % 16 == 0) && aligned16(x) && aligned16(y) && aligned16(y2);
  // per-warp curve ownership for the bisection mode (measured faster there; the uniform-grid
  // mode, whose per-query work is small, keeps the CTA-wide pack)
  if (bulk && cpb >= 8 && cpb % 8 == 0 && MODE == MODE_BISECT)
    return launch_warps_k<T, MODE>(x, y, y2, n, batch, q, m, out, idx, cpb, nitems, st);
  if (bulk) return launch_staged_k<T, MODE, VW, true>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
  if (vec) return launch_staged_k<T, MODE, VW, false>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
  return launch_staged_k<T, MODE, 1, false>(x, y, y2, n, batch, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
}

// Sorted runs with 4 queries per lane: q, out aligned to 4 elements (32 B fp64, 16 B fp32), idx to
// 16 B, m a multiple of 4.
template <typename T> bool sorted_v4_ok(const T *q, int64_t m, const T *out, const int32_t *idx) {
  constexpr uintptr_t A = 4 * sizeof(T) - 1;
  return m % 4 == 0 && (((uintptr_t)q | (uintptr_t)out) & A) == 0 && (!idx || ((uintptr_t)idx & 15) == 0);
}

#ifndef FS_SORTED_WALK
#define FS_SORTED_WALK 0  // A/B: 1.54 vs 1.10 ms on cfg4
#endif
template <typename T, int V, int FORM = FORM_RECORD>
int launch_sorted_k(const T *x, const T *y, const T *y2, int n, int64_t batch, const T *q, int64_t m, T *out,
                    int32_t *idx, cudaStream_t st) {
  // runs of ~8192 queries per warp (2048: +2%, 16384: +5% on cfg4), but at least ~8 warps per SM of work
  int64_t qrun = 8192;
  while (qrun > 256 && batch * ((m + qrun - 1) / qrun) < 148 * 32) qrun >>= 1;
  qrun = (qrun + 32 * V - 1) / (32 * V) * (32 * V);
  // dense runs with 32-byte aligned q / out and m % 8 == 0: every lane walks its own queries
  if (FS_SORTED_WALK && FORM == FORM_RECORD && m >= (int64_t)kSortWinDensity * (n - 1) && m % 8 == 0 &&
      ((((uintptr_t)q) | ((uintptr_t)out)) & 31) == 0 && (!idx || (((uintptr_t)idx) & (sizeof(T) == 4 ? 31 : 15)) == 0)) {
    const int64_t qw = (qrun + kWalkQ - 1) / kWalkQ * kWalkQ;
    const int64_t rpcw = (m + qw - 1) / qw;
    const int64_t ntw = batch * rpcw;
    return launch_pdl(k_eval_walk<T>, dim3((unsigned)((ntw + 7) / 8)), dim3(256), 0, st, tl_status, x, y, y2, n, q, m,
                      out, idx, qw, rpcw, ntw);
  }
  const int64_t rpc = (m + qrun - 1) / qrun;
  const int64_t ntasks = batch * rpc;
  const int64_t grid = (ntasks + 7) / 8;
  if (FORM == FORM_RECORD && m >= (int64_t)kSortWinDensity * (n - 1))  // dense: the record window pays
    return launch_pdl(k_eval_sorted<T, V, FORM_RECORD, true>, dim3((unsigned)grid), dim3(256), 0, st, tl_status, x, y, y2, n, q,
                      m, out, idx, qrun, rpc, ntasks);
  return launch_pdl(k_eval_sorted<T, V, FORM>, dim3((unsigned)grid), dim3(256), 0, st, tl_status, x, y, y2, n, q, m, out, idx,
                    qrun, rpc, ntasks);
}

template <typename T, int L2>
int launch_curvewarp_k(const T *x, const T *y, const T *y2, int n, int64_t batch, const T *q, int m, T *out,
                       int32_t *idx, cudaStream_t st) {
  auto kern = k_eval_curvewarp<T, L2>;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kCwWarps * 32, 0) != cudaSuccess || occ < 1) occ = 1;
  const int64_t grid = std::min<int64_t>((batch + kCwWarps - 1) / kCwWarps, (int64_t)occ * num_sms());
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kCwWarps * 32), 0, st, tl_status, x, y, y2, n, batch, q, m, out, idx);
}
template <typename T>
int launch_curvewarp(const T *x, const T *y, const T *y2, int n, int64_t batch, const T *q, int m, T *out,
                     int32_t *idx, cudaStream_t st) {
  switch (eytz_levels(n)) {
    case 2: return launch_curvewarp_k<T, 2>(x, y, y2, n, batch, q, m, out, idx, st);
    case 3: return launch_curvewarp_k<T, 3>(x, y, y2, n, batch, q, m, out, idx, st);
    case 4: return launch_curvewarp_k<T, 4>(x, y, y2, n, batch, q, m, out, idx, st);
    case 5: return launch_curvewarp_k<T, 5>(x, y, y2, n, batch, q, m, out, idx, st);
    default: return launch_curvewarp_k<T, 6>(x, y, y2, n, batch, q, m, out, idx, st);
  }
}

// k_eval_small's shapes: fp32, n <= 8, m <= 32 with m % 4 == 0, 16-byte aligned q, out, idx
template <typename T> bool small_eval_ok(int64_t n, const T *q, int64_t m, const T *out, const int32_t *idx) {
  return sizeof(T) == 4 && n <= kSmallN && m > 0 && m <= kSmallM && m % 4 == 0 && aligned16(q) && aligned16(out) &&
         (!idx || aligned16(idx));
}

// ---- one long curve, many unsorted queries: queries bucketed by L2-sized chunks (eval_bucket.cuh)
constexpr size_t kBkChunkBytes = size_t(24) << 20;  // x, y, y2 of one chunk: 2-3 chunks live in the 126 MB L2
template <typename T> bool bucket_eligible(int64_t n, int64_t batch, int64_t m) {
  // the curve must dwarf L2 (else the record gathers hit L2 anyway) and carry many queries;
  // FASTSPLINE_BUCKET_MIN_N (test tooling: sanitizer runs on small shapes) lowers the size bar
  static const int64_t min_n = [] {
    const char *e = getenv("FASTSPLINE_BUCKET_MIN_N");
    return e && *e ? (int64_t)atoll(e) : (int64_t)-1;
  }();
  if (min_n >= 0) return batch == 1 && n >= min_n && m >= n / 4;
  return batch == 1 && 3 * sizeof(T) * (size_t)n > 4 * kBkChunkBytes && m >= (int64_t)1 << 20 && m >= n / 4;
}
template <typename T>
int eval_bucketed(const T *x, const T *y, const T *y2, int64_t n, const T *q, int64_t m, T *out, int32_t *idx,
                  cudaStream_t st) {
  int64_t K = (int64_t)(kBkChunkBytes / sizeof(Knot<T>));
  K = std::min<int64_t>(K, std::max<int64_t>(1024, (n - 1) / 8));  // at least ~8 chunks on shorter curves
  K = std::max<int64_t>(K, (n - 1 + kBkMaxBuckets - 1) / kBkMaxBuckets);
  const int nb = (int)((n - 1 + K - 1) / K);
  const int64_t ntiles = (m + kBkTile - 1) / kBkTile;
  const int64_t L = (int64_t)(nb + 1) * ntiles;  // (bucket, tile) runs, bucket-major
  const int64_t nblk = (L + kScanBlock - 1) / kScanBlock;
  const int64_t neval = (m + kBkEvalPer - 1) / kBkEvalPer;
  if (ntiles >= (int64_t(1) << 31) || L >= (int64_t(1) << 31) || neval >= (int64_t(1) << 31) ||
      m >= (int64_t(1) << 32))
    return SPLINE_EINVAL;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t bk = al(sizeof(Knot<T>) * (size_t)n), bq = al(sizeof(T) * (size_t)m);
  const size_t bp = al(2 * (size_t)m), bi = idx ? al(4 * (size_t)m) : 0;
  const size_t bc = al(4 * (size_t)L), bs = al(4 * (size_t)nblk), bv = al(sizeof(unsigned long long));
  char *ws = nullptr;
  if (int rc = ws_alloc((void **)&ws, bk + 2 * bq + bp + bi + bc + bs + bv, st)) return rc;
  char *p = ws;
  auto take = [&](size_t b) { char *r = p; p += b; return r; };
  Knot<T> *kn = (Knot<T> *)take(bk);
  T *qs = (T *)take(bq);
  T *os = (T *)take(bq);
  uint16_t *perm = (uint16_t *)take(bp);
  int32_t *is = idx ? (int32_t *)take(bi) : nullptr;
  int *cnt = (int *)take(bc);
  int *bsum = (int *)take(bs);
  unsigned long long *dev = (unsigned long long *)take(bv);  // the knots' deviation from the guess
  int rc = set_smem(k_bucket_scatter<T>, bucket_scatter_smem<T>());
  if (!rc) rc = set_smem(k_bucket_gather<T>, bucket_gather_smem<T>());
  // the knot packing (bandwidth-bound) runs on an internal stream beside the counting and the
  // scatter (shared-memory-atomic-bound); the evaluation waits for both
  HostStreams *hs = nullptr;
  CallEvents ev;
  if (!rc) rc = host_streams(&hs);
  if (!rc) rc = ev.init();
  if (!rc) rc = cuda_rc(cudaEventRecord(ev.start, st));
  if (!rc) rc = cuda_rc(cudaStreamWaitEvent(hs->s[0], ev.start, 0));
  if (!rc) {
    const int64_t pg = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    rc = cuda_rc(cudaMemsetAsync(dev, 0, sizeof(unsigned long long), hs->s[0]));
    if (!rc) k_pack_knots<T><<<(unsigned)pg, 256, 0, hs->s[0]>>>(x, y, y2, n, kn, kBkBand ? dev : nullptr);
    rc = launch_rc();
  }
  if (!rc) rc = cuda_rc(cudaEventRecord(ev.ready, hs->s[0]));
  if (!rc)
    rc = launch_pdl(k_bucket_count<T>, dim3((unsigned)ntiles), dim3(kBkScThreads), 0, st, x, (int)n, K, nb, q, m, cnt);
  if (!rc) {
    k_scan_blocks<<<(unsigned)nblk, 1024, 0, st>>>(cnt, L, bsum);
    k_scan_top<<<1, 1024, 0, st>>>(bsum, (int)nblk);
    k_bucket_scatter<T><<<(unsigned)ntiles, kBkScThreads, bucket_scatter_smem<T>(), st>>>(x, (int)n, K, nb, q, m, cnt,
                                                                                           bsum, qs, perm);
    cudaStreamWaitEvent(st, ev.ready, 0);  // the packed knots
    k_bucket_eval<T><<<(unsigned)neval, kBkThreads, 0, st>>>(tl_status, kn, (int)n, K, nb, m, cnt, bsum, qs, os,
                                                             is, kBkBand ? dev : nullptr);
    k_bucket_gather<T><<<(unsigned)ntiles, kBkGaThreads, bucket_gather_smem<T>(), st>>>(os, is, perm, m, cnt, bsum, nb,
                                                                                         out, idx);
    rc = launch_rc();
  }
  cudaFreeAsync(ws, st);
  return rc;
}

template <typename T>
int eval_t(const T *x, const T *y, const T *y2, int64_t n, int64_t batch, const T *q, int64_t m, T *out,
           int32_t *idx, int flags, cudaStream_t st) {
  const bool xshared = (flags & SPLINE_X_SHARED) && batch > 1;
  flags &= ~SPLINE_X_SHARED;
  if (xshared && !small_eval_ok<T>(n, q, m, out, idx)) {  // no native knot-row stride: broadcast x
    T *xb = nullptr;
    int rc = broadcast_x<T>(x, n, batch, st, &xb);
    if (!rc) rc = eval_t<T>(xb, y, y2, n, batch, q, m, out, idx, flags, st);
    if (xb) cudaFreeAsync(xb, st);
    return rc;
  }
  if (flags & SPLINE_Q_SORTED) {
    constexpr int VW = 16 / sizeof(T);
    // 4 queries per lane and step (fp64: one 256-bit access each for q and out)
    if (sorted_v4_ok(q, m, out, idx)) return launch_sorted_k<T, 4>(x, y, y2, (int)n, batch, q, m, out, idx, st);
    const bool vec = (m % VW == 0) && aligned16(q) && aligned16(out) && (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0));
    if (vec) return launch_sorted_k<T, VW>(x, y, y2, (int)n, batch, q, m, out, idx, st);
    return launch_sorted_k<T, 1>(x, y, y2, (int)n, batch, q, m, out, idx, st);
  }
  if constexpr (sizeof(T) == 4) {  // very short curves with few queries (cfg3): k_eval_small
    if (small_eval_ok<T>(n, q, m, out, idx)) {
      const int vecn = n == kSmallN && aligned16(x) && aligned16(y) && aligned16(y2);
      const int64_t ntiles = (batch + 31) / 32;
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_small<false>, kSmallWarps * 32, 0) !=
              cudaSuccess ||
          occ < 1)
        occ = 1;
      const int64_t grid = std::min<int64_t>((ntiles + kSmallWarps - 1) / kSmallWarps, (int64_t)occ * num_sms());
      return launch_pdl(k_eval_small<false>, dim3((unsigned)grid), dim3(kSmallWarps * 32), 0, st, tl_status, x, y, y2, (int)n,
                        batch, q, (int)m, out, idx, vecn, 0, (const float *)nullptr, (const float *)nullptr,
                        (float *)nullptr, xshared ? (int64_t)0 : n);
    }
  }
  {  // curves of up to 64 knots, unsorted queries: one warp per curve (k_eval_curvewarp)
    constexpr int VW = 16 / sizeof(T);
    // (enough curves to give every SM several warps; few long query runs are split by the staged path)
    if (!(flags & SPLINE_X_UNIFORM) && n <= kCwMaxN && batch >= 4 * (int64_t)num_sms() && m > 0 && m % VW == 0 &&
        aligned16(q) && aligned16(out) &&
        (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0)))
      return launch_curvewarp<T>(x, y, y2, (int)n, batch, q, (int)m, out, idx, st);
  }
  if (n < 65535) {
    const int nn = (int)n;
    if ((flags & SPLINE_X_UNIFORM) && stage_total<T>(1, nn, MODE_UNIFORM, kQMax) <= kSmemCap)
      return launch_staged<T, MODE_UNIFORM>(x, y, y2, nn, batch, q, m, out, idx, st);
    // short curves: branch-free bisection; longer curves with many queries per knot: the
    // bucket table (its O(n) build per item is amortised over the queries)
    if (n <= 512 && stage_total<T>(1, nn, MODE_BISECT, kQMax) <= kSmemCap)
      return launch_staged<T, MODE_BISECT>(x, y, y2, nn, batch, q, m, out, idx, st);
    if (stage_total<T>(1, nn, MODE_TABLE, kQMax) <= kSmemCap)
      return launch_staged<T, MODE_TABLE>(x, y, y2, nn, batch, q, m, out, idx, st);
    if (stage_total<T>(1, nn, MODE_BSEARCH, kQMax) <= kSmemCap)
      return launch_staged<T, MODE_BSEARCH>(x, y, y2, nn, batch, q, m, out, idx, st);
  }
  if (bucket_eligible<T>(n, batch, m) && !(flags & kEvalNoBucket))
    return eval_bucketed<T>(x, y, y2, n, q, m, out, idx, st);
  const int64_t total = batch * m;
  // interval records in a pooled workspace: one gather round trip per query
  const size_t rec_bytes = sizeof(Ival<T>) * (size_t)n * batch, hdr_bytes = sizeof(CurveHdr<T>) * (size_t)batch;
  void *ws = nullptr;
  if (ws_alloc(&ws, rec_bytes + hdr_bytes, st) == SPLINE_OK) {
    Ival<T> *R = reinterpret_cast<Ival<T> *>(ws);
    CurveHdr<T> *H = reinterpret_cast<CurveHdr<T> *>(reinterpret_cast<char *>(ws) + rec_bytes);
    const int64_t pg = std::min<int64_t>(((n + 3) / 4 * batch + 255) / 256, (int64_t)num_sms() * 16);
    int rc = launch_pdl(k_pack_records<T>, dim3((unsigned)pg), dim3(256), 0, st, x, y, y2, (int)n, batch, R, H);
    if (!rc) {
      const int64_t grid = std::min<int64_t>((total + 1023) / 1024, (int64_t)num_sms() * 16);
      k_eval_records<T><<<(unsigned)grid, 256, 0, st>>>(tl_status, R, H, (int)n, batch, q, m, out, idx);
      rc = launch_rc();
    }
    cudaFreeAsync(ws, st);
    return rc;
  }
  cudaGetLastError();  // clear the failed allocation: the caller sees SPLINE_ENOMEM
  return SPLINE_ENOMEM;
}

// ------------------------------------------------------------------ fused build + eval

template <typename T, int MODE, int L2, int SOLVE, bool WOWN>
int launch_fused_k(const T *x, const T *y, int n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                   const T *q, int64_t m, T *out, int32_t *idx, int cpb, int nchunks, int qchunk, int64_t nitems,
                   cudaStream_t st) {
  if constexpr (MODE == MODE_BISECT && L2 == 0) {
    const int l2 = eytz_levels(n);
    if constexpr (SOLVE == SOLVE_REGS) {  // n <= 8
      if (l2 <= 2) return launch_fused_k<T, MODE, 2, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      return launch_fused_k<T, MODE, 3, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
    } else {
    switch (l2) {
      case 2: return launch_fused_k<T, MODE, 2, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 3: return launch_fused_k<T, MODE, 3, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 4: return launch_fused_k<T, MODE, 4, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 5: return launch_fused_k<T, MODE, 5, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      case 6: return launch_fused_k<T, MODE, 6, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
      default: return launch_fused_k<T, MODE, 7, SOLVE, WOWN>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb, nchunks, qchunk, nitems, st);
    }
    }
  } else {
    const int qmax = (cpb > 1) ? cpb * (int)m : qchunk;
    const FusedLayout<T> L(cpb, n, qmax, SOLVE, MODE, WOWN);
    const size_t sm = L.total;
    auto kern = k_fused_staged<T, MODE, L2, SOLVE, WOWN>;
    if (int rc = set_smem(kern, sm)) return rc;
    int occ = 0;
    constexpr int NT = fused_threads(WOWN);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, sm) != cudaSuccess || occ < 1) occ = 1;
    const int64_t grid = std::min<int64_t>(nitems, (int64_t)occ * num_sms());
    kern<<<(unsigned)grid, NT, sm, st>>>(tl_status, x, y, n, batch, bc, yp1, ypn, y2, q, (int)m, out, idx, cpb, nchunks,
                                                   qchunk, qmax, nitems, FastDiv((uint32_t)n), FastDiv((uint32_t)m));
    return launch_rc();
  }
}

constexpr size_t kFusedItemSmem = 72 * 1024;  // per-CTA target (3 CTAs per SM)
constexpr int kFusedMaxN = 128;

template <typename T> bool fused_eligible(const T *x, const T *y, int64_t n, const T *q, int64_t m, const T *out,
                                          const int32_t *idx, const T *y2) {
  constexpr int VW = 16 / sizeof(T);
  if (n > kFusedMaxN || (n * sizeof(T)) % 16 != 0 || m % VW != 0) return false;
  if (!aligned16(x) || !aligned16(y) || !aligned16(q) || !aligned16(out) || (y2 && !aligned16(y2))) return false;
  if (idx && ((uintptr_t)idx & (4 * VW - 1)) != 0) return false;
  const int mode = MODE_BISECT;  // the larger footprint of the two modes
  const int solve = n <= kRegsNMax ? SOLVE_REGS : SOLVE_BABE;
  return FusedLayout<T>(1, (int)n, kQMax, solve, mode, false).total <= kSmemCap;
}

template <typename T, int MODE>
int launch_fused(const T *x, const T *y, int n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2, const T *q,
                 int64_t m, T *out, int32_t *idx, cudaStream_t st) {
  constexpr int VW = 16 / sizeof(T);
  const int solve = n <= kRegsNMax ? SOLVE_REGS : SOLVE_BABE;
  int cpb = 1, nchunks = 1, qchunk = (int)m;
  int64_t nitems;
  if (m >= 2048 || batch == 1) {
    const int64_t want = (4 * 148 + batch - 1) / batch;
    nchunks = (int)std::max<int64_t>({(int64_t)1, std::min<int64_t>(want, (m + 1023) / 1024),
                                      (m + kQMax - 1) / kQMax});
    qchunk = (int)((m + nchunks - 1) / nchunks);
    qchunk = (qchunk + VW - 1) / VW * VW;
    nchunks = (int)((m + qchunk - 1) / qchunk);
    nitems = batch * nchunks;
  } else {
    int64_t c = std::max<int64_t>(1, kQMax / m);
    c = std::min<int64_t>(c, batch);
    while (c > 1 && FusedLayout<T>((int)c, n, (int)(c * m), solve, MODE, c >= 8).total > kFusedItemSmem) --c;
    while (c > 1 && (uint64_t)c * m * m >= (1ull << 32)) c >>= 1;  // FastDiv range
    cpb = (int)std::max<int64_t>(1, c);
    nitems = (batch + cpb - 1) / cpb;
  }
  // per-warp curve ownership needs whole curves for each of the 8 evaluator warps
  if (cpb >= 8) {
    cpb = cpb / 8 * 8;
    nitems = (batch + cpb - 1) / cpb;
    if (solve == SOLVE_REGS)
      return launch_fused_k<T, MODE, 0, SOLVE_REGS, true>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb,
                                                          nchunks, qchunk, nitems, st);
    return launch_fused_k<T, MODE, 0, SOLVE_BABE, true>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb,
                                                        nchunks, qchunk, nitems, st);
  }
  if (solve == SOLVE_REGS)
    return launch_fused_k<T, MODE, 0, SOLVE_REGS, false>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb,
                                                         nchunks, qchunk, nitems, st);
  return launch_fused_k<T, MODE, 0, SOLVE_BABE, false>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, cpb,
                                                       nchunks, qchunk, nitems, st);
}

// ---- fused build + eval of mid-length curves with sorted queries (k_tile_eval) ---------------
template <typename T, int R, int V, bool WIN>
int launch_tile_eval_k(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                       const T *q, int64_t m, T *out, int32_t *idx, cudaStream_t st) {
  auto kern = k_tile_eval<T, R, V, WIN>;
  const size_t sm = tile_eval_smem_bytes<T, R>();
  if (int rc = set_smem(kern, sm)) return rc;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTileThreads, sm) != cudaSuccess || occ < 1) occ = 1;
  // few curves: split each curve's queries over several CTAs (each solves the curve again, on
  // chip) so that the grid still fills ~3 waves of the GPU
  const int64_t slots = (int64_t)occ * num_sms();
  int nchunks = 1;
  while (batch * nchunks < 3 * slots && m / (2 * nchunks) >= (int64_t)kTileEvalWarps * 32 * V * 8 && nchunks < 1024)
    nchunks *= 2;
  int64_t qchunk = (m + nchunks - 1) / nchunks;
  qchunk = (qchunk + 32 * V - 1) / (32 * V) * (32 * V);
  nchunks = (int)((m + qchunk - 1) / qchunk);
  if (batch * nchunks >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  kern<<<(unsigned)(batch * nchunks), kTileThreads, sm, st>>>(tl_status, x, y, (int)n, bc, yp1, ypn, y2, q, m, out, idx,
                                                              nchunks, qchunk);
  return launch_rc();
}
template <typename T, int R>
int launch_tile_eval_r(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                       const T *q, int64_t m, T *out, int32_t *idx, cudaStream_t st) {
  constexpr int VW = 16 / sizeof(T);
  const bool vec = (m % VW == 0) && aligned16(q) && aligned16(out) && (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0));
  const bool win = m >= (int64_t)kSortWinDensity * (n - 1);  // dense runs: the record window pays (as eval_t)
  if (sorted_v4_ok(q, m, out, idx)) {
    if (win) return launch_tile_eval_k<T, R, 4, true>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
    return launch_tile_eval_k<T, R, 4, false>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  }
  if (vec) {
    if (win) return launch_tile_eval_k<T, R, VW, true>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
    return launch_tile_eval_k<T, R, VW, false>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  }
  if (win) return launch_tile_eval_k<T, R, 1, true>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  return launch_tile_eval_k<T, R, 1, false>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
}
template <typename T>
int launch_tile_eval(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                     const T *q, int64_t m, T *out, int32_t *idx, cudaStream_t st) {
  if (n <= 256 * 1) return launch_tile_eval_r<T, 1>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  if (n <= 256 * 2) return launch_tile_eval_r<T, 2>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  if (n <= 256 * 4) return launch_tile_eval_r<T, 4>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  if (n <= 256 * 8) return launch_tile_eval_r<T, 8>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  if (n <= 256 * 16) return launch_tile_eval_r<T, 16>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  if constexpr (rmax<T>() >= 32) {
    if (n <= 256 * 32) return launch_tile_eval_r<T, 32>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  }
  return SPLINE_EINVAL;
}

template <typename T, int N, int L2>
int launch_build_eval_warp_k(const T *x, const T *y, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                             const T *q, int m, T *out, int32_t *idx, cudaStream_t st) {
  auto kern = k_build_eval_warp<T, N, L2>;
  const size_t sm = kBwWarps * sizeof(BwStage<T, N>);
  if (int rc = set_smem(kern, sm)) return rc;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBwWarps * 32, sm) != cudaSuccess || occ < 1) occ = 1;
  const int64_t grid = std::min<int64_t>((batch + kBwWarps - 1) / kBwWarps, (int64_t)occ * num_sms());
  kern<<<(unsigned)grid, kBwWarps * 32, sm, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2, q, m, out, idx);
  return launch_rc();
}
template <typename T>
int launch_build_eval_warp(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn,
                           T *y2, const T *q, int m, T *out, int32_t *idx, cudaStream_t st) {
  if (n == 16) return launch_build_eval_warp_k<T, 16, 4>(x, y, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  if constexpr (sizeof(T) == 4) {
    if (n == 32) return launch_build_eval_warp_k<T, 32, 5>(x, y, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
    if (n == 64) return launch_build_eval_warp_k<T, 64, 6>(x, y, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  }
  return SPLINE_EINVAL;
}

template <typename T>
int build_eval_t(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                 const T *q, int64_t m, T *out, int32_t *idx, int flags, cudaStream_t st) {
  const bool xshared = (flags & SPLINE_X_SHARED) && batch > 1;
  flags &= ~SPLINE_X_SHARED;
  if (m == 0) return y2 ? build_t<T>(x, y, n, batch, bc, yp1, ypn, y2, st, xshared) : SPLINE_OK;
  if constexpr (sizeof(T) == 4) {  // very short fp32 curves, few queries: solve + eval in k_eval_small<true>
    if (!(flags & (SPLINE_PATH_FUSED | SPLINE_PATH_SPLIT)) && small_eval_ok<T>(n, q, m, out, idx)) {
      const int vecn = n == kSmallN && aligned16(x) && aligned16(y) && (!y2 || aligned16(y2));
      const int64_t ntiles = (batch + 31) / 32;
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_eval_small<true>, kSmallWarps * 32, 0) !=
              cudaSuccess ||
          occ < 1)
        occ = 1;
      const int64_t grid = std::min<int64_t>((ntiles + kSmallWarps - 1) / kSmallWarps, (int64_t)occ * num_sms());
      return launch_pdl(k_eval_small<true>, dim3((unsigned)grid), dim3(kSmallWarps * 32), 0, st, tl_status, x, y,
                        (const float *)nullptr, (int)n, batch, q, (int)m, out, idx, vecn, bc, yp1, ypn, y2,
                        xshared ? (int64_t)0 : n);
    }
  }
  if (xshared) {  // the other kernels read a knot row per curve: broadcast the knot vector first
    T *xb = nullptr;
    int rc = broadcast_x<T>(x, n, batch, st, &xb);
    if (!rc) rc = build_eval_t<T>(xb, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, flags, st);
    if (xb) cudaFreeAsync(xb, st);
    return rc;
  }
  {  // a few K1h-sized curves with few queries: one CTA per curve does the whole call
    constexpr int VW = 16 / sizeof(T);
    const bool k1h_n = n == 16 || (sizeof(T) == 4 && (n == 32 || n == 64));
    if (!(flags & (SPLINE_PATH_FUSED | SPLINE_PATH_SPLIT | kNoFusedStaged)) && k1h_n && batch <= 16 && m <= 8192 &&
        m % VW == 0 && aligned16(x) && aligned16(y) && aligned16(q) && aligned16(out) && (!y2 || aligned16(y2)) &&
        (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0))) {
      const unsigned g = (unsigned)batch;  // y2 == nullptr: the kernel keeps it on chip only
      if (n == 16) k_build_eval_tiny<T, 16, 4><<<g, 256, 0, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2, q, (int)m, out, idx);
      if constexpr (sizeof(T) == 4) {
        if (n == 32) k_build_eval_tiny<T, 32, 5><<<g, 256, 0, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2, q, (int)m, out, idx);
        if (n == 64) k_build_eval_tiny<T, 64, 6><<<g, 256, 0, st>>>(tl_status, x, y, batch, bc, yp1, ypn, y2, q, (int)m, out, idx);
      }
      return launch_rc();
    }
  }
  {  // many K1h-sized curves, unsorted (or sorted) queries: solve + evaluate per warp
    constexpr int VW = 16 / sizeof(T);
    const bool k1h_n = n == 16 || (sizeof(T) == 4 && (n == 32 || n == 64));
    if (kBuildEvalWarp && !(flags & (SPLINE_PATH_FUSED | SPLINE_PATH_SPLIT | SPLINE_X_UNIFORM)) && k1h_n &&
        batch >= 4 * (int64_t)num_sms() && m > 0 && m <= INT32_MAX && m % VW == 0 && aligned16(x) && aligned16(y) &&
        aligned16(q) && aligned16(out) && (!y2 || aligned16(y2)) && (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0)))
      return launch_build_eval_warp<T>(x, y, n, batch, bc, yp1, ypn, y2, q, (int)m, out, idx, st);
  }
  // mid-length curves (K2's range) with sorted queries: solve and evaluate in one kernel -- on
  // request only: measured on cfg4 the split path is faster (1.29 vs 1.69 ms: the evaluation is
  // issue-bound and needs the 32 warps/SM that the solve's 94 KB tile leaves it no room for)
  if ((flags & SPLINE_Q_SORTED) && (flags & SPLINE_PATH_FUSED) && n > kK1MaxN && n <= 256 * rmax<T>())
    return launch_tile_eval<T>(x, y, n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  const bool want_fused =
      (flags & SPLINE_PATH_FUSED) ||
      (!(flags & (SPLINE_PATH_SPLIT | kNoFusedStaged)) && batch * m <= kFuseMaxWork);
  flags &= (SPLINE_Q_SORTED | SPLINE_X_UNIFORM);
  if (want_fused && fused_eligible<T>(x, y, n, q, m, out, idx, y2)) {
    if (flags & SPLINE_X_UNIFORM)
      return launch_fused<T, MODE_UNIFORM>(x, y, (int)n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
    return launch_fused<T, MODE_BISECT>(x, y, (int)n, batch, bc, yp1, ypn, y2, q, m, out, idx, st);
  }
  // not fusable (long curves, unaligned or ragged arrays): the two kernels back to back
  T *yy = y2;
  if (!yy) {
    if (int rc = ws_alloc((void **)&yy, sizeof(T) * (size_t)n * batch, st)) return rc;
  }
  int rc;
  if (kSplitOverlap && n > kK1MaxN && n <= 256 * rmax<T>() && batch >= 8 * (int64_t)num_sms()) {
    // many mid-length curves (cfg4): the partition build is latency-bound at 2 CTAs/SM, the
    // evaluation issue-bound -- build the second half of the batch on an internal stream while
    // the first half is evaluated:  st: build A -> eval A -> (wait B) -> eval B;  s2: build B
    HostStreams *hs = nullptr;
    CallEvents ev;
    rc = host_streams(&hs);
    if (!rc) rc = ev.init();
    const int64_t h = batch / 2;
    cudaStream_t s2 = hs ? hs->s[0] : st;
    if (!rc) rc = build_t<T>(x, y, n, h, bc, yp1, ypn, yy, st);
    if (!rc) rc = cuda_rc(cudaEventRecord(ev.start, st));
    if (!rc) rc = cuda_rc(cudaStreamWaitEvent(s2, ev.start, 0));
    if (!rc) rc = build_t<T>(x + h * n, y + h * n, n, batch - h, bc, (bc & 1) ? yp1 + h : yp1, (bc & 2) ? ypn + h : ypn,
                             yy + h * n, s2);
    if (!rc) rc = cuda_rc(cudaEventRecord(ev.done[0], s2));
    if (!rc) rc = eval_t<T>(x, y, yy, n, h, q, m, out, idx, flags, st);
    if (!rc) rc = cuda_rc(cudaStreamWaitEvent(st, ev.done[0], 0));
    if (!rc) rc = eval_t<T>(x + h * n, y + h * n, yy + h * n, n, batch - h, q + h * m, m, out + h * m,
                            idx ? idx + h * m : nullptr, flags, st);
  } else {
    rc = build_t<T>(x, y, n, batch, bc, yp1, ypn, yy, st);
    if (!rc) rc = eval_t<T>(x, y, yy, n, batch, q, m, out, idx, flags, st);
  }
  if (!y2) cudaFreeAsync(yy, st);
  return rc;
}

// ---- host-resident arrays: chunked, copies overlapped with the kernels -------------------
// spline_build_eval_host: the batch is cut into chunks of whole curves; chunk i runs on
// internal stream i % kHostStreams: H2D of its x, y, q (and slopes), the device
// build+eval, D2H of its y2, out, idx -- so one chunk's H2D, another's kernels and a third's
// D2H overlap (PCIe is full duplex).  Device buffers come from the library pool; the call is
// ordered after prior work on `stream`, and `stream` waits for all of it.  Pinned host memory
// gives the overlap; pageable memory is correct but serialises the copies.
// One long curve with many queries: the knots go up and the build runs first (every query
// needs the whole y2), then the queries flow in chunks through the internal streams (each
// chunk: H2D q, eval, D2H out/idx), overlapping the two PCIe directions.  Few, large chunks:
// an eval call on a long curve re-packs its interval records.
template <typename T>
int build_eval_host_one_t(const T *x, const T *y, int64_t n, int bc, const T *yp1, const T *ypn, T *y2, const T *q,
                          int64_t m, T *out, int32_t *idx, int flags, cudaStream_t st, HostStreams *hs) {
  CallEvents ev;
  if (int rc = ev.init()) return rc;
  const size_t s = sizeof(T);
  const int64_t K = std::max<int64_t>(2, std::min<int64_t>(8, (int64_t)(((size_t)m * (2 * s + 4)) / (256u << 20))));
  const int64_t QC = (m + K - 1) / K;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t bx = al(s * n), bq = al(s * QC), bi = al(4 * (size_t)QC), bs = al(s);
  const size_t slot = 2 * bq + bi;
  char *base = nullptr;
  if (int rc = ws_alloc((void **)&base, 3 * bx + 2 * bs + kHostStreams * slot, st)) return rc;
  T *dx = (T *)base, *dy = (T *)(base + bx), *dz = (T *)(base + 2 * bx);
  T *ds1 = (T *)(base + 3 * bx), *ds2 = (T *)(base + 3 * bx + bs);
  char *sb = base + 3 * bx + 2 * bs;
  int rc = cuda_rc(cudaEventRecord(ev.start, st));
  cudaStream_t s0 = hs->s[0];
  if (!rc) rc = cuda_rc(cudaStreamWaitEvent(s0, ev.start, 0));
  if (!rc) rc = cuda_rc(cudaMemcpyAsync(dx, x, s * n, cudaMemcpyHostToDevice, s0));
  if (!rc) rc = cuda_rc(cudaMemcpyAsync(dy, y, s * n, cudaMemcpyHostToDevice, s0));
  if (!rc && (bc & 1)) rc = cuda_rc(cudaMemcpyAsync(ds1, yp1, s, cudaMemcpyHostToDevice, s0));
  if (!rc && (bc & 2)) rc = cuda_rc(cudaMemcpyAsync(ds2, ypn, s, cudaMemcpyHostToDevice, s0));
  if (!rc) rc = build_t<T>(dx, dy, n, 1, bc, (bc & 1) ? ds1 : nullptr, (bc & 2) ? ds2 : nullptr, dz, s0);
  if (!rc) rc = cuda_rc(cudaEventRecord(ev.ready, s0));  // y2 ready
  for (int k = 1; !rc && k < kHostStreams; ++k) rc = cuda_rc(cudaStreamWaitEvent(hs->s[k], ev.ready, 0));
  if (!rc && y2) rc = cuda_rc(cudaMemcpyAsync(y2, dz, s * n, cudaMemcpyDeviceToHost, s0));
  const int fl = flags & (SPLINE_Q_SORTED | SPLINE_X_UNIFORM);
  for (int64_t i = 0; !rc && i < K; ++i) {
    const int k = (int)(i % kHostStreams);
    cudaStream_t ss = hs->s[k];
    const int64_t k0 = i * QC, mc = std::min<int64_t>(QC, m - k0);
    if (mc <= 0) break;
    char *b = sb + slot * k;
    T *dq = (T *)b, *dout = (T *)(b + bq);
    int32_t *didx = (int32_t *)(b + 2 * bq);
    rc = cuda_rc(cudaMemcpyAsync(dq, q + k0, s * mc, cudaMemcpyHostToDevice, ss));
    if (!rc) rc = eval_t<T>(dx, dy, dz, n, 1, dq, mc, dout, idx ? didx : nullptr, fl, ss);
    if (!rc) rc = cuda_rc(cudaMemcpyAsync(out + k0, dout, s * mc, cudaMemcpyDeviceToHost, ss));
    if (!rc && idx) rc = cuda_rc(cudaMemcpyAsync(idx + k0, didx, 4 * (size_t)mc, cudaMemcpyDeviceToHost, ss));
  }
  for (int k = 0; k < kHostStreams; ++k) {
    cudaEventRecord(ev.done[k], hs->s[k]);
    cudaStreamWaitEvent(st, ev.done[k], 0);
  }
  cudaFreeAsync(base, st);
  return rc;
}

template <typename T>
int build_eval_host_t(const T *x, const T *y, int64_t n, int64_t batch, int bc, const T *yp1, const T *ypn, T *y2,
                      const T *q, int64_t m, T *out, int32_t *idx, int flags, cudaStream_t st) {
  HostStreams *hs = nullptr;
  if (int rc = host_streams(&hs)) return rc;
  // the whole problem's fused/split choice, kept for every chunk
  if (!(flags & (SPLINE_PATH_FUSED | SPLINE_PATH_SPLIT)))
    if (batch * m > kFuseMaxWork) flags |= kNoFusedStaged;  // chunks must not pick the small-problem kernel
  if (batch == 1) flags &= ~SPLINE_X_SHARED;
  const bool xsh = (flags & SPLINE_X_SHARED) != 0;  // one knot vector: every chunk copies only it
  const size_t s = sizeof(T);
  const size_t per_curve = s * ((xsh ? 2 : 3) * (size_t)n + 2 * (size_t)m + 2) + 4 * (size_t)m;  // device B/curve
  int64_t C = std::max<int64_t>(1, (int64_t)(kHostChunkBytes / per_curve));
  C = std::max<int64_t>(C, 2 * (int64_t)num_sms());            // keep every chunk GPU-wide
  C = std::min<int64_t>(C, std::max<int64_t>(1, (int64_t)(kMaxSlotBytes / per_curve)));  // within memory
  C = std::min<int64_t>(C, (batch + kHostStreams - 1) / kHostStreams);  // and at least kHostStreams chunks
  C = std::max<int64_t>(1, std::min<int64_t>(C, batch));
  const int64_t nchunk = (batch + C - 1) / C;
  if (nchunk == 1 && batch == 1 && (size_t)m * (2 * s + 4) > 8 * kHostChunkBytes)
    return build_eval_host_one_t<T>(x, y, n, bc, yp1, ypn, y2, q, m, out, idx, flags, st, hs);
  const int nslot = (int)std::min<int64_t>(kHostStreams, nchunk);
  // slot layout (16-byte aligned pieces)
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t bx = al(s * C * n), bq = al(s * C * m), bi = al(4 * (size_t)C * m), bs = al(s * C);
  const size_t slot = 3 * bx + 2 * bq + bi + 2 * bs;
  char *base = nullptr;
  if (int rc = ws_alloc((void **)&base, slot * nslot, st)) return rc;
  CallEvents ev;
  if (int rc = ev.init()) {
    cudaFreeAsync(base, st);
    return rc;
  }
  int rc = cuda_rc(cudaEventRecord(ev.start, st));
  for (int k = 0; !rc && k < nslot; ++k) rc = cuda_rc(cudaStreamWaitEvent(hs->s[k], ev.start, 0));
  for (int64_t i = 0; !rc && i < nchunk; ++i) {
    const int k = (int)(i % nslot);
    cudaStream_t ss = hs->s[k];
    const int64_t c0 = i * C, nc = std::min<int64_t>(C, batch - c0);
    char *b = base + slot * k;
    T *dx = (T *)b, *dy = (T *)(b + bx), *dz = (T *)(b + 2 * bx), *dq = (T *)(b + 3 * bx), *dout = (T *)(b + 3 * bx + bq);
    int32_t *didx = (int32_t *)(b + 3 * bx + 2 * bq);
    T *ds1 = (T *)(b + 3 * bx + 2 * bq + bi), *ds2 = (T *)(b + 3 * bx + 2 * bq + bi + bs);
    const size_t kn = s * nc * n, km = s * nc * m;
    rc = cuda_rc(cudaMemcpyAsync(dx, xsh ? x : x + c0 * n, xsh ? s * n : kn, cudaMemcpyHostToDevice, ss));
    if (!rc) rc = cuda_rc(cudaMemcpyAsync(dy, y + c0 * n, kn, cudaMemcpyHostToDevice, ss));
    if (!rc && m) rc = cuda_rc(cudaMemcpyAsync(dq, q + c0 * m, km, cudaMemcpyHostToDevice, ss));
    if (!rc && (bc & 1)) rc = cuda_rc(cudaMemcpyAsync(ds1, yp1 + c0, s * nc, cudaMemcpyHostToDevice, ss));
    if (!rc && (bc & 2)) rc = cuda_rc(cudaMemcpyAsync(ds2, ypn + c0, s * nc, cudaMemcpyHostToDevice, ss));
    if (!rc)
      rc = build_eval_t<T>(dx, dy, n, nc, bc, (bc & 1) ? ds1 : nullptr, (bc & 2) ? ds2 : nullptr, dz, dq, m, dout,
                           idx ? didx : nullptr, flags, ss);
    if (!rc && y2) rc = cuda_rc(cudaMemcpyAsync(y2 + c0 * n, dz, kn, cudaMemcpyDeviceToHost, ss));
    if (!rc && m) rc = cuda_rc(cudaMemcpyAsync(out + c0 * m, dout, km, cudaMemcpyDeviceToHost, ss));
    if (!rc && m && idx) rc = cuda_rc(cudaMemcpyAsync(idx + c0 * m, didx, 4 * (size_t)nc * m, cudaMemcpyDeviceToHost, ss));
  }
  for (int k = 0; k < nslot; ++k) {
    cudaEventRecord(ev.done[k], hs->s[k]);
    cudaStreamWaitEvent(st, ev.done[k], 0);
  }
  cudaFreeAsync(base, st);
  return rc;
}

template <typename T, int FORM>
int ablation_form(const T *x, const T *y, const T *y2, int64_t n, int64_t batch, const T *q, int64_t m, T *out,
                  int32_t *idx, cudaStream_t st) {
  constexpr int VW = 16 / sizeof(T);
  const bool vec = (m % VW == 0) && aligned16(q) && aligned16(out) && (!idx || (((uintptr_t)idx & (4 * VW - 1)) == 0));
  if (vec) return launch_sorted_k<T, VW, FORM>(x, y, y2, (int)n, batch, q, m, out, idx, st);
  return launch_sorted_k<T, 1, FORM>(x, y, y2, (int)n, batch, q, m, out, idx, st);
}

template <typename T>
int ablation_t(const T *x, const T *y, const T *y2, int64_t n, int64_t batch, const T *q, int64_t m, T *out,
               int32_t *idx, int form, cudaStream_t st) {
  switch (form) {
    case FORM_RECORD: return ablation_form<T, FORM_RECORD>(x, y, y2, n, batch, q, m, out, idx, st);
    case FORM_SPLINT_DIV: return ablation_form<T, FORM_SPLINT_DIV>(x, y, y2, n, batch, q, m, out, idx, st);
    case FORM_SPLINT_MUL: return ablation_form<T, FORM_SPLINT_MUL>(x, y, y2, n, batch, q, m, out, idx, st);
    case FORM_NEWINT_ORIG: return ablation_form<T, FORM_NEWINT_ORIG>(x, y, y2, n, batch, q, m, out, idx, st);
    case FORM_NEWINT_NOINV: return ablation_form<T, FORM_NEWINT_NOINV>(x, y, y2, n, batch, q, m, out, idx, st);
    case FORM_NOOP: return ablation_form<T, FORM_NOOP>(x, y, y2, n, batch, q, m, out, idx, st);
    default: return SPLINE_EINVAL;
  }
}

template <typename T>
int probe_t(const T *x, const T *y, const T *y2, int64_t n, int64_t batch, const T *q, int64_t m,
            const int32_t *idx_in, T *out, int32_t *idx, int mode, cudaStream_t st) {
  const int64_t total = batch * m;
  const int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
  if (mode == 0) {
    k_probe_raw<T><<<(unsigned)grid, 256, 0, st>>>(x, y, y2, (int)n, batch, q, m, idx_in, out, idx);
    return launch_rc();
  }
  const size_t rec_bytes = sizeof(Ival<T>) * (size_t)n * batch, hdr_bytes = sizeof(CurveHdr<T>) * (size_t)batch;
  void *ws = nullptr;
  if (int rc = ws_alloc(&ws, rec_bytes + hdr_bytes, st)) return rc;
  Ival<T> *R = reinterpret_cast<Ival<T> *>(ws);
  CurveHdr<T> *H = reinterpret_cast<CurveHdr<T> *>(reinterpret_cast<char *>(ws) + rec_bytes);
  const int64_t pg = std::min<int64_t>(((n + 3) / 4 * batch + 255) / 256, (int64_t)num_sms() * 16);
  k_pack_records<T><<<(unsigned)pg, 256, 0, st>>>(x, y, y2, (int)n, batch, R, H);
  int rc = launch_rc();
  if (!rc) {
    k_probe_rec<T><<<(unsigned)grid, 256, 0, st>>>(R, (int)n, batch, q, m, idx_in, out, idx);
    rc = launch_rc();
  }
  cudaFreeAsync(ws, st);
  return rc;
}

int check_build(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1, const void *ypn,
                const void *y2, int dtype) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || batch < 0 || batch >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  bc &= ~SPLINE_X_SHARED;
  if (bc < 0 || bc > 3) return SPLINE_EINVAL;
  if (batch == 0) return SPLINE_OK;
  if (!x || !y || !y2) return SPLINE_EINVAL;
  if ((bc & 1) && !yp1) return SPLINE_EINVAL;
  if ((bc & 2) && !ypn) return SPLINE_EINVAL;
  return SPLINE_OK;
}

}  // namespace

namespace {
template <typename T>
int spike_reduce_t(const T *x, const T *y, int64_t n, int64_t rb, int64_t re, int bc, const T *yp1, const T *ypn,
                   T *record, void *workspace, cudaStream_t st) {
  constexpr int R = rmax<T>();
  const int64_t ntiles = (re - rb + 256 * R - 1) / (256 * R);
  SpikeWs w;
  spike_ws_layout<T>(ntiles, 1, &w, (char *)workspace);
  int rc = cuda_rc(cudaMemsetAsync(w.badflag, 0, sizeof(int), st));
  if (!rc) rc = launch_tile_part<T, TILE_REDUCE>(x, y, n, rb, re, 1, bc, yp1, ypn, nullptr, w, st);
  if (!rc) rc = launch_top<T>((const T *)w.tile_rec, (int)ntiles, 1, 1, nullptr, nullptr, record, (T *)w.foldq, st);
  return rc;
}

template <typename T>
int spike_finish_t(const T *x, const T *y, int64_t n, int64_t rb, int64_t re, int bc, const T *yp1, const T *ypn,
                   const T *all_records, int nranks, int rank, T *y2_shard, void *workspace, cudaStream_t st) {
  constexpr int R = rmax<T>();
  const int64_t ntiles = (re - rb + 256 * R - 1) / (256 * R);
  SpikeWs w;
  spike_ws_layout<T>(ntiles, 1, &w, (char *)workspace);
  // Rank level: every rank solves the G-record reduced system redundantly (the outer
  // (L, R) of the whole curve are irrelevant: a_0 = 0 and c_{n-1} = 0).
  int rc = launch_top<T>(all_records, nranks, 1, 0, nullptr, (T *)w.rank_ext, nullptr, (T *)w.rank_foldq, st);
  if (!rc) rc = launch_top<T>((const T *)w.tile_rec, (int)ntiles, 1, 0, (const T *)w.rank_ext + 2 * rank,
                              (T *)w.tile_ext, nullptr, (T *)w.foldq, st);
  if (!rc) rc = launch_tile_part<T, TILE_FINISH>(x, y, n, rb, re, 1, bc, yp1, ypn, y2_shard, w, st);
  return rc;
}

// Recompute instead of communicate: the tile records of rows [rb, rb + k TS)
// (K3 only; every rank its own tiles), then -- given ALL tile records of the curve -- the reduced
// solve (K4) and the finish (K5) of the whole curve on every rank: the full y2 without moving it.
template <typename T>
int spike_tile_records_t(const T *x, const T *y, int64_t n, int64_t rb, int64_t re, int bc, const T *yp1,
                         const T *ypn, T *recs, void *workspace, cudaStream_t st) {
  constexpr int R = rmax<T>();
  const int64_t ntiles = (re - rb + 256 * R - 1) / (256 * R);
  SpikeWs w;
  spike_ws_layout<T>(ntiles, 1, &w, (char *)workspace);
  w.tile_rec = recs;
  int rc = cuda_rc(cudaMemsetAsync(w.badflag, 0, sizeof(int), st));
  if (!rc) rc = launch_tile_part<T, TILE_REDUCE>(x, y, n, rb, re, 1, bc, yp1, ypn, nullptr, w, st);
  return rc;
}
template <typename T>
int spike_finish_tiles_t(const T *x, const T *y, int64_t n, int bc, const T *yp1, const T *ypn, const T *all_recs,
                         T *y2, void *workspace, cudaStream_t st) {
  constexpr int R = rmax<T>();
  const int64_t ntiles = (n + 256 * R - 1) / (256 * R);
  SpikeWs w;
  spike_ws_layout<T>(ntiles, 1, &w, (char *)workspace);
  int rc = cuda_rc(cudaMemsetAsync(w.badflag, 0, sizeof(int), st));
  if (!rc) {
    if (ntiles > 2 * kGroupTiles && (ntiles + kGroupTiles - 1) / kGroupTiles <= kMaxRanks)
      rc = launch_top_grouped<T>(all_recs, (int)ntiles, w, st);
    else
      rc = launch_top<T>(all_recs, (int)ntiles, 1, 0, nullptr, (T *)w.tile_ext, nullptr, (T *)w.foldq, st);
  }
  if (!rc) rc = launch_tile_part<T, TILE_FINISH>(x, y, n, 0, n, 1, bc, yp1, ypn, y2, w, st);
  return rc;
}

int check_spike(const void *x, const void *y, int64_t n, int64_t rb, int64_t re, int bc, const void *yp1,
                const void *ypn, const void *ws, int dtype) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || rb < 0 || re > n || re <= rb || bc < 0 || bc > 3) return SPLINE_EINVAL;
  if (!x || !y || !ws) return SPLINE_EINVAL;
  if (((bc & 1) && !yp1) || ((bc & 2) && !ypn)) return SPLINE_EINVAL;
  return SPLINE_OK;
}
}  // namespace

// ---- the multi-GPU long-curve build over an NCCL communicator (spline_build_dist) ------------
// NCCL is resolved at run time (dlopen: the process's already-loaded libnccl.so.2, else the one
// SPLINE_NCCL_LIB names, else the loader's), so the library needs no link-time NCCL and a
// missing NCCL is an error code (SPLINE_ENCCL), not a load failure.
namespace {
typedef int (*nccl_count_fn)(void *, int *);
typedef int (*nccl_rank_fn)(void *, int *);
typedef int (*nccl_allgather_fn)(const void *, void *, size_t, int, void *, cudaStream_t);
struct NcclApi {
  nccl_count_fn count = nullptr;
  nccl_rank_fn rank = nullptr;
  nccl_allgather_fn allgather = nullptr;
  bool ok = false;
};
const NcclApi &nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = nullptr;
    const char *env = getenv("SPLINE_NCCL_LIB");
    if (env && *env) {
      h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    }
    if (!h) return;
    api.count = (nccl_count_fn)dlsym(h, "ncclCommCount");
    api.rank = (nccl_rank_fn)dlsym(h, "ncclCommUserRank");
    api.allgather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
    api.ok = api.count && api.rank && api.allgather;
  });
  return api;
}
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8;  // ncclDataType_t (nccl.h)

template <typename T>
int build_dist_t(const T *x, const T *y, int64_t n, int bc, const T *yp1, const T *ypn, T *y2_shard, void *comm,
                 cudaStream_t st) {
  const NcclApi &nc = nccl_api();
  if (!nc.ok) return SPLINE_ENCCL;
  int G = 0, r = 0;
  if (nc.count(comm, &G) != 0 || nc.rank(comm, &r) != 0 || G < 1 || r < 0 || r >= G) return SPLINE_ENCCL;
  if (G > kMaxRanks) return SPLINE_EINVAL;
  const int64_t rb = n * r / G, re = n * (r + 1) / G;  // this rank's rows (dist.shard_rows)
  if (re <= rb) return SPLINE_EINVAL;                  // more ranks than rows
  constexpr int R = rmax<T>();
  const int64_t ntiles = (re - rb + 256 * R - 1) / (256 * R);
  const size_t wsb = (spike_ws_layout<T>(ntiles, 1, nullptr, nullptr) + 255) & ~(size_t)255;
  const size_t recb = (sizeof(T) * 6 * (size_t)(G + 1) + 255) & ~(size_t)255;
  char *base = nullptr;
  if (int rc = ws_alloc((void **)&base, wsb + recb, st)) return rc;
  T *rec = (T *)(base + wsb), *all = rec + 6;
  int rc = spike_reduce_t<T>(x, y, n, rb, re, bc, yp1, ypn, rec, base, st);
  // the exchange step of the partitioned solve: every rank's 6-scalar block record to every rank
  if (!rc && nc.allgather(rec, all, 6, sizeof(T) == 8 ? kNcclFloat64 : kNcclFloat32, comm, st) != 0) rc = SPLINE_ENCCL;
  if (!rc) rc = spike_finish_t<T>(x, y, n, rb, re, bc, yp1, ypn, all, G, r, y2_shard, base, st);
  cudaFreeAsync(base, st);
  return rc;
}
}  // namespace

extern "C" {

int spline_build(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1, const void *ypn,
                 void *y2, int dtype, spline_stream_t stream) {
  if (int rc = check_build(x, y, n, batch, bc, yp1, ypn, y2, dtype)) return rc;
  if (batch == 0) return SPLINE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  const bool xsh = (bc & SPLINE_X_SHARED) != 0;
  bc &= ~SPLINE_X_SHARED;
  if (dtype == SPLINE_F32)
    return build_t<float>((const float *)x, (const float *)y, n, batch, bc, (const float *)yp1, (const float *)ypn,
                          (float *)y2, st, xsh);
  return build_t<double>((const double *)x, (const double *)y, n, batch, bc, (const double *)yp1,
                         (const double *)ypn, (double *)y2, st, xsh);
}

int spline_eval(const void *x, const void *y, const void *y2, int64_t n, int64_t batch, const void *q, int64_t m,
                void *out, int32_t *idx, int flags, int dtype, spline_stream_t stream) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || batch < 0 || m < 0 || m >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  if (flags & ~(SPLINE_Q_SORTED | SPLINE_X_UNIFORM | SPLINE_NO_BUCKET | SPLINE_X_SHARED)) return SPLINE_EINVAL;
  if (batch == 0 || m == 0) return SPLINE_OK;
  if (!x || !y || !y2 || !q || !out) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return eval_t<float>((const float *)x, (const float *)y, (const float *)y2, n, batch, (const float *)q, m,
                         (float *)out, idx, flags, st);
  return eval_t<double>((const double *)x, (const double *)y, (const double *)y2, n, batch, (const double *)q, m,
                        (double *)out, idx, flags, st);
}

int spline_build_eval(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1,
                      const void *ypn, void *y2, const void *q, int64_t m, void *out, int32_t *idx, int flags,
                      int dtype, spline_stream_t stream) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || batch < 0 || batch >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  if (m < 0 || m >= (int64_t(1) << 31) || bc < 0 || bc > 3) return SPLINE_EINVAL;
  if (flags & ~(SPLINE_Q_SORTED | SPLINE_X_UNIFORM | SPLINE_PATH_FUSED | SPLINE_PATH_SPLIT | SPLINE_X_SHARED))
    return SPLINE_EINVAL;
  if ((flags & SPLINE_PATH_FUSED) && (flags & SPLINE_PATH_SPLIT)) return SPLINE_EINVAL;
  if (batch == 0) return SPLINE_OK;
  if (!x || !y || ((bc & 1) && !yp1) || ((bc & 2) && !ypn)) return SPLINE_EINVAL;
  if (m > 0 && (!q || !out)) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return build_eval_t<float>((const float *)x, (const float *)y, n, batch, bc, (const float *)yp1,
                               (const float *)ypn, (float *)y2, (const float *)q, m, (float *)out, idx, flags, st);
  return build_eval_t<double>((const double *)x, (const double *)y, n, batch, bc, (const double *)yp1,
                              (const double *)ypn, (double *)y2, (const double *)q, m, (double *)out, idx, flags, st);
}

int spline_build_eval_host(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1,
                           const void *ypn, void *y2, const void *q, int64_t m, void *out, int32_t *idx, int flags,
                           int dtype, spline_stream_t stream) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || batch < 0 || batch >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  if (m < 0 || m >= (int64_t(1) << 31) || bc < 0 || bc > 3) return SPLINE_EINVAL;
  if (flags & ~(SPLINE_Q_SORTED | SPLINE_X_UNIFORM | SPLINE_PATH_FUSED | SPLINE_PATH_SPLIT | SPLINE_X_SHARED))
    return SPLINE_EINVAL;
  if ((flags & SPLINE_PATH_FUSED) && (flags & SPLINE_PATH_SPLIT)) return SPLINE_EINVAL;
  if (batch == 0) return SPLINE_OK;
  if (!x || !y || ((bc & 1) && !yp1) || ((bc & 2) && !ypn)) return SPLINE_EINVAL;
  if (m > 0 && (!q || !out)) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return build_eval_host_t<float>((const float *)x, (const float *)y, n, batch, bc, (const float *)yp1,
                                    (const float *)ypn, (float *)y2, (const float *)q, m, (float *)out, idx, flags, st);
  return build_eval_host_t<double>((const double *)x, (const double *)y, n, batch, bc, (const double *)yp1,
                                   (const double *)ypn, (double *)y2, (const double *)q, m, (double *)out, idx, flags,
                                   st);
}

int spline_eval_ablation(const void *x, const void *y, const void *y2, int64_t n, int64_t batch, const void *q,
                         int64_t m, void *out, int32_t *idx, int form, int dtype, spline_stream_t stream) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || batch < 0 || m < 0 || m >= (int64_t(1) << 31)) return SPLINE_EINVAL;
  if (form < SPLINE_FORM_RECORD || form > SPLINE_FORM_NOOP) return SPLINE_EINVAL;
  if (batch == 0 || m == 0) return SPLINE_OK;
  if (!x || !y || !y2 || !q || !out) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return ablation_t<float>((const float *)x, (const float *)y, (const float *)y2, n, batch, (const float *)q, m,
                             (float *)out, idx, form, st);
  return ablation_t<double>((const double *)x, (const double *)y, (const double *)y2, n, batch, (const double *)q, m,
                            (double *)out, idx, form, st);
}

int spline_gather_probe(const void *x, const void *y, const void *y2, int64_t n, int64_t batch, const void *q,
                        int64_t m, const int32_t *idx_in, void *out, int32_t *idx, int mode, int dtype,
                        spline_stream_t stream) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || batch < 0 || m < 0 || (mode != 0 && mode != 1)) return SPLINE_EINVAL;
  if (batch == 0 || m == 0) return SPLINE_OK;
  if (!x || !y || !y2 || !q || !idx_in || !out || !idx) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return probe_t<float>((const float *)x, (const float *)y, (const float *)y2, n, batch, (const float *)q, m,
                          idx_in, (float *)out, idx, mode, st);
  return probe_t<double>((const double *)x, (const double *)y, (const double *)y2, n, batch, (const double *)q, m,
                         idx_in, (double *)out, idx, mode, st);
}

int spline_build_f32(const float *x, const float *y, int64_t n, int64_t batch, int bc, const float *yp1,
                     const float *ypn, float *y2, spline_stream_t stream) {
  return spline_build(x, y, n, batch, bc, yp1, ypn, y2, SPLINE_F32, stream);
}
int spline_build_f64(const double *x, const double *y, int64_t n, int64_t batch, int bc, const double *yp1,
                     const double *ypn, double *y2, spline_stream_t stream) {
  return spline_build(x, y, n, batch, bc, yp1, ypn, y2, SPLINE_F64, stream);
}
int spline_eval_f32(const float *x, const float *y, const float *y2, int64_t n, int64_t batch, const float *q,
                    int64_t m, float *out, int32_t *idx, int flags, spline_stream_t stream) {
  return spline_eval(x, y, y2, n, batch, q, m, out, idx, flags, SPLINE_F32, stream);
}
int spline_eval_f64(const double *x, const double *y, const double *y2, int64_t n, int64_t batch, const double *q,
                    int64_t m, double *out, int32_t *idx, int flags, spline_stream_t stream) {
  return spline_eval(x, y, y2, n, batch, q, m, out, idx, flags, SPLINE_F64, stream);
}

int spline_status(spline_stream_t stream, unsigned int *bits_out) {
  cudaStream_t st = (cudaStream_t)stream;
  unsigned int bits = 0;
  unsigned *w = status_word(st);
  if (!w) return SPLINE_ENOMEM;
  // read, then clear, this stream's word -- both ordered on the stream after its prior work
  cudaError_t e = cudaMemcpyAsync(&bits, w, sizeof(bits), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(w, 0, sizeof(unsigned), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (bits_out) *bits_out = bits;
  return cuda_rc(e);
}

size_t spline_spike_workspace_size(int64_t n, int64_t row_begin, int64_t row_end, int dtype) {
  (void)n;
  const int R = dtype == SPLINE_F64 ? rmax<double>() : rmax<float>();
  const int64_t ntiles = (row_end - row_begin + 256 * R - 1) / (256 * R);
  return dtype == SPLINE_F64 ? spike_ws_layout<double>(ntiles, 1, nullptr, nullptr)
                             : spike_ws_layout<float>(ntiles, 1, nullptr, nullptr);
}


int spline_spike_reduce(const void *x, const void *y, int64_t n, int64_t row_begin, int64_t row_end, int bc,
                        const void *yp1, const void *ypn, void *record, void *workspace, int dtype,
                        spline_stream_t stream) {
  if (int rc = check_spike(x, y, n, row_begin, row_end, bc, yp1, ypn, workspace, dtype)) return rc;
  if (!record) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return spike_reduce_t<float>((const float *)x, (const float *)y, n, row_begin, row_end, bc, (const float *)yp1,
                                 (const float *)ypn, (float *)record, workspace, st);
  return spike_reduce_t<double>((const double *)x, (const double *)y, n, row_begin, row_end, bc,
                                (const double *)yp1, (const double *)ypn, (double *)record, workspace, st);
}

int spline_spike_finish(const void *x, const void *y, int64_t n, int64_t row_begin, int64_t row_end, int bc,
                        const void *yp1, const void *ypn, const void *all_records, int nranks, int rank,
                        void *y2_shard, void *workspace, int dtype, spline_stream_t stream) {
  if (int rc = check_spike(x, y, n, row_begin, row_end, bc, yp1, ypn, workspace, dtype)) return rc;
  if (!all_records || !y2_shard || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return spike_finish_t<float>((const float *)x, (const float *)y, n, row_begin, row_end, bc, (const float *)yp1,
                                 (const float *)ypn, (const float *)all_records, nranks, rank, (float *)y2_shard,
                                 workspace, st);
  return spike_finish_t<double>((const double *)x, (const double *)y, n, row_begin, row_end, bc,
                                (const double *)yp1, (const double *)ypn, (const double *)all_records, nranks, rank,
                                (double *)y2_shard, workspace, st);
}

int64_t spline_spike_tile_rows(int dtype) { return 256 * (dtype == SPLINE_F64 ? rmax<double>() : rmax<float>()); }

int spline_spike_tile_records(const void *x, const void *y, int64_t n, int64_t row_begin, int64_t row_end, int bc,
                              const void *yp1, const void *ypn, void *tile_records, void *workspace, int dtype,
                              spline_stream_t stream) {
  if (int rc = check_spike(x, y, n, row_begin, row_end, bc, yp1, ypn, workspace, dtype)) return rc;
  if (!tile_records || row_begin % spline_spike_tile_rows(dtype) != 0) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return spike_tile_records_t<float>((const float *)x, (const float *)y, n, row_begin, row_end, bc,
                                       (const float *)yp1, (const float *)ypn, (float *)tile_records, workspace, st);
  return spike_tile_records_t<double>((const double *)x, (const double *)y, n, row_begin, row_end, bc,
                                      (const double *)yp1, (const double *)ypn, (double *)tile_records, workspace, st);
}

int spline_spike_finish_tiles(const void *x, const void *y, int64_t n, int bc, const void *yp1, const void *ypn,
                              const void *all_tile_records, void *y2, void *workspace, int dtype,
                              spline_stream_t stream) {
  if (int rc = check_spike(x, y, n, 0, n, bc, yp1, ypn, workspace, dtype)) return rc;
  if (!all_tile_records || !y2) return SPLINE_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return spike_finish_tiles_t<float>((const float *)x, (const float *)y, n, bc, (const float *)yp1,
                                       (const float *)ypn, (const float *)all_tile_records, (float *)y2, workspace, st);
  return spike_finish_tiles_t<double>((const double *)x, (const double *)y, n, bc, (const double *)yp1,
                                      (const double *)ypn, (const double *)all_tile_records, (double *)y2, workspace,
                                      st);
}

int spline_build_dist(const void *x, const void *y, int64_t n, int bc, const void *yp1, const void *ypn,
                      void *y2_shard, spline_nccl_comm_t comm, int dtype, spline_stream_t stream) {
  if (dtype != SPLINE_F32 && dtype != SPLINE_F64) return SPLINE_EINVAL;
  if (n < 3 || n >= (int64_t(1) << 31) || bc < 0 || bc > 3) return SPLINE_EINVAL;
  if (!x || !y || !y2_shard || !comm || ((bc & 1) && !yp1) || ((bc & 2) && !ypn)) return SPLINE_EINVAL;
  if (!nccl_api().ok) return SPLINE_ENCCL;
  cudaStream_t st = (cudaStream_t)stream;
  StatusScope scope(st);
  if (!scope.ok()) return SPLINE_ENOMEM;
  if (dtype == SPLINE_F32)
    return build_dist_t<float>((const float *)x, (const float *)y, n, bc, (const float *)yp1, (const float *)ypn,
                               (float *)y2_shard, (void *)comm, st);
  return build_dist_t<double>((const double *)x, (const double *)y, n, bc, (const double *)yp1, (const double *)ypn,
                              (double *)y2_shard, (void *)comm, st);
}
int spline_build_dist_f32(const float *x, const float *y, int64_t n, int bc, const float *yp1, const float *ypn,
                          float *y2_shard, spline_nccl_comm_t comm, spline_stream_t stream) {
  return spline_build_dist(x, y, n, bc, yp1, ypn, y2_shard, comm, SPLINE_F32, stream);
}
int spline_build_dist_f64(const double *x, const double *y, int64_t n, int bc, const double *yp1, const double *ypn,
                          double *y2_shard, spline_nccl_comm_t comm, spline_stream_t stream) {
  return spline_build_dist(x, y, n, bc, yp1, ypn, y2_shard, comm, SPLINE_F64, stream);
}

const char *spline_version(void) { return "fastspline-b200 0.2 (sm_100a)"; }

#if FS_TILE_PHASES
// Diagnostic build only: the accumulated per-phase SM cycles of tile_solve (thread 0 of every
// tile), copied to out[0..7] and reset.
int spline_debug_tile_phases(unsigned long long *out) {
  if (cudaMemcpyFromSymbol(out, g_tile_phase, sizeof(unsigned long long) * 8) != cudaSuccess) return SPLINE_ECUDA;
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (cudaMemcpyToSymbol(g_tile_phase, z, sizeof(z)) != cudaSuccess) return SPLINE_ECUDA;
  return SPLINE_OK;
}
#endif
}  // extern "C"
