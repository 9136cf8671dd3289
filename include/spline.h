/*
 * spline.h -- C ABI of the B200-native cubic-spline library (libfastspline.so).
 *
 * The hot path of Hornbeck, "Fast Cubic Spline Interpolation" (arXiv 2001.09253):
 *   construction  -- the knot second derivatives y2 ("y''") solve the tridiagonal
 *                    system of Eq. init_val with natural ends
 *                    (y2 = 0) or clamped ends
 *                    (P:955-971 start row; P:1017-1018 end row);
 *   evaluation    -- each query q is located in its knot interval j and the cubic
 *                    of Eq. nr_formula is applied.
 *
 * Conventions (all entry points):
 *   - Every array argument is a DEVICE pointer owned by the caller (e.g. a torch
 *     CUDA tensor's data_ptr()), C-contiguous and curve-major: x, y, y2 are
 *     [batch][n]; q, out, idx are [batch][m]; yp1, ypn are [batch].  Element type
 *     is float (SPLINE_F32) or double (SPLINE_F64), selected by `dtype` or by the
 *     _f32/_f64 wrapper.  idx is int32 (0-based interval index).
 *   - All curves of one call share n, and all share m (ragged batches: one call
 *     per (n, m) group).
 *   - Work is enqueued on `stream` (NULL = the legacy default stream) and the call
 *     returns without synchronising.  The library is re-entrant; the only shared
 *     mutable state is the per-stream data-error words read by spline_status() (one device
 *     word per stream handle, allocated on a device's first call: make one call, e.g.
 *     spline_status, before capturing a CUDA graph).
 *   - Temporary workspace (long-curve SPIKE records; y2 scratch of an unfused
 *     spline_build_eval called without y2) comes from a library-owned stream-ordered
 *     memory pool per device (cudaMallocFromPoolAsync on `stream`) that keeps its
 *     memory between calls.
 *
 * Errors:
 *   - Argument errors are synchronous: the call returns SPLINE_EINVAL and enqueues
 *     nothing (NULL required pointer, n < 3 [P:746, P:1047], batch < 0, m < 0,
 *     unknown bc/dtype, NULL yp1/ypn for a clamped end, n or m >= 2^31).
 *     batch == 0 or m == 0 is a valid no-op.
 *   - CUDA launch/allocation failures return SPLINE_ECUDA / SPLINE_ENOMEM.
 *   - Data errors are asynchronous (cuSOLVER devInfo pattern) and OR'ed into the
 *     launching stream's status word, read (and cleared) by spline_status(stream):
 *       SPLINE_STATUS_BAD_KNOTS: a curve's knots are not strictly increasing or a
 *         value/slope is not finite; that curve's y2 is all NaN.
 *       SPLINE_STATUS_Q_OUT_OF_RANGE: a query is outside [x_0, x_{n-1}] or NaN
 *         (Eq. nr_formula requires x_j <= x <= x_{j+1}); its idx is -1 and
 *         its out is NaN.  No extrapolation.
 */
#ifndef FASTSPLINE_SPLINE_H
#define FASTSPLINE_SPLINE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *spline_stream_t; /* identical to cudaStream_t */
typedef struct ncclComm *spline_nccl_comm_t; /* identical to ncclComm_t (nccl.h) */

enum { SPLINE_F32 = 0, SPLINE_F64 = 1 };
enum { SPLINE_OK = 0, SPLINE_EINVAL = -1, SPLINE_ECUDA = -2, SPLINE_ENOMEM = -3, SPLINE_ENCCL = -4 };
/* Boundary condition: a bitmask, the two ends are independent (the paper tests
 * its natural-end sentinel separately per end).  The 0.99e30
 * sentinel itself is never interpreted by the library. */
enum {
  SPLINE_BC_NATURAL = 0,     /* y2_0 = y2_{n-1} = 0 */
  SPLINE_BC_CLAMP_START = 1, /* y'(x_0) = yp1[c]: 2h_0 y2_0 + h_0 y2_1 = 6(dd_0 - yp1) */
  SPLINE_BC_CLAMP_END = 2,   /* y'(x_{n-1}) = ypn[c]: h y2_{n-2} + 2h y2_{n-1} = 6(ypn - dd_{n-2}) */
  SPLINE_BC_CLAMPED = 3
};
/* Evaluation hints: may change speed, never results (every guess is corrected by
 * comparisons against the same locate rule).  SPLINE_PATH_* (spline_build_eval only) pick
 * the fused single kernel or the two kernels instead of the library's choice; both give
 * bitwise the same y2, out and idx. */
/* SPLINE_NO_BUCKET (spline_eval only): on one curve too long for L2 with many unsorted queries, do
 * not bucket the queries by curve chunk (eval_bucket.cuh); use the one-gather-per-query record
 * path instead (measurement and A/B; same results bitwise). */
/* SPLINE_X_SHARED (shared-knot mode): every curve of the batch has the SAME knots; x is then ONE
 * row [n] (not [batch][n]).  Given in `bc` of spline_build and in `flags` of spline_eval /
 * spline_build_eval / spline_build_eval_host.  The paper evaluates on one grid right after the
 * build; BASELINE cfg3's grid is one uniform grid.  Native (knots read once per
 * curve tile, not per curve) in the short-curve kernels (n <= 8: K1r, and k_eval_small for fp32
 * with m <= 32); other shapes broadcast the row into stream-ordered scratch first.  Results are
 * bitwise those of the same call with the row repeated per curve. */
enum { SPLINE_Q_SORTED = 1, SPLINE_X_UNIFORM = 2, SPLINE_PATH_FUSED = 4, SPLINE_PATH_SPLIT = 8, SPLINE_NO_BUCKET = 16,
       SPLINE_X_SHARED = 32 };
/* Asynchronous data-error bits (spline_status). */
enum { SPLINE_STATUS_BAD_KNOTS = 1, SPLINE_STATUS_Q_OUT_OF_RANGE = 2 };

/*
 * spline_build -- knot second derivatives for `batch` independent curves.
 *   x, y   [batch][n] knots (strictly increasing per curve) and values.
 *   bc     SPLINE_BC_* bitmask; yp1 / ypn are [batch] end slopes, required
 *          (non-NULL) iff that end is clamped, ignored otherwise.
 *   y2     [batch][n] output: the unique solution of the (strictly diagonally
 *          dominant) tridiagonal system; natural ends are exactly 0.
 * Kernels by n: <= 128 batched Thomas (one thread per curve);
 * <= 4096 (f64) / 8192 (f32) one CTA per curve (partition + merge tree);
 * longer: tiled SPIKE (tile records -> reduced solve -> finish).
 */
int spline_build(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1,
                 const void *ypn, void *y2, int dtype, spline_stream_t stream);

/*
 * spline_eval -- fused locate + evaluate.
 *   x, y, y2  [batch][n] as produced/consumed by spline_build.
 *   q         [batch][m] queries of curve c are q[c*m .. c*m+m-1].
 *   out       [batch][m] Eq. nr_formula at q on interval idx.
 *   idx       [batch][m] int32, nullable: the largest j in [0, n-2] with
 *             x_j <= q (so a query on an interior knot x_k gets k, q = x_{n-1}
 *             gets n-2); -1 if q is outside [x_0, x_{n-1}] or NaN.
 *   flags     SPLINE_Q_SORTED | SPLINE_X_UNIFORM hints (speed only).
 */
int spline_eval(const void *x, const void *y, const void *y2, int64_t n, int64_t batch, const void *q,
                int64_t m, void *out, int32_t *idx, int flags, int dtype, spline_stream_t stream);

/*
 * spline_build_eval -- construction and evaluation in one call: the same y2, out and
 * idx (bitwise) as spline_build followed by spline_eval on the same stream.
 *   x, y, bc, yp1, ypn   as spline_build.
 *   y2                   [batch][n] output, NULLABLE: NULL = do not write y2 (it then never
 *                        leaves the chip on the fused path).
 *   q, m, out, idx       as spline_eval (q and out required when m > 0; idx nullable).
 *   flags                SPLINE_Q_SORTED | SPLINE_X_UNIFORM | SPLINE_PATH_* hints (speed only).
 * The fused kernel (one launch; x, y read once from HBM, y2 produced and consumed on chip:
 * SURVEY.md §8(f) row 1, the paper evaluating right after the build) runs when
 * 3 <= n <= 128, n*sizeof(T) % 16 == 0, m % (16/sizeof(T)) == 0 and x, y, y2, q, out are
 * 16-byte aligned (idx 16-byte aligned for f32, 8-byte for f64); otherwise the two kernels run
 * back to back (with stream-ordered scratch for y2 when y2 is NULL).  Without a PATH hint the
 * library fuses only launch-latency-bound problems (batch*m <= 2^17): on B200 the larger
 * staged evaluations are bound by shared-memory bandwidth, which fusion does not relieve
 * (measured: DESIGN.md).  Also without a hint: a few curves of n = 16 (or fp32 n = 32, 64)
 * run in one CTA per curve, and fp32 curves of n <= 8 with m <= 32 queries (m % 4 == 0) in
 * one solve+eval kernel -- the same results bitwise.  m == 0 builds only.
 * Errors: the union of spline_build's and spline_eval's.
 */
int spline_build_eval(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1,
                      const void *ypn, void *y2, const void *q, int64_t m, void *out, int32_t *idx, int flags,
                      int dtype, spline_stream_t stream);

/*
 * spline_build_eval_host -- spline_build_eval on HOST-resident arrays (same arguments, same
 * results bitwise, every pointer a host pointer; y2 and idx nullable).  The batch is cut into
 * chunks of whole curves that flow through internal streams: one chunk's host->device copy,
 * another's kernels and a third's device->host copy overlap.  Pinned (page-locked) host memory
 * gives the overlap; pageable memory works but serialises the copies.  Device scratch comes
 * from the library pool.  Ordered after prior work on `stream`; `stream` waits for the whole
 * call (synchronise it before reading the outputs).  The fused/split choice is the whole
 * problem's.  Errors: as spline_build_eval.
 */
int spline_build_eval_host(const void *x, const void *y, int64_t n, int64_t batch, int bc, const void *yp1,
                           const void *ypn, void *y2, const void *q, int64_t m, void *out, int32_t *idx, int flags,
                           int dtype, spline_stream_t stream);

/*
 * spline_eval_ablation -- the paper's evaluation-variant experiment on the GPU (SURVEY.md
 * §8(f) row 2): spline_eval's sorted-run kernel (every
 * query located by the carried-bracket scan, valid for any query order) with
 * the interpolation arithmetic replaced by
 *   SPLINE_FORM_RECORD       the product's form (1/h per interval, records; = spline_eval bits)
 *   SPLINE_FORM_SPLINT_DIV   Eq. nr_formula literally: A, B divided by h, C, D divided by 6
 *   SPLINE_FORM_SPLINT_MUL   the same with the /6 replaced by *(1/6)
 *   SPLINE_FORM_NEWINT_ORIG  the paper's newint: one 1/h, multiplied last
 *   SPLINE_FORM_NEWINT_NOINV newint dividing by h last instead
 *   SPLINE_FORM_NOOP         locate only, out = y_j (the paper's no-op loop)
 * Arguments and errors as spline_eval (flags are implied: sorted runs).  idx is exact for
 * every form; out meets the north-star tolerance for forms 0-4.
 */
enum { SPLINE_FORM_RECORD = 0, SPLINE_FORM_SPLINT_DIV = 1, SPLINE_FORM_SPLINT_MUL = 2, SPLINE_FORM_NEWINT_ORIG = 3,
       SPLINE_FORM_NEWINT_NOINV = 4, SPLINE_FORM_NOOP = 5 };
int spline_eval_ablation(const void *x, const void *y, const void *y2, int64_t n, int64_t batch, const void *q,
                         int64_t m, void *out, int32_t *idx, int form, int dtype, spline_stream_t stream);

/*
 * spline_gather_probe -- diagnostic: the random-gather ceiling of evaluation
 * on long curves.  With the intervals ALREADY KNOWN (idx_in [batch][m], e.g. spline_eval's
 * idx; -1 = out of range), evaluate without any search:
 *   mode 0: gather x_j, x_{j+1}, y_j, y_{j+1}, y2_j, y2_{j+1} from the three arrays;
 *   mode 1: build the interval records (as spline_eval does for long curves) and gather one
 *           record per query.
 * Writes out (the cubic; NaN where idx_in < 0) and idx (= idx_in).  Its time is what the
 * access pattern itself costs; spline_eval's long-curve path is reported against it.
 */
int spline_gather_probe(const void *x, const void *y, const void *y2, int64_t n, int64_t batch, const void *q,
                        int64_t m, const int32_t *idx_in, void *out, int32_t *idx, int mode, int dtype,
                        spline_stream_t stream);

/* Typed thin wrappers (same semantics). */
int spline_build_f32(const float *x, const float *y, int64_t n, int64_t batch, int bc, const float *yp1,
                     const float *ypn, float *y2, spline_stream_t stream);
int spline_build_f64(const double *x, const double *y, int64_t n, int64_t batch, int bc, const double *yp1,
                     const double *ypn, double *y2, spline_stream_t stream);
int spline_eval_f32(const float *x, const float *y, const float *y2, int64_t n, int64_t batch, const float *q,
                    int64_t m, float *out, int32_t *idx, int flags, spline_stream_t stream);
int spline_eval_f64(const double *x, const double *y, const double *y2, int64_t n, int64_t batch,
                    const double *q, int64_t m, double *out, int32_t *idx, int flags, spline_stream_t stream);

/* Synchronises `stream`, writes the OR of the data-error bits raised ON THIS STREAM since the
 * last call into *bits_out (host pointer) and clears them (other streams' words are untouched).
 * Returns SPLINE_OK, SPLINE_ECUDA or SPLINE_ENOMEM (the word could not be allocated). */
int spline_status(spline_stream_t stream, unsigned int *bits_out);

/*
 * Two-phase SPIKE seam for one long curve whose rows are partitioned across
 * ranks (the partition method with a merge tree of block
 * records).  Rank r owns rows [row_begin, row_end) of the n-row system and holds
 * the full x and y (replicated, device).  A block record is 6 values of dtype:
 *   (Gp, Vp, Wp, Gq, Vq, Wq) with y_p = Gp - Vp*y_{p-1} - Wp*y_{q+1} and
 *   y_q = Gq - Vq*y_{p-1} - Wq*y_{q+1} for the block's first row p and last row q.
 *
 * spline_spike_reduce: writes this rank's block record (6 values) to `record`.
 * The caller all-gathers the G records in rank order into `all_records` [G][6].
 * spline_spike_finish: solves the G-record reduced system redundantly, then writes
 *   y2 for rows [row_begin, row_end) into y2_shard[0 .. row_end-row_begin).
 * `workspace` (device, spline_spike_workspace_size bytes) must be the same buffer
 * for the reduce and finish calls of one rank.  bc/yp1/ypn as spline_build
 * (yp1/ypn point to one value each).  Data errors: as spline_build, per shard.
 */
size_t spline_spike_workspace_size(int64_t n, int64_t row_begin, int64_t row_end, int dtype);
int spline_spike_reduce(const void *x, const void *y, int64_t n, int64_t row_begin, int64_t row_end, int bc,
                        const void *yp1, const void *ypn, void *record, void *workspace, int dtype,
                        spline_stream_t stream);
int spline_spike_finish(const void *x, const void *y, int64_t n, int64_t row_begin, int64_t row_end, int bc,
                        const void *yp1, const void *ypn, const void *all_records, int nranks, int rank,
                        void *y2_shard, void *workspace, int dtype, spline_stream_t stream);

/*
 * Recompute instead of communicate -- the multi-GPU long-curve build that
 * leaves the FULL y2 on every rank without moving y2 between GPUs.  The curve's rows are cut in
 * tiles of spline_spike_tile_rows(dtype) rows from row 0 (the last tile ragged); rank r owns a
 * contiguous range of whole tiles.
 * spline_spike_tile_records: the block record (6 values, as above) of every tile of rows
 *   [row_begin, row_end) (row_begin a multiple of the tile rows; row_end a multiple or n), in
 *   tile order, to tile_records [ceil((row_end - row_begin) / tile_rows)][6].  The caller
 *   all-gathers them into the curve's full [ntiles][6] table.
 * spline_spike_finish_tiles: from that full table, the reduced solve and the finish of EVERY
 *   tile: writes y2[0 .. n).  workspace: spline_spike_workspace_size(n, 0, n, dtype) bytes.
 * A tile with bad knots has a NaN record: y2 is then NaN on every rank (BAD_KNOTS is raised by the
 * rank that owns the tile).
 */
int64_t spline_spike_tile_rows(int dtype);
int spline_spike_tile_records(const void *x, const void *y, int64_t n, int64_t row_begin, int64_t row_end, int bc,
                              const void *yp1, const void *ypn, void *tile_records, void *workspace, int dtype,
                              spline_stream_t stream);
int spline_spike_finish_tiles(const void *x, const void *y, int64_t n, int bc, const void *yp1, const void *ypn,
                              const void *all_tile_records, void *y2, void *workspace, int dtype,
                              spline_stream_t stream);

/*
 * spline_build_dist -- the second derivatives of ONE long curve whose rows are partitioned over
 * the G ranks of an NCCL communicator (the partitioned solve the paper points to
 * for parallel hardware).  Rank r = ncclCommUserRank(comm) owns rows
 * [r*n/G, (r+1)*n/G) (integer division) and writes their y2 to y2_shard[0 .. (r+1)*n/G - r*n/G).
 *   x, y     [n] the WHOLE curve on this rank's device (replicated input);
 *   bc       as spline_build; yp1 / ypn point to ONE value each (device), required iff clamped.
 *   comm     an initialised NCCL communicator whose ranks each call this function (collective);
 *            its device is the current device.
 * Steps, all enqueued on `stream`: the rank's rows reduced to one 6-scalar block record
 * (spline_spike_reduce), ncclAllGather of the G records (48 B per rank in fp64 -- the only
 * exchange), the G-record reduced system solved redundantly and the rank's rows finished
 * (spline_spike_finish).  Bitwise the two-phase seam's result.
 * Errors: SPLINE_EINVAL (bad arguments, NULL comm, more ranks than rows, G > 1024);
 * SPLINE_ENCCL (NCCL not loadable -- it is resolved at run time: the process's libnccl.so.2, or
 * the path in the SPLINE_NCCL_LIB environment variable -- or an NCCL call failed); data errors
 * as spline_build (BAD_KNOTS for this rank's rows; the whole curve's bad flag is per shard).
 */
int spline_build_dist(const void *x, const void *y, int64_t n, int bc, const void *yp1, const void *ypn,
                      void *y2_shard, spline_nccl_comm_t comm, int dtype, spline_stream_t stream);
int spline_build_dist_f32(const float *x, const float *y, int64_t n, int bc, const float *yp1, const float *ypn,
                          float *y2_shard, spline_nccl_comm_t comm, spline_stream_t stream);
int spline_build_dist_f64(const double *x, const double *y, int64_t n, int bc, const double *yp1, const double *ypn,
                          double *y2_shard, spline_nccl_comm_t comm, spline_stream_t stream);

/* Library version string (static storage). */
const char *spline_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FASTSPLINE_SPLINE_H */
