// common.cuh -- small device helpers shared by the sm_100a kernels of libfastspline.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fs {

// Data-error bits (see spline_status in include/spline.h).  Every kernel receives the
// launching stream's status word (`status`, a device pointer chosen by the host per stream),
// so bits raised on one stream never reach another stream's spline_status.
constexpr unsigned kBadKnots = 1u;
constexpr unsigned kOutOfRange = 2u;

__device__ __forceinline__ void raise_status(unsigned *status, unsigned bits) { atomicOr(status, bits); }

// Warp-aggregated status raise: one atomic per warp at most.
__device__ __forceinline__ void raise_status_warp(unsigned *status, bool pred, unsigned bits) {
  unsigned mask = __activemask();
  unsigned any = __ballot_sync(mask, pred);
  if (any && (threadIdx.x & 31) == (__ffs(mask) - 1)) atomicOr(status, bits);
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

template <typename T> __device__ __forceinline__ T qnan();
template <> __device__ __forceinline__ float qnan<float>() { return __int_as_float(0x7fc00000); }
template <> __device__ __forceinline__ double qnan<double>() { return __longlong_as_double(0x7ff8000000000000ll); }
template <typename T> __device__ __forceinline__ T inf_of();
template <> __device__ __forceinline__ float inf_of<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double inf_of<double>() { return __longlong_as_double(0x7ff0000000000000ll); }

template <typename T> __device__ __forceinline__ bool finite(T v) { return isfinite(v); }

// Unsigned division by a runtime constant d: floor(e / d) == __umulhi(e, M) with
// M = ceil(2^32 / d), exact whenever e * d < 2^32 (M = (2^32 + r)/d with r < d, so the
// rounding term e*r/(d*2^32) stays below 1/d).  Callers keep e * d < 2^32.
struct FastDiv {
  uint32_t d, M;
  __host__ __device__ FastDiv() : d(1), M(0) {}
  __host__ explicit FastDiv(uint32_t dd) : d(dd), M((uint32_t)((((uint64_t)1 << 32) + dd - 1) / dd)) {}
  __device__ __forceinline__ uint32_t div(uint32_t e) const { return d == 1 ? e : __umulhi(e, M); }
};

// Streaming (read-once) global loads / stores: do not pollute L1, evict early from L2.
__device__ __forceinline__ float ld_stream(const float *p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float *p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double *p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(int32_t *p, int32_t v) { __stcs(p, v); }

// Explicitly rounded arithmetic (no contraction freedom): every eval kernel and every
// hint produces bitwise-identical out for the same (interval, query).
__device__ __forceinline__ float r_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double r_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float r_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double r_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float r_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double r_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float r_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double r_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
// The interval records' 1/h (make_cub): fp32 rcp.approx (subnormal-preserving) + one Newton
// step, within ~1 ulp of 1/h -- the correctly rounded __frcp_rn costs a multi-instruction path
// per knot on the eval pack
__device__ __forceinline__ float r_rcp(float a) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return __fmaf_rn(r, __fmaf_rn(-a, r, 1.0f), r);
}
__device__ __forceinline__ double r_rcp(double a);  // fp64: rcp.approx + 2 Newton steps (below)

// Reciprocal for the solver sweeps: hardware approximation refined by Newton-Raphson
// (fp32: one step; fp64: two steps after the 23-bit MUFU seed), |relative error| <= ~1 ulp
// of the correctly rounded value, no special-case branch.  Only used on finite, normal,
// nonzero arguments (interval widths and pivots of a strictly diagonally dominant system).
__device__ __forceinline__ float nr_rcp(float a) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  const float e = __fmaf_rn(-a, r, 1.0f);
  return __fmaf_rn(r, e, r);
}
#ifndef FS_BUILD_RCP_RN
#define FS_BUILD_RCP_RN 0
#endif
__device__ __forceinline__ double nr_rcp(double a) {
#if FS_BUILD_RCP_RN
  return __drcp_rn(a);  // correctly rounded (A/B: DESIGN.md)
#else
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = __fma_rn(-a, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-a, r, 1.0);
  return __fma_rn(r, e, r);
#endif
}
// The eval kernels' fp64 reciprocal: the correctly rounded __drcp_rn costs a slow-path
// sequence per query in the sorted-run kernel; the Newton-refined seed is within ~1 ulp and is
// what every eval kernel uses (so all of them still give identical bits).
__device__ __forceinline__ double r_rcp(double a) { return nr_rcp(a); }

// Eq. nr_formula on one interval [x0, x1], in the factored form every eval kernel
// uses.  With h = x1 - x0, B = (q - x0)/h, A = 1 - B and zs_k = y2_k h^2/6:
//     A y0 + B y1 + (A^3 - A) zs0 + (B^3 - B) zs1
//       = y0 + B dy - B (1 - B) (e1 + B e2),   dy = y1 - y0, e1 = 2 zs0 + zs1, e2 = zs1 - zs0
// (A^3 - A = -B(1-B)(2-B), B^3 - B = -B(1-B)(1+B)).  Every factor is bounded like the NR
// terms (B, 1-B in [0, 1]), so it is as well conditioned as Eq. nr_formula (an expansion in
// powers of (q - x0) is not: its terms cancel catastrophically near x1 when y2 is large).
// An interval carries Cub {1/h, y0, dy, e1} (16 B fp32: one shared-memory vector load) and e2;
// x0 comes from the search.  1/h (the paper's inv_ba) is a Newton-refined reciprocal
// within ~1 ulp (r_rcp).  Every operation is explicitly rounded, so every kernel and hint gives
// the same bits.
template <typename T> struct Cub { T ih, y0, dy, e1; };

template <typename T>
__device__ __forceinline__ Cub<T> make_cub(T x0, T x1, T y0, T y1, T z0, T z1, T &e2) {
  const T h = r_sub(x1, x0);
  const T h26 = r_mul(r_mul(h, h), T(1) / T(6));
  const T zs0 = r_mul(z0, h26), zs1 = r_mul(z1, h26);
  e2 = r_sub(zs1, zs0);
  return Cub<T>{r_rcp(h), y0, r_sub(y1, y0), r_fma(T(2), zs0, zs1)};
}

template <typename T> __device__ __forceinline__ T cub_eval(const Cub<T> &c, T e2, T x0, T q) {
  const T B = r_mul(r_sub(q, x0), c.ih);
  const T w = r_mul(B, r_sub(T(1), B));
  const T lin = r_fma(B, c.dy, c.y0);
  return r_fma(-w, r_fma(B, e2, c.e1), lin);
}

// Interval record of the long-curve path (HBM): the bracket [x0, x1] and the cubic
// (32 B fp32 / 64 B fp64: one or two 256-bit accesses).
template <typename T> struct Ival { T x0, x1, ih, y0, dy, e1, e2, pad; };

template <typename T> __device__ __forceinline__ Ival<T> make_ival(T x0, T x1, T y0, T y1, T z0, T z1) {
  T e2;
  const Cub<T> c = make_cub<T>(x0, x1, y0, y1, z0, z1, e2);
  return Ival<T>{x0, x1, c.ih, c.y0, c.dy, c.e1, e2, T(0)};
}

template <typename T> __device__ __forceinline__ T ival_interp(const Ival<T> &r, T q) {
  return cub_eval<T>(Cub<T>{r.ih, r.y0, r.dy, r.e1}, r.e2, r.x0, q);
}

// ---- the paper's evaluation variants (the division ablation) -------
// All compute Eq. nr_formula on [x0, x1]; they differ only in where the
// divisions are.  IEEE division (no -use_fast_math); contraction allowed.
enum { FORM_RECORD = 0,        // the product: the factored form of make_cub / cub_eval
       FORM_SPLINT_DIV = 1,    // NR splint: A, B divide by h, C, D divide by 6
       FORM_SPLINT_MUL = 2,    // same, /6 replaced by *(1/6)
       FORM_NEWINT_ORIG = 3,   // newint: one reciprocal inv_ba, multiplied at the end
       FORM_NEWINT_NOINV = 4,  // newint with the final multiply replaced by / ba
       FORM_NOOP = 5 };        // locate only, out = y_j (the paper's no-op loop)

template <typename T, int FORM>
__device__ __forceinline__ T interp_form(T q, T x0, T x1, T y0, T y1, T z0, T z1) {
  if constexpr (FORM == FORM_RECORD) {
    T e2;
    const Cub<T> c = make_cub<T>(x0, x1, y0, y1, z0, z1, e2);
    return cub_eval<T>(c, e2, x0, q);
  } else if constexpr (FORM == FORM_SPLINT_DIV || FORM == FORM_SPLINT_MUL) {
    const T h = x1 - x0;
    const T A = (x1 - q) / h, B = (q - x0) / h;
    const T cd = (A * A * A - A) * z0 + (B * B * B - B) * z1;
    if constexpr (FORM == FORM_SPLINT_DIV) return A * y0 + B * y1 + cd * (h * h) / T(6);
    else return A * y0 + B * y1 + cd * (h * h) * (T(1) / T(6));
  } else if constexpr (FORM == FORM_NEWINT_ORIG || FORM == FORM_NEWINT_NOINV) {
    const T ba = x1 - x0, xa = q - x0, bx = x1 - q, ba2 = ba * ba;
    const T lower = xa * y1 + bx * y0;
    const T C = (xa * xa - ba2) * xa * z1;
    const T D = (bx * bx - ba2) * bx * z0;
    if constexpr (FORM == FORM_NEWINT_ORIG) {
      const T inv_ba = T(1) / ba;
      return (lower + (T(1) / T(6)) * (C + D)) * inv_ba;
    } else {
      return (lower + (T(1) / T(6)) * (C + D)) / ba;
    }
  } else {
    return y0;
  }
}

// From the raw arrays (kernels that do not stage the curve).
template <typename T>
__device__ __forceinline__ T nr_interp(T q, T x0, T x1, T y0, T y1, T z0, T z1) {
  T e2;
  const Cub<T> c = make_cub<T>(x0, x1, y0, y1, z0, z1, e2);
  return cub_eval<T>(c, e2, x0, q);
}

// Shared-knot mode (SPLINE_X_SHARED) for kernels that read a knot row per curve: the one
// knot vector broadcast into a [batch][n] scratch (row r = x).  out[i] = x[i mod n].
template <typename T>
__global__ void __launch_bounds__(256) k_broadcast_rows(const T *__restrict__ x, int64_t n, int64_t total,
                                                        T *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(x + i % n);
}

}  // namespace fs

namespace fs {

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on a shared-memory mbarrier.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// Programmatic dependent launch (PDL): a build kernel lets the next kernel of the stream be
// scheduled before it finishes (pdl_trigger, at its start: the dependent's CTAs then launch as
// the build's CTAs drain, all of which have started); an eval kernel waits for its predecessor
// to complete -- with all memory visible -- before reading x, y, y2 (pdl_wait).  Both are
// no-ops when the launch carries no programmatic dependency.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Plain arrival (release semantics) on an mbarrier.
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Orders this thread's earlier generic-proxy shared-memory accesses before later async-proxy
// (TMA) accesses, e.g. before a bulk copy overwrites a stage that was read.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One lane per warp arrives on a shared counter of `nwarps` arrivals; returns true (to that
// lane) for the last arrival, after resetting the counter.  Used to let the last warp done
// with a stage issue its refill without any warp waiting for the others.
__device__ __forceinline__ bool last_warp_arrival(int *counter, int nwarps) {
  __threadfence_block();
  const int old = atomicAdd(counter, 1);
  __threadfence_block();
  if (old == nwarps - 1) {
    *counter = 0;
    return true;
  }
  return false;
}

// try_wait suspends the thread until the phase completes or this many ns pass, so waiting
// warps do not spin through the issue slots of the working ones
constexpr uint32_t kMbarSuspendNs = 1000000;
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase), "r"(kMbarSuspendNs)
        : "memory");
  } while (!done);
}

// Global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bulk prefetch of [p, p + bytes) into L2 (cp.async.bulk.prefetch.L2; p 16-byte aligned, bytes a
// multiple of 16).
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// ---- 16-byte vector types per element type
template <typename T> struct Vec16;
template <> struct Vec16<float> { using V = float4; using I = int4; static constexpr int N = 4; };
template <> struct Vec16<double> { using V = double2; using I = int2; static constexpr int N = 2; };

// 32-byte (256-bit) streaming accesses: one instruction per full sector (LDG.E.256 / STG.E.256)
__device__ __forceinline__ void ld_cs_256(const double *p, double *v) {
  asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld_cs_256(const float *p, float *v) {
  asm volatile("ld.global.cs.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void st_cs_256(double *p, const double *v) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}
__device__ __forceinline__ void st_cs_256(float *p, const float *v) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void st_cs_256(int32_t *p, const int *v) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

template <typename T, int V> struct VecIO {
  // loads V consecutive elements (16-byte aligned when V > 1; 32-byte aligned when V elements
  // are 32 bytes)
  static __device__ __forceinline__ void load(const T *p, T *v) {
    if constexpr (V == 1) {
      v[0] = ld_stream(p);
    } else if constexpr (V * sizeof(T) == 32) {
      ld_cs_256(p, v);
    } else {
      using VT = typename Vec16<T>::V;
      const VT t = __ldcs(reinterpret_cast<const VT *>(p));
      const T *tt = reinterpret_cast<const T *>(&t);
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = tt[i];
    }
  }
  static __device__ __forceinline__ void load_shared(const T *p, T *v) {
    if constexpr (V == 1) {
      v[0] = p[0];
    } else {
      using VT = typename Vec16<T>::V;
      const VT t = *reinterpret_cast<const VT *>(p);
      const T *tt = reinterpret_cast<const T *>(&t);
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = tt[i];
    }
  }
  static __device__ __forceinline__ void store(T *p, const T *v) {
    if constexpr (V == 1) {
      st_stream(p, v[0]);
    } else if constexpr (V * sizeof(T) == 32) {
      st_cs_256(p, v);
    } else {
      using VT = typename Vec16<T>::V;
      VT t;
      T *tt = reinterpret_cast<T *>(&t);
#pragma unroll
      for (int i = 0; i < V; ++i) tt[i] = v[i];
      __stcs(reinterpret_cast<VT *>(p), t);
    }
  }
  static __device__ __forceinline__ void store_idx(int32_t *p, const int *j) {
    if constexpr (V == 1) {
      st_stream(p, j[0]);
    } else if constexpr (V == 8) {
      st_cs_256(p, j);
    } else if constexpr (V == 4) {
      __stcs(reinterpret_cast<int4 *>(p), make_int4(j[0], j[1], j[2], j[3]));
    } else {
      __stcs(reinterpret_cast<int2 *>(p), make_int2(j[0], j[1]));
    }
  }
};

}  // namespace fs
