// Streaming ceiling of the sorted-eval traffic (read q 8 B, write out 8 B + idx 4 B per query) for
// two work distributions: grid-stride (all warps in one moving window) and per-warp contiguous
// runs of R queries (the k_eval_sorted task layout: each warp walks its own run).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_chunk_probe stream_chunk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double4 ld4(const double4 *p) {
  double4 v;
  asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(double4 *p, double4 v) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
__global__ void __launch_bounds__(256) k_grid(const double4 *__restrict__ q, double4 *__restrict__ out,
                                              int4 *__restrict__ idx, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    double4 v = ld4(q + i);
    st4(out + i, v);
    __stcs(idx + i, make_int4((int)v.x, (int)v.y, (int)v.z, (int)v.w));
  }
}
// warp task t (grid-stride over tasks) walks queries [t R, (t+1) R), 128 per step (4 per lane)
__global__ void __launch_bounds__(256) k_runs(const double4 *__restrict__ q, double4 *__restrict__ out,
                                              int4 *__restrict__ idx, int64_t n4, int64_t run4) {
  const int lane = threadIdx.x & 31;
  const int64_t ntask = (n4 + run4 - 1) / run4;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntask; t += nw) {
    const int64_t e = (t + 1) * run4 < n4 ? (t + 1) * run4 : n4;
    for (int64_t i = t * run4 + lane; i < e; i += 32) {
      double4 v = ld4(q + i);
      st4(out + i, v);
      __stcs(idx + i, make_int4((int)v.x, (int)v.y, (int)v.z, (int)v.w));
    }
  }
}
int main() {
  const int64_t n = int64_t(1) << 28, n4 = n / 4;  // cfg4's 268M queries
  double4 *q, *out; int4 *idx;
  cudaMalloc(&q, n * 8); cudaMalloc(&out, n * 8); cudaMalloc(&idx, n * 4);
  cudaMemset(q, 0, n * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)n * 20;
  auto run = [&](const char *name, auto launch) {
    for (int i = 0; i < 2; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-34s %.3f ms  %.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  run("grid-stride, 4 CTAs x 256 / SM", [&] { k_grid<<<sms * 4, 256>>>(q, out, idx, n4); });
  for (int64_t R : {1024, 2048, 8192, 32768}) {
    char nm[64]; snprintf(nm, 64, "per-warp runs of %lld queries", (long long)R);
    run(nm, [&] { k_runs<<<sms * 4, 256>>>(q, out, idx, n4, R / 4); });
  }
  return 0;
}
