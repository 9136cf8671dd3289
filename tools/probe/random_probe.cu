// Random-access ceiling of this B200's memory system (an independent ceiling for the
// long-curve evaluation, not the library's own gather).  A 4 GiB array; every thread issues U
// independent loads of W bytes (32 = one sector, 64 = two) at pseudo-random W-aligned offsets
// (a counter hash, no dependence between loads), at full occupancy; reports random accesses/s
// and bytes/s -- over the whole array (DRAM-bound) and over an L2-sized window (24 MB, the
// bucketed evaluation's chunk: L2-bound).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o random_probe random_probe.cu && ./random_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t z) {  // splitmix64 finaliser
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <int W, int U>
__global__ void __launch_bounds__(256) k_random(const double *__restrict__ a, uint64_t nblk, uint64_t seed,
                                                int iters, double *__restrict__ sink) {
  constexpr int E = W / 8;  // doubles per access
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double v[U][E];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t b = mix(seed + (tid * iters + it) * U + u) % nblk;
      const double *p = a + b * E;
      if constexpr (E == 4) {
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3]) : "l"(p));
      } else {
#pragma unroll
        for (int h = 0; h < E / 4; ++h)
          asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                       : "=d"(v[u][4 * h]), "=d"(v[u][4 * h + 1]), "=d"(v[u][4 * h + 2]), "=d"(v[u][4 * h + 3])
                       : "l"(p + 4 * h));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < E; ++e) acc += v[u][e];
  }
  if (acc == 1.2345) sink[0] = acc;  // keeps the loads alive
}

template <int W, int U> double run(const double *a, uint64_t bytes, int sms) {
  const uint64_t nblk = bytes / W;
  const int blocks = sms * 8, iters = 64;
  double *sink;
  cudaMalloc(&sink, 8);
  k_random<W, U><<<blocks, 256>>>(a, nblk, 1, 4, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_random<W, U><<<blocks, 256>>>(a, nblk, 7, iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(sink);
  return (double)blocks * 256 * iters * U / (ms * 1e-3);  // accesses per second
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t big = 4ull << 30, chunk = 24ull << 20;
  double *a;
  if (cudaMalloc(&a, big) != cudaSuccess) return 1;
  cudaMemset(a, 0, big);
  printf("{\"probe\": \"random_access\", \"sms\": %d, \"results\": [", sms);
  const char *sep = "";
  auto rep = [&](const char *what, int W, uint64_t region, double acc) {
    printf("%s{\"region_bytes\": %llu, \"access_bytes\": %d, \"what\": \"%s\", \"accesses_per_s\": %.4g, "
           "\"GB_per_s\": %.1f}", sep, (unsigned long long)region, W, what, acc, acc * W / 1e9);
    sep = ", ";
  };
  rep("4 GiB array (DRAM)", 32, big, run<32, 8>(a, big, sms));
  rep("4 GiB array (DRAM)", 64, big, run<64, 8>(a, big, sms));
  rep("24 MB window (L2)", 32, chunk, run<32, 8>(a, chunk, sms));
  rep("24 MB window (L2)", 64, chunk, run<64, 8>(a, chunk, sms));
  printf("]}\n");
  cudaFree(a);
  return 0;
}
