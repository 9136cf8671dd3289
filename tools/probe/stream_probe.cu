// Streaming ceiling for the sorted-eval traffic pattern: read q (8 B), write out (8 B) + idx (4 B)
// per query, 16-byte vectors, grid-stride.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) k_stream(const double2 *__restrict__ q, double2 *__restrict__ out,
                                                int2 *__restrict__ idx, int64_t n2, int unroll) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldcs(q + i);
    v.x = v.x * 2.0 + 1.0;
    v.y = v.y * 2.0 + 1.0;
    __stcs(out + i, v);
    __stcs(idx + i, make_int2((int)v.x, (int)v.y));
  }
}
__global__ void __launch_bounds__(256) k_stream_q(const double2 *__restrict__ q, double2 *__restrict__ out, int64_t n2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldcs(q + i);
    __stcs(out + i, v);
  }
}
int main() {
  const int64_t nq = 268435456, n2 = nq / 2;
  double2 *q, *out; int2 *idx;
  cudaMalloc(&q, nq * 8); cudaMalloc(&out, nq * 8); cudaMalloc(&idx, nq * 4);
  cudaMemset(q, 0, nq * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int g : {148 * 8, 148 * 16, 148 * 32}) {
    for (int it = 0; it < 2; ++it) k_stream<<<g, 256>>>(q, out, idx, n2, 1);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) k_stream<<<g, 256>>>(q, out, idx, n2, 1);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("q->out+idx grid %d: %.3f ms  %.1f GB/s\n", g, ms, nq * 20.0 / ms / 1e6);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) k_stream_q<<<g, 256>>>(q, out, n2);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("q->out      grid %d: %.3f ms  %.1f GB/s\n", g, ms, nq * 16.0 / ms / 1e6);
  }
  return 0;
}
