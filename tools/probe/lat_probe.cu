// Dependent-chain latency of the fp64 operations on the build's critical path (one warp, clock64).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lat_probe lat_probe.cu && ./lat_probe
#include <cstdio>
__device__ __forceinline__ double nr_rcp(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = __fma_rn(-a, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-a, r, 1.0);
  return __fma_rn(r, e, r);
}
__global__ void k(double *o, long long *t, double a, double b) {
  double v = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) v = __fma_rn(v, b, a);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) v = nr_rcp(v + 1.5);
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { float f = __double2float_rn(v); v = (double)__fdividef(1.f, f + 1.5f); }
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) v = __shfl_down_sync(0xffffffffu, v, 1) + 1.0;
  long long t4 = clock64();
  o[threadIdx.x] = v;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; }
}
int main() {
  double *o; long long *t, h[4];
  cudaMalloc(&o, 256 * 8); cudaMalloc(&t, 32);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, t, 0.5, 0.999);
  cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
  printf("cycles per dependent step: dfma %.1f  (dadd+nr_rcp) %.1f  (f2f+frcp) %.1f  (shfl.f64+dadd) %.1f\n",
         h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0, h[3] / 1024.0);
  return 0;
}
