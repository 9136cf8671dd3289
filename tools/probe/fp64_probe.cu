// fp64 issue throughput per SM (DFMA, DMUL+DADD mix, MUFU.RCP64H) at full occupancy.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_probe fp64_probe.cu && ./fp64_probe
#include <cstdio>
template <int OP> __global__ void k(double *o, double a, double b, int iters) {
  double v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = a + threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) v[i] = __fma_rn(v[i], b, a);
      if (OP == 1) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[i])); v[i] = r; }
      if (OP == 2) { float f = (float)v[i]; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(f)); v[i] = f; }
      if (OP == 3) v[i] = __dadd_rn(v[i], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *o; cudaMalloc(&o, sizeof(double) * sms * 4 * 256);
  const char *names[] = {"DFMA", "MUFU.RCP64H", "F2F+MUFU.RCP+F2F", "DADD"};
  for (int op = 0; op < 4; ++op) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<sms * 4, 256>>>(o, 0.5, 0.999, iters);
      if (op == 1) k<1><<<sms * 4, 256>>>(o, 0.5, 0.999, iters);
      if (op == 2) k<2><<<sms * 4, 256>>>(o, 0.5, 0.999, iters);
      if (op == 3) k<3><<<sms * 4, 256>>>(o, 0.5, 0.999, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_instr = (double)sms * 4 * 8 * iters * 8;  // per kernel
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-18s %.3f ms  %.3f warp-instr/clk/SM (at the %d MHz max clock)\n", names[op], ms, warp_instr / cyc / sms, clk / 1000);
  }
  return 0;
}
