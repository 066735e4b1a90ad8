// Throughput of MUFU.RCP64H (rcp.approx.ftz.f64) vs DFMA on B200: 8 independent
// streams per thread, full occupancy.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE, int IT>
__global__ void k(double* out, const double* __restrict__ in) {
  double v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = in[(threadIdx.x & 31) * 8 + q];
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[q])); v[q] = r; }
      else if (MODE == 1) v[q] = fma(v[q], 0.999999999, 1e-12);
      else { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[q]));
             v[q] = fma(r, 0.999999999, 1e-12); v[q] = fma(v[q], 1.000000001, -1e-12);
             v[q] = fma(v[q], 0.999999999, 1e-12); v[q] = fma(v[q], 1.000000001, -1e-12); }
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += v[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, int sms, double per) {
  const int IT = 2048, tpb = 512, blocks = sms * 4;
  double *o, *in; cudaMalloc(&o, sizeof(double) * tpb * blocks); cudaMalloc(&in, 256 * 8);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0 + i * 1e-3; cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  k<MODE, IT><<<blocks, tpb>>>(o, in); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<MODE, IT><<<blocks, tpb>>>(o, in); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 8.0 * IT * tpb * blocks;
  printf("%-36s %.3f ms  %.1f G%s/s  -> %.1f per clk per SM at 1965 MHz\n", name, ms, n * per / (ms * 1e6),
         "op", n * per / (ms * 1e-3) / 1.965e9 / sms);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("MUFU.RCP64H (lanes)", sms, 1.0);
  run<1>("DFMA (lanes)", sms, 1.0);
  run<2>("1 MUFU : 4 DFMA mix (MUFU lanes)", sms, 1.0);
  return 0;
}
