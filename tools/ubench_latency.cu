// Dependent-chain latencies on B200: DFMA, DADD, DMUL, MUFU.RCP64H (rcp.approx.f64),
// LDS.64 (shared round trip).  One warp, clock64 around a chain of N dependent ops.
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void lat(double* out, long long* cyc, double a, double b) {
  __shared__ double s[64];
  double x = threadIdx.x * 1e-3 + 1.0;
  s[threadIdx.x] = x;
  __syncwarp();
  long long t0, t1;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, a, b);
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + b;
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * a;
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t1 = clock64(); cyc[3] = t1 - t0;
  int idx = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { double v = s[idx]; idx = ((int)v) & 31; }
  t1 = clock64(); cyc[4] = t1 - t0;
  out[threadIdx.x] = x + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  lat<<<1, 32>>>(o, c, 0.999999, 1e-9); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 0.999999, 1e-9); cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[5] = {"DFMA", "DADD", "DMUL", "MUFU.RCP64H", "LDS.64 (+F2I)"};
  for (int i = 0; i < 5; ++i) printf("%-14s dependent latency %.2f cycles\n", nm[i], (double)h[i] / N);
  return 0;
}
