// Does a DFMA with three distinct register operands issue at the FP64 pipe rate
// (2 cycles/warp/SMSP) or at the register-file bank limit (3 distinct even/odd
// registers -> 3 cycles)?  8 independent chains per thread, operands rotated
// so the reuse cache cannot serve them.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE, int IT>
__global__ void k(double* out, long long* clk, const double* __restrict__ in) {
  double a[8], b[8], r[8];
#pragma unroll
  const double* p = in + (threadIdx.x & 31) * 24;
  for (int q = 0; q < 8; ++q) { a[q] = p[q]; b[q] = p[8 + q]; r[q] = p[16 + q]; }
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) r[q] = fma(a[0], b[0], r[q]);          // shared operands: reuse-friendly
      else if (MODE == 1) r[q] = fma(a[q], b[q], r[q]);     // 3 distinct regs per DFMA
      else if (MODE == 2) r[q] = fma(a[q], r[q], 1e-9);     // 2 regs + immediate
      else r[q] = r[q] * a[q];                              // DMUL, 2 regs
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += r[q] + a[q] + b[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, int sms) {
  const int IT = 4096, tpb = 512, blocks = sms * 4;
  double* o; long long* c; double* in; cudaMalloc(&o, sizeof(double) * tpb * blocks); cudaMalloc(&c, 8);
  cudaMalloc(&in, 24 * 8 * 32);
  double hin[24 * 32]; for (int q = 0; q < 24 * 32; ++q) hin[q] = (q % 24) < 8 ? 1.0 - 1e-12 * q : 1e-12 * q;
  cudaMemcpy(in, hin, sizeof(hin), cudaMemcpyHostToDevice);
  k<MODE, IT><<<blocks, tpb>>>(o, c, in); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<MODE, IT><<<blocks, tpb>>>(o, c, in); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double ops = 8.0 * IT * tpb * blocks;
  printf("%-40s %.3f ms  %.1f FP64 ops/clk/SM (at %.0f MHz from clock64)\n", name, ms,
         ops / (ms * 1e-3) / (h / (ms * 1e-3)) / sms, h / (ms * 1e3));
  cudaFree(o); cudaFree(c);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("DFMA r=fma(r,a0,b0) shared operands", sms);
  run<1>("DFMA r=fma(r,a_q,b_q) 3 distinct regs", sms);
  run<2>("DFMA r=fma(r,a_q,imm) 2 regs + imm", sms);
  run<3>("DMUL r=r*a_q 2 distinct regs", sms);
  return 0;
}
