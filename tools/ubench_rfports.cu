// Register-file read-port test: does an independent integer IMAD (3 fresh
// 32-bit operands) slow a DFMA stream that already runs at the FP64 pipe rate?
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE, int IT>
__global__ void k(double* out, const double* __restrict__ in, const int* __restrict__ iin) {
  const int l = threadIdx.x & 31;
  double r[8];
  int a[8], b[8], c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { r[q] = in[l * 8 + q]; a[q] = iin[l * 24 + q]; b[q] = iin[l * 24 + 8 + q]; c[q] = iin[l * 24 + 16 + q]; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      r[q] = fma(r[q], 0.999999999, 1e-12);                        // DFMA: 1 fresh pair + consts
      if (MODE >= 1) c[q] = a[q] * b[q] + c[q];                    // IMAD: 3 fresh regs
      if (MODE >= 2) { a[q] = b[q] * c[q] + a[q]; }                // second IMAD
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += r[q] + a[q] + b[q] + c[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, int sms) {
  const int IT = 2048, tpb = 512, blocks = sms * 4;
  double *o, *in; int* iin;
  cudaMalloc(&o, sizeof(double) * tpb * blocks); cudaMalloc(&in, 256 * 8); cudaMalloc(&iin, 32 * 24 * 4);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0 + i * 1e-3; cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int hi[768]; for (int i = 0; i < 768; ++i) hi[i] = i * 7 + 1; cudaMemcpy(iin, hi, sizeof(hi), cudaMemcpyHostToDevice);
  k<MODE, IT><<<blocks, tpb>>>(o, in, iin); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<MODE, IT><<<blocks, tpb>>>(o, in, iin); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 8.0 * IT * tpb * blocks;
  printf("%-44s %.3f ms  DFMA %.1f per clk per SM (1965 MHz)\n", name, ms, n / (ms * 1e-3) / 1.965e9 / sms);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("DFMA only", sms);
  run<1>("DFMA + 1 independent IMAD (3 fresh regs)", sms);
  run<2>("DFMA + 2 independent IMADs", sms);
  return 0;
}
