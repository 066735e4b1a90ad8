// Does a warp shuffle compete with shared-memory loads for the same datapath?
// Times three kernels with the same number of 64-bit moves per thread:
// LDS.64 only, SHFL (two 32-bit shuffles per double) only, and both interleaved.
// If "both" takes about as long as the sum, shuffles cannot relieve a
// shared-memory-bound transpose.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_shfl tools/ubench_shfl.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kThreads = 512;

__global__ void k_lds(double* out) {
  __shared__ double s_[kThreads * 2];
  volatile double* s = s_;
  s[threadIdx.x] = threadIdx.x;
  s[threadIdx.x + kThreads] = 2.0 * threadIdx.x;
  __syncthreads();
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int idx = threadIdx.x;
#pragma unroll 4
  for (int it = 0; it < kIters; it += 4) {
    a0 += s[idx];
    a1 += s[idx ^ 32];
    a2 += s[idx ^ 64];
    a3 += s[idx ^ 96];
    idx ^= kThreads;  // alternate halves (defeats hoisting)
  }
  out[blockIdx.x * kThreads + threadIdx.x] = a0 + a1 + a2 + a3;
}

__global__ void k_shfl(double* out) {
  double v = threadIdx.x;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int it = 0; it < kIters; it += 4) {
    a0 += __shfl_sync(0xffffffffu, v, lane ^ 1);
    a1 += __shfl_sync(0xffffffffu, v, lane ^ 2);
    a2 += __shfl_sync(0xffffffffu, v, lane ^ 4);
    a3 += __shfl_sync(0xffffffffu, v, lane ^ 8);
    v += 1.0;
  }
  out[blockIdx.x * kThreads + threadIdx.x] = a0 + a1 + a2 + a3;
}

__global__ void k_both(double* out) {
  __shared__ double s_[kThreads * 2];
  volatile double* s = s_;
  s[threadIdx.x] = threadIdx.x;
  s[threadIdx.x + kThreads] = 2.0 * threadIdx.x;
  __syncthreads();
  double v = threadIdx.x;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int idx = threadIdx.x, lane = threadIdx.x & 31;
#pragma unroll 4
  for (int it = 0; it < kIters; it += 4) {
    a0 += s[idx];
    a1 += __shfl_sync(0xffffffffu, v, lane ^ 1);
    a2 += s[idx ^ 64];
    a3 += __shfl_sync(0xffffffffu, v, lane ^ 4);
    idx ^= kThreads;
    v += 1.0;
  }
  out[blockIdx.x * kThreads + threadIdx.x] = a0 + a1 + a2 + a3;
}

template <typename K>
float time_it(K k, double* out, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<blocks, kThreads>>>(out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<blocks, kThreads>>>(out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * kThreads);
  const double moves = (double)blocks * kThreads * kIters;  // 64-bit values moved
  const float t_lds = time_it(k_lds, out, blocks);
  const float t_shfl = time_it(k_shfl, out, blocks);
  const float t_both = time_it(k_both, out, blocks);
  const double cyc = 1e-3 * clk * 1e3;  // cycles per ms at the nominal clock
  printf("SMs %d, nominal clock %.0f MHz, %d threads x %d blocks x %d 64-bit moves\n", sms, clk / 1e3, kThreads, blocks,
         kIters);
  printf("LDS.64 only      %8.3f ms  %6.1f B/clk/SM\n", t_lds, moves * 8 / (t_lds * cyc * sms));
  printf("SHFL (2x32) only %8.3f ms  %6.1f B/clk/SM\n", t_shfl, moves * 8 / (t_shfl * cyc * sms));
  printf("half / half      %8.3f ms  %6.1f B/clk/SM  (sum of halves would be %.3f ms)\n", t_both,
         moves * 8 / (t_both * cyc * sms), 0.5 * (t_lds + t_shfl));
  return 0;
}
