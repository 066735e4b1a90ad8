// FP64 pipe sharing between DMMA.8x8x4 and DFMA on one SM partition: for a
// group size G, each warp issues G independent DMMAs then 8G independent
// DFMAs per thread (equal FMA counts), in program order (asm volatile).
// Reports FMA/clk/SM for warps-per-SM in {4, 8, 12, 16}.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dfma(double& r, double a, double b) {
  asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(r) : "d"(a), "d"(b));
}

template <int G, int MODE>  // MODE 0 mixed, 1 DMMA only, 2 DFMA only, 3 warp-specialised (even warps DMMA, odd DFMA)
__global__ void k(double* out, int iters, long long* clk) {
  double acc[8][2], r[64];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-12;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = i;
#pragma unroll
  for (int i = 0; i < 64; ++i) r[i] = i;
  long long c0 = clock64();
  const bool dmma_warp = MODE != 3 || ((threadIdx.x >> 5) & 1) == 0;
  const bool dfma_warp = MODE != 3 || ((threadIdx.x >> 5) & 1) == 1;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 2 && dmma_warp) {
#pragma unroll
      for (int g = 0; g < G; ++g) dmma(acc[g][0], acc[g][1], a, b);
    }
    if (MODE != 1 && dfma_warp) {
#pragma unroll
      for (int g = 0; g < 8 * G; ++g) dfma(r[g], a, b);
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < 64; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int G, int MODE>
void run(const char* name, int warps_per_sm, double* out, long long* clk) {
  int sms = 148;
  const int iters = 4096 / G;
  dim3 grid(sms * warps_per_sm / 4), block(128);
  k<G, MODE><<<grid, block>>>(out, iters, clk);
  cudaDeviceSynchronize();
  long long h[2048];
  cudaMemcpy(h, clk, grid.x * sizeof(long long), cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (unsigned i = 0; i < grid.x; ++i) cmax = h[i] > cmax ? h[i] : cmax;
  // FMAs per SM: blocks per SM * warps per block * per warp per iter
  const double fma_per_warp_iter = MODE == 3 ? G * 256.0 : (MODE != 2 ? G * 256.0 : 0) + (MODE != 1 ? 8.0 * G * 32 : 0);
  const double per_sm = (double)warps_per_sm * iters * fma_per_warp_iter;
  printf("%-8s G=%d warps/SM=%2d: %6.1f FMA/clk/SM\n", name, G, warps_per_sm, per_sm / cmax);
}

int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 148 * 16 * 32 * 8 * 4);
  cudaMalloc(&clk, 2048 * 8);
  for (int w : {4, 8, 12, 16}) {
    run<1, 0>("mixed", w, out, clk);
    run<2, 0>("mixed", w, out, clk);
    run<4, 0>("mixed", w, out, clk);
    run<8, 0>("mixed", w, out, clk);
    run<4, 1>("dmma", w, out, clk);
    run<1, 3>("wspec", w, out, clk);
    run<4, 3>("wspec", w, out, clk);
    run<4, 2>("dfma", w, out, clk);
  }
  return 0;
}
