// FP64 pipe microbenchmarks for B200 (sm_100a).
//
// MEASURED_PEAKS.json carries HBM copy and bf16 GEMM peaks only; the AxLocal
// trilinear kernel is bound by the FP64 pipe, so its roofline denominator is
// measured here: DFMA (register and constant-bank operands), warp-level DMMA
// (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), DFMA+DMMA concurrently (are they
// separate pipes?), and shared-memory LDS.64/LDS.128 throughput.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 ubench_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__constant__ double cD[64];

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

// 8 independent DFMA chains per thread.
template <int ITERS>
__global__ void k_dfma(double* out, double a, double b, unsigned long long* clk) {
  double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  long long c0 = clock64(); unsigned long long t0 = gtimer();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
    r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
  }
  long long c1 = clock64(); unsigned long long t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}

// DFMA with a constant-bank multiplier (the pattern of D from __constant__).
template <int ITERS>
__global__ void k_dfma_const(double* out, unsigned long long* clk) {
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = threadIdx.x + q;
  long long c0 = clock64(); unsigned long long t0 = gtimer();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = fma(r[q], cD[n * 8 + q], cD[63 - q]);
    }
  }
  long long c1 = clock64(); unsigned long long t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
  double s = 0; for (int q = 0; q < 8; ++q) s += r[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// NACC independent m8n8k4 accumulators per warp.
template <int ITERS, int NACC>
__global__ void k_dmma(double* out, unsigned long long* clk) {
  double acc[NACC][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int q = 0; q < NACC; ++q) { acc[q][0] = q; acc[q][1] = -q; }
  long long c0 = clock64(); unsigned long long t0 = gtimer();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) dmma(acc[q][0], acc[q][1], a, b);
  }
  long long c1 = clock64(); unsigned long long t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
  double s = 0;
#pragma unroll
  for (int q = 0; q < NACC; ++q) s += acc[q][0] + acc[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Interleaved in one warp: per iteration 4 DMMA (1024 FMA/warp) and 32 DFMA/thread (1024 FMA/warp).
template <int ITERS>
__global__ void k_mixed(double* out, double a, double b, unsigned long long* clk) {
  double acc[4][2];
  double ma = 1.0 + threadIdx.x * 1e-9, mb = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int q = 0; q < 4; ++q) { acc[q][0] = q; acc[q][1] = -q; }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = threadIdx.x + q;
  long long c0 = clock64(); unsigned long long t0 = gtimer();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dmma(acc[q][0], acc[q][1], ma, mb);
#pragma unroll
      for (int p = 0; p < 8; ++p) r[p] = fma(r[p], a, b);
    }
  }
  long long c1 = clock64(); unsigned long long t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += acc[q][0] + acc[q][1];
#pragma unroll
  for (int p = 0; p < 8; ++p) s += r[p];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Shared memory read throughput: conflict-free LDS.64 or LDS.128.
template <int ITERS, int VEC>
__global__ void k_lds(double* out, unsigned long long* clk) {
  __shared__ __align__(16) double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc0 = 0, acc1 = 0;
  int base = threadIdx.x * VEC;
  long long c0 = clock64(); unsigned long long t0 = gtimer();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int idx = (base + u * 256 * VEC / 2 + it * 8) & (4096 - VEC);
      if (VEC == 2) {
        double2 v = *reinterpret_cast<const double2*>(&s[idx]);
        acc0 += v.x; acc1 += v.y;
      } else {
        acc0 += s[idx];
      }
    }
  }
  long long c1 = clock64(); unsigned long long t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1;
}

struct Res { float ms; double mhz; };

template <typename F>
Res timeit(F launch, unsigned long long* dclk) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(); CK(cudaDeviceSynchronize());
  float best = 1e30f; double mhz = 0;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long h[2]; CK(cudaMemcpy(h, dclk, 16, cudaMemcpyDeviceToHost));
    if (ms < best) { best = ms; mhz = h[1] ? (double)h[0] / (double)h[1] * 1e3 : 0; }
  }
  return {best, mhz};
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s, %d SMs\n", p.name, sms);
  double hD[64]; for (int i = 0; i < 64; ++i) hD[i] = 0.999 + 1e-6 * i;
  CK(cudaMemcpyToSymbol(cD, hD, sizeof(hD)));
  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  unsigned long long* clk; CK(cudaMalloc(&clk, 16));
  const int IT = 1 << 14;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    Res r = timeit([&] { k_dfma<IT><<<blocks, tpb>>>(out, 0.9999999, 1e-7, clk); }, clk);
    double fl = 2.0 * 8 * IT * (double)blocks * tpb;
    printf("DFMA reg   tpb=%4d: %8.3f ms  %7.2f TFLOP/s  SM clk %.0f MHz  -> %.1f FMA/clk/SM\n", tpb, r.ms,
           fl / r.ms / 1e9, r.mhz, fl / 2 / (r.ms * 1e-3) / (r.mhz * 1e6) / sms);
  }
  {
    const int IC = 1 << 10;
    int tpb = 256, blocks = sms * 8;
    Res r = timeit([&] { k_dfma_const<IC><<<blocks, tpb>>>(out, clk); }, clk);
    double fl = 2.0 * 64 * IC * (double)blocks * tpb;
    printf("DFMA const tpb=%4d: %8.3f ms  %7.2f TFLOP/s  SM clk %.0f MHz  -> %.1f FMA/clk/SM\n", tpb, r.ms,
           fl / r.ms / 1e9, r.mhz, fl / 2 / (r.ms * 1e-3) / (r.mhz * 1e6) / sms);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (1024 / tpb);
    const int ID = 1 << 12;
    Res r = timeit([&] { k_dmma<ID, 8><<<blocks, tpb>>>(out, clk); }, clk);
    double fl = 2.0 * 256 * 8 * ID * (double)blocks * (tpb / 32);
    printf("DMMA 8acc  tpb=%4d: %8.3f ms  %7.2f TFLOP/s  SM clk %.0f MHz  -> %.1f FMA/clk/SM\n", tpb, r.ms,
           fl / r.ms / 1e9, r.mhz, fl / 2 / (r.ms * 1e-3) / (r.mhz * 1e6) / sms);
  }
  {
    int tpb = 256, blocks = sms * 8;
    const int ID = 1 << 12;
    Res r = timeit([&] { k_dmma<ID, 4><<<blocks, tpb>>>(out, clk); }, clk);
    double fl = 2.0 * 256 * 4 * ID * (double)blocks * (tpb / 32);
    printf("DMMA 4acc  tpb=%4d: %8.3f ms  %7.2f TFLOP/s  SM clk %.0f MHz  -> %.1f FMA/clk/SM\n", tpb, r.ms,
           fl / r.ms / 1e9, r.mhz, fl / 2 / (r.ms * 1e-3) / (r.mhz * 1e6) / sms);
  }
  {
    int tpb = 256, blocks = sms * 8;
    const int IM = 1 << 12;
    Res r = timeit([&] { k_mixed<IM><<<blocks, tpb>>>(out, 0.9999999, 1e-7, clk); }, clk);
    double fl = 2.0 * (4 * 256 + 4 * 8 * 32) * IM * (double)blocks * (tpb / 32);
    printf("MIXED      tpb=%4d: %8.3f ms  %7.2f TFLOP/s  SM clk %.0f MHz  -> %.1f FMA/clk/SM (half DMMA, half DFMA)\n",
           tpb, r.ms, fl / r.ms / 1e9, r.mhz, fl / 2 / (r.ms * 1e-3) / (r.mhz * 1e6) / sms);
  }
  {
    int tpb = 256, blocks = sms * 8;
    const int IL = 1 << 13;
    Res r = timeit([&] { k_lds<IL, 1><<<blocks, tpb>>>(out, clk); }, clk);
    double by = 8.0 * 8 * IL * (double)blocks * tpb;
    printf("LDS.64     tpb=%4d: %8.3f ms  %7.1f GB/s   SM clk %.0f MHz  -> %.1f B/clk/SM\n", tpb, r.ms,
           by / r.ms / 1e6, r.mhz, by / (r.ms * 1e-3) / (r.mhz * 1e6) / sms);
    Res r2 = timeit([&] { k_lds<IL, 2><<<blocks, tpb>>>(out, clk); }, clk);
    by *= 2;
    printf("LDS.128    tpb=%4d: %8.3f ms  %7.1f GB/s   SM clk %.0f MHz  -> %.1f B/clk/SM\n", tpb, r2.ms,
           by / r2.ms / 1e6, r2.mhz, by / (r2.ms * 1e-3) / (r2.mhz * 1e6) / sms);
  }
  return 0;
}
