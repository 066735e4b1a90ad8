// Shared definitions for the AxLocal kernels (sm_100a).
//
// Basis constants live in __constant__ memory.  Every translation unit gets its
// own static copy (the library is built without -rdc so the per-order kernel
// files compile in parallel); hx_set_basis() uploads into every copy through
// the per-TU hx_upload_basis_* hooks declared at the bottom.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hx_axlocal.h"

namespace hx {

constexpr int kMaxN1 = 16;

// Packed offsets of order-n1 data inside the constant arrays (n1 = 1..16).
__host__ __device__ constexpr int off_d(int n1) { return (n1 - 1) * n1 * (2 * n1 - 1) / 6; }
__host__ __device__ constexpr int off_p(int n1) { return (n1 - 1) * n1 / 2; }
constexpr int kDTotal = off_d(kMaxN1 + 1);
constexpr int kPTotal = off_p(kMaxN1 + 1);

}  // namespace hx

// D[i][n] row-major, 1-D weights and points, per order.
static __constant__ double c_D[hx::kDTotal];
static __constant__ double c_W[hx::kPTotal];
static __constant__ double c_X[hx::kPTotal];

template <int N1>
__device__ __forceinline__ double cD(int i, int n) { return c_D[hx::off_d(N1) + i * N1 + n]; }
template <int N1>
__device__ __forceinline__ double cW(int i) { return c_W[hx::off_p(N1) + i]; }
template <int N1>
__device__ __forceinline__ double cX(int i) { return c_X[hx::off_p(N1) + i]; }

static inline cudaError_t hx_upload_basis_local(int n1, const double* pts, const double* w, const double* d) {
  cudaError_t e = cudaMemcpyToSymbol(c_D, d, sizeof(double) * n1 * n1, sizeof(double) * hx::off_d(n1));
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(c_W, w, sizeof(double) * n1, sizeof(double) * hx::off_p(n1));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_X, pts, sizeof(double) * n1, sizeof(double) * hx::off_p(n1));
}

namespace hx {

// Factor-stage bookkeeping shared by all kernels (axlocal.py:171-211).
// grad_scale multiplies (rr, ss, tt) after the symmetric product; mass_scale
// multiplies x for the Helmholtz mass term.
struct NodeFactors {
  double g0, g1, g2, g3, g4, g5;
  double grad_scale;  // 1 when the variant has none
  double mass_scale;  // 0 for Poisson
};

// det of the 3x3 matrix with columns c0, c1, c2 (entry [a][b] = c_b[a]),
// cofactor expansion in the reference's order (geometry.py:216-222).
__device__ __forceinline__ double det3_cols(const double c0[3], const double c1[3], const double c2[3]) {
  return c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) - c0[1] * (c1[0] * c2[2] - c1[2] * c2[0]) +
         c0[2] * (c1[0] * c2[1] - c1[1] * c2[0]);
}

// Per-thread trilinear common terms of JT = 8J for fixed (i, j)
// (common_terms, geometry.py:135-184; Algorithm 2 lines 1-14).
struct TrilinearPencil {
  double dr_base[3], dr_slope[3], ds_base[3], ds_slope[3], dt_col[3];
};

__device__ __forceinline__ void trilinear_pencil(const double* __restrict__ v, double xi_i, double xi_j,
                                                 TrilinearPencil& p) {
  const double a0j = 1.0 - xi_j, a1j = 1.0 + xi_j;
  const double a0i = 1.0 - xi_i, a1i = 1.0 + xi_i;
  const double w00 = a0j * a0i, w01 = a0j * a1i, w10 = a1j * a0i, w11 = a1j * a1i;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double v0 = v[0 * 3 + c], v1 = v[1 * 3 + c], v2 = v[2 * 3 + c], v3 = v[3 * 3 + c];
    const double v4 = v[4 * 3 + c], v5 = v[5 * 3 + c], v6 = v[6 * 3 + c], v7 = v[7 * 3 + c];
    const double tmp1 = a0j * (v1 - v0) + a1j * (v3 - v2);
    const double tmp2 = a0j * (v5 - v4) + a1j * (v7 - v6);
    const double tmp3 = a0i * (v2 - v0) + a1i * (v3 - v1);
    const double tmp4 = a0i * (v6 - v4) + a1i * (v7 - v5);
    p.dr_base[c] = tmp1 + tmp2;
    p.dr_slope[c] = tmp2 - tmp1;
    p.ds_base[c] = tmp3 + tmp4;
    p.ds_slope[c] = tmp4 - tmp3;
    p.dt_col[c] = w00 * (v4 - v0) + w01 * (v5 - v1) + w11 * (v7 - v3) + w10 * (v6 - v2);
  }
}

// Unscaled adjugate factors of K = JT^T JT at reference coordinate t
// (trilinear_factors, geometry.py:319-339) plus det(JT).
__device__ __forceinline__ void trilinear_node(const TrilinearPencil& p, double t, double g[6], double& det) {
  double c0[3], c1[3], c2[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    c0[c] = p.dr_base[c] + t * p.dr_slope[c];
    c1[c] = p.ds_base[c] + t * p.ds_slope[c];
    c2[c] = p.dt_col[c];
  }
  const double k00 = c0[0] * c0[0] + c0[1] * c0[1] + c0[2] * c0[2];
  const double k01 = c0[0] * c1[0] + c0[1] * c1[1] + c0[2] * c1[2];
  const double k02 = c0[0] * c2[0] + c0[1] * c2[1] + c0[2] * c2[2];
  const double k11 = c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2];
  const double k12 = c1[0] * c2[0] + c1[1] * c2[1] + c1[2] * c2[2];
  const double k22 = c2[0] * c2[0] + c2[1] * c2[1] + c2[2] * c2[2];
  g[0] = k11 * k22 - k12 * k12;
  g[1] = k02 * k12 - k01 * k22;
  g[2] = k01 * k12 - k02 * k11;
  g[3] = k00 * k22 - k02 * k02;
  g[4] = k01 * k02 - k00 * k12;
  g[5] = k00 * k11 - k01 * k01;
  det = det3_cols(c0, c1, c2);
}

}  // namespace hx

// Per-translation-unit basis upload hooks (defined by HX_DEFINE_UPLOAD_HOOK).
#define HX_DEFINE_UPLOAD_HOOK(NAME)                                                                   \
  extern "C" cudaError_t NAME(int n1, const double* pts, const double* w, const double* d) {         \
    return hx_upload_basis_local(n1, pts, w, d);                                                     \
  }

// ---------------------------------------------------------------------------
// mbarrier + 1-D bulk async copy (TMA) helpers (PTX ISA 8.x, sm_90+).
namespace hx {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Order earlier generic-proxy shared accesses before later async-proxy (TMA) writes.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

// global -> shared bulk copy completing `bytes` transactions on `bar` (16 B aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Prefetch the line holding p into L2.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}

// Bulk prefetch of [src, src + bytes) into L2 (no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

}  // namespace hx

// ---------------------------------------------------------------------------
// Race-detection build (-DHX_PERTURB, tools/race_perturb.sh).  compute-sanitizer
// is not available on the GPU pool, so shared-memory races are hunted by timing
// perturbation instead: every barrier first stalls the calling thread for a
// pseudo-random 0..4095 ns (different per thread, CTA, call and run), so that
// any shared access not ordered by a barrier interleaves differently from the
// normal build; the outputs of both builds are then compared bit for bit.
#ifdef HX_PERTURB
__device__ __forceinline__ void hx_dbg_jitter(unsigned site) {
  unsigned h = (threadIdx.x + 97u * threadIdx.y) * 2654435761u;
  h ^= (blockIdx.x * 40503u + blockIdx.y * 9176u) ^ (site * 2246822519u) ^ (unsigned)clock();
  h ^= h >> 15;
  h *= 2246822519u;
  h ^= h >> 13;
  __nanosleep(h & 4095u);
}
__device__ __forceinline__ void hx_dbg_syncthreads() {
  hx_dbg_jitter(1);
  __syncthreads();
  hx_dbg_jitter(2);
}
__device__ __forceinline__ void hx_dbg_syncwarp() {
  hx_dbg_jitter(3);
  __syncwarp();
  hx_dbg_jitter(4);
}
#define __syncthreads() hx_dbg_syncthreads()
#define __syncwarp() hx_dbg_syncwarp()
#endif
