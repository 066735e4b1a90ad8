// Low-order AxLocal kernel: one thread per element (compiled per -DHX_N1 for
// n1 = 2, 3).
//
// At N = 1, 2 an element is 8 / 27 nodes: a thread block per element leaves
// most lanes idle through the per-element geometry setup (the slice and fast
// kernels reach 40 % of the HBM roofline at N = 1), while one thread holding a
// whole element in registers needs no shared memory and no barriers.  The
// block's elements are contiguous, so x / y move through shared memory in
// coalesced block-wide copies (padded so the per-thread accesses are
// bank-conflict free).  Factors come per node from node_factors.cuh (every
// source); per-column arithmetic is identical, so n_col=3 == 3 x n_col=1.
#include "hx_common.cuh"
#include "node_factors.cuh"

#ifndef HX_N1
#error "compile with -DHX_N1=<points per direction>"
#endif

namespace hx {
namespace {

constexpr int N1 = HX_N1;
constexpr int N3 = N1 * N1 * N1;
constexpr int TPB = N1 == 2 ? 128 : 64;  // elements (threads) per block
// CTAs per SM for the launch bounds (trilinear sources; the others use 7 / 1): n1 = 2
// caps registers at 128 (70 for the others, 268 vs 211 GDOF/s for ppd at N = 1);
// n1 = 3 holds 2 x 27 doubles per thread and gets all 255
#ifndef HX_LOW_MINB  // A/B builds (tools/build_variant.sh)
#define HX_LOW_MINB (N1 == 2 ? 4 : 1)
#endif
constexpr int MINB = HX_LOW_MINB;
// stored / parallelepiped sources: n1 = 2 at 7 CTAs / SM; n1 = 3 parallelepiped at 6
// for n_col = 1 (168 registers, ~100 B of spills: 250 -> 293 GDOF/s), else 1 (n_col = 3
// spills at 168: -9 %; stored -14 %)
constexpr int minb_other(int src, int ncol) {
  return N1 == 2 ? 7 : (src == HX_PARALLELEPIPED && ncol == 1 ? 6 : 1);
}
constexpr int PAD = N3 | 1;    // odd stride in doubles: conflict-free 64-bit smem accesses

__host__ __device__ constexpr bool tri_src(int src) {
  return src == HX_TRILINEAR || src == HX_TRILINEAR_MERGED || src == HX_TRILINEAR_PARTIAL;
}

// Block copies between a block's contiguous global rows (W doubles per element,
// n_col-strided) and padded shared rows.  Full blocks issue a batch of loads
// (stores) per thread before the first shared store (global store): the copies are
// latency bound otherwise (one 8-byte load in flight per thread per iteration);
// batches of kBatch bound the registers the copy holds next to the element state.
#ifndef HX_LOW_BATCH
#define HX_LOW_BATCH 8
#endif
constexpr int kBatch = HX_LOW_BATCH;
template <int W, int P, int STRIDE>
__device__ __forceinline__ void stage_in(double* __restrict__ s, const double* __restrict__ g, int nb) {
  if (nb == TPB) {
#pragma unroll
    for (int u0 = 0; u0 < W; u0 += kBatch) {
      double v[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (u0 + u < W) v[u] = __ldg(g + (int64_t)((u0 + u) * TPB + threadIdx.x) * STRIDE);
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (u0 + u < W) {
          const int idx = (u0 + u) * TPB + threadIdx.x, l = idx / W, q = idx - l * W;
          s[l * P + q] = v[u];
        }
    }
  } else {
    for (int idx = threadIdx.x; idx < nb * W; idx += TPB) {
      const int l = idx / W, q = idx - l * W;
      s[l * P + q] = __ldg(g + (int64_t)idx * STRIDE);
    }
  }
}

template <int W, int P, int STRIDE>
__device__ __forceinline__ void stage_out(double* __restrict__ g, const double* __restrict__ s, int nb) {
  if (nb == TPB) {
#pragma unroll
    for (int u0 = 0; u0 < W; u0 += kBatch) {
      double v[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (u0 + u < W) {
          const int idx = (u0 + u) * TPB + threadIdx.x, l = idx / W, q = idx - l * W;
          v[u] = s[l * P + q];
        }
#pragma unroll
      for (int u = 0; u < kBatch; ++u)
        if (u0 + u < W) g[(int64_t)((u0 + u) * TPB + threadIdx.x) * STRIDE] = v[u];
    }
  } else {
    for (int idx = threadIdx.x; idx < nb * W; idx += TPB) {
      const int l = idx / W, q = idx - l * W;
      g[(int64_t)idx * STRIDE] = s[l * P + q];
    }
  }
}

template <int NCOL, int SRC, bool HELM>
__global__ void __launch_bounds__(TPB, tri_src(SRC) ? MINB : minb_other(SRC, NCOL)) ax_low(const hx_axlocal_args a) {
  constexpr int VP = 25;  // padded vertex stride (odd: conflict-free)
  __shared__ double s_v[TPB * PAD];                     // x / y of one column
  __shared__ double s_vert[tri_src(SRC) ? TPB * VP : 1];  // the block's vertices (trilinear sources)
  const int64_t e0 = (int64_t)blockIdx.x * TPB;
  const int64_t left = a.n_elements - e0;
  const int nb = left < TPB ? (int)left : TPB;  // elements in this block
  const int64_t e = e0 + threadIdx.x;
  const bool valid = threadIdx.x < nb;
  Factors<N1, SRC, HELM> fac;
  const double* vtx = s_vert + threadIdx.x * VP;  // this thread's element, read by each column's pencil
  if constexpr (tri_src(SRC)) {
    // coalesced block copy of the vertices, then each thread keeps its element's 24
    stage_in<24, VP, 1>(s_vert, a.verts + e0 * 24, nb);
    __syncthreads();
  }
#pragma unroll 1
  for (int c = 0; c < NCOL; ++c) {
    // coalesced block copy of column c: x[(e0 + l) N3 + q] -> s_v[l PAD + q]
    stage_in<N3, PAD, NCOL>(s_v, a.x + e0 * N3 * NCOL + c, nb);
    __syncthreads();
    double x[N3], y[N3];
#pragma unroll
    for (int q = 0; q < N3; ++q) {
      x[q] = s_v[threadIdx.x * PAD + q];
      y[q] = 0.0;
    }
    if (valid) {
#pragma unroll
      for (int j = 0; j < N1; ++j)
#pragma unroll
        for (int i = 0; i < N1; ++i) {
          if constexpr (tri_src(SRC))
            fac.init_from(vtx, a, e, i, j);
          else
            fac.init(a, e, i, j);
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            const int node = (k * N1 + j) * N1 + i;
            const NodeFactors f = fac.at(node, i, j, k);
            double x0 = 0.0, x1 = 0.0, x2 = 0.0;
#pragma unroll
            for (int n = 0; n < N1; ++n) {
              x0 = fma(cD<N1>(i, n), x[(k * N1 + j) * N1 + n], x0);
              x1 = fma(cD<N1>(j, n), x[(k * N1 + n) * N1 + i], x1);
              x2 = fma(cD<N1>(k, n), x[(n * N1 + j) * N1 + i], x2);
            }
            double rr = f.g0 * x0 + f.g1 * x1 + f.g2 * x2;
            double ss = f.g1 * x0 + f.g3 * x1 + f.g4 * x2;
            double tt = f.g2 * x0 + f.g4 * x1 + f.g5 * x2;
            if (Factors<N1, SRC, HELM>::kHasGradScale) {
              rr *= f.grad_scale;
              ss *= f.grad_scale;
              tt *= f.grad_scale;
            }
#pragma unroll
            for (int m = 0; m < N1; ++m) {  // D^T: y_m += D(i, m) rr_i etc.
              y[(k * N1 + j) * N1 + m] = fma(cD<N1>(i, m), rr, y[(k * N1 + j) * N1 + m]);
              y[(k * N1 + m) * N1 + i] = fma(cD<N1>(j, m), ss, y[(k * N1 + m) * N1 + i]);
              y[(m * N1 + j) * N1 + i] = fma(cD<N1>(k, m), tt, y[(m * N1 + j) * N1 + i]);
            }
            if (HELM) y[node] = fma(f.mass_scale, x[node], y[node]);
          }
        }
    }
    __syncthreads();  // every thread has read its x
#pragma unroll
    for (int q = 0; q < N3; ++q) s_v[threadIdx.x * PAD + q] = y[q];
    __syncthreads();
    stage_out<N3, PAD, NCOL>(a.y + e0 * N3 * NCOL + c, s_v, nb);
    if (NCOL > 1) __syncthreads();
  }
}

template <int NCOL, int SRC, bool HELM>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  const int64_t blocks = (a.n_elements + TPB - 1) / TPB;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  ax_low<NCOL, SRC, HELM><<<(unsigned)blocks, TPB, 0, s>>>(a);
  return cudaGetLastError();
}

template <int NCOL>
cudaError_t dispatch_src(const hx_axlocal_args& a, cudaStream_t s) {
  const bool helm = a.equation == HX_HELMHOLTZ;
  switch (a.factor_source) {
    case HX_STORED:
      return helm ? launch<NCOL, HX_STORED, true>(a, s) : launch<NCOL, HX_STORED, false>(a, s);
    case HX_PARALLELEPIPED:
      return helm ? launch<NCOL, HX_PARALLELEPIPED, true>(a, s) : launch<NCOL, HX_PARALLELEPIPED, false>(a, s);
    case HX_TRILINEAR:
      return helm ? launch<NCOL, HX_TRILINEAR, true>(a, s) : launch<NCOL, HX_TRILINEAR, false>(a, s);
    case HX_TRILINEAR_MERGED:
      return launch<NCOL, HX_TRILINEAR_MERGED, true>(a, s);
    case HX_TRILINEAR_PARTIAL:
      return launch<NCOL, HX_TRILINEAR_PARTIAL, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace
}  // namespace hx

#define HX_CAT2(a, b) a##b
#define HX_CAT(a, b) HX_CAT2(a, b)

extern "C" cudaError_t HX_CAT(hx_low_launch_, HX_N1)(const hx_axlocal_args* a, cudaStream_t s) {
  return a->n_col == 3 ? hx::dispatch_src<3>(*a, s) : hx::dispatch_src<1>(*a, s);
}

// basis upload for this translation unit's __constant__ copy
HX_DEFINE_UPLOAD_HOOK(HX_CAT(hx_upload_basis_low_, HX_N1))
