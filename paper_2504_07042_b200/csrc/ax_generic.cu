// Generic AxLocal kernel for one order (compiled once per n1 with -DHX_N1=n1).
//
// Structure of the paper's 2-D thread block (Algorithm 4):
// one n1 x n1 thread layer per element, thread (i, j) owns the k-fiber
// X[:, j, i] in registers; the r/s contractions of slice k go through a padded
// shared-memory slice, the t contraction and its transpose stay in registers
// with D read from the __constant__ bank at compile-time offsets.  Factors are
// produced per node by the variant's getFactors (axlocal.py:171-211), once per
// node and reused by every field column (the paper's loop swap, §4.1).
//
// This kernel covers every (order, equation, n_col, factor source); the
// specialised kernels in ax_n8.cu take over where they exist.
#include "hx_common.cuh"
#include "node_factors.cuh"

#ifndef HX_N1
#error "compile with -DHX_N1=<points per direction>"
#endif

namespace hx {
namespace {

// Columns processed per pass: all at once while the register fibers stay
// small, else one at a time (factors then recomputed per column; per-column
// arithmetic is identical either way, so n_col=3 == 3 x n_col=1 bitwise).
template <int N1, int NCOL>
struct Pass {
  static constexpr int C = (NCOL * N1 <= 24) ? NCOL : 1;
};

template <int N1, int NCOL, int SRC, bool HELM>
__global__ void __launch_bounds__(GCfg<N1>::TPE * GCfg<N1>::EPB)
    ax_generic(const hx_axlocal_args a) {
  using Cfg = GCfg<N1>;
  constexpr int N3 = Cfg::N3, EPB = Cfg::EPB, P = Cfg::P;
  constexpr int CP = Pass<N1, NCOL>::C;
  __shared__ double s_D[N1][N1];   // s_D[n][i] = D[n][i]
  __shared__ double s_DT[N1][N1];  // s_DT[n][i] = D[i][n]
  __shared__ double s_x[EPB][CP][N1][P];
  __shared__ double s_r[EPB][CP][N1][P];
  __shared__ double s_s[EPB][CP][N1][P];

  const int i = threadIdx.x, j = threadIdx.y, le = threadIdx.z;
  const int tid = (le * N1 + j) * N1 + i;
  for (int q = tid; q < N1 * N1; q += Cfg::TPE * EPB) {
    const int r = q / N1, c = q % N1;
    s_D[r][c] = cD<N1>(r, c);
    s_DT[r][c] = cD<N1>(c, r);
  }
  const int64_t e_raw = (int64_t)blockIdx.x * EPB + le;
  const bool valid = e_raw < a.n_elements;
  const int64_t e = valid ? e_raw : 0;

  Factors<N1, SRC, HELM> fac;
  fac.init(a, e, i, j);

  for (int c0 = 0; c0 < NCOL; c0 += CP) {
    double xk[CP][N1], y[CP][N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = (k * N1 + j) * N1 + i;
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        xk[c][k] = valid ? __ldg(a.x + (e * N3 + node) * NCOL + c0 + c) : 0.0;
        y[c][k] = 0.0;
      }
    }
    __syncthreads();

#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = (k * N1 + j) * N1 + i;
      const NodeFactors f = fac.at(node, i, j, k);
#pragma unroll
      for (int c = 0; c < CP; ++c) s_x[le][c][j][i] = xk[c][k];
      __syncthreads();
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        double x0 = 0.0, x1 = 0.0, x2 = 0.0;
#pragma unroll
        for (int n = 0; n < N1; ++n) {
          x0 = fma(s_DT[n][i], s_x[le][c][j][n], x0);
          x1 = fma(s_DT[n][j], s_x[le][c][n][i], x1);
          x2 = fma(cD<N1>(k, n), xk[c][n], x2);
        }
        double rr = f.g0 * x0 + f.g1 * x1 + f.g2 * x2;
        double ss = f.g1 * x0 + f.g3 * x1 + f.g4 * x2;
        double tt = f.g2 * x0 + f.g4 * x1 + f.g5 * x2;
        if (Factors<N1, SRC, HELM>::kHasGradScale) {
          rr *= f.grad_scale;
          ss *= f.grad_scale;
          tt *= f.grad_scale;
        }
        s_r[le][c][j][i] = rr;
        s_s[le][c][j][i] = ss;
#pragma unroll
        for (int n = 0; n < N1; ++n) y[c][n] = fma(cD<N1>(k, n), tt, y[c][n]);
        if (HELM) y[c][k] = fma(f.mass_scale, xk[c][k], y[c][k]);
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int n = 0; n < N1; ++n) {
          acc = fma(s_D[n][i], s_r[le][c][j][n], acc);
          acc = fma(s_D[n][j], s_s[le][c][n][i], acc);
        }
        y[c][k] += acc;
      }
    }
    if (valid) {
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const int node = (k * N1 + j) * N1 + i;
#pragma unroll
        for (int c = 0; c < CP; ++c) a.y[(e * N3 + node) * NCOL + c0 + c] = y[c][k];
      }
    }
    __syncthreads();
  }
}

template <int N1, int NCOL, int SRC, bool HELM>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  using Cfg = GCfg<N1>;
  const int64_t blocks = (a.n_elements + Cfg::EPB - 1) / Cfg::EPB;
  dim3 block(N1, N1, Cfg::EPB);
  // grid.x limit is 2^31-1; E never comes close.
  ax_generic<N1, NCOL, SRC, HELM><<<(unsigned)blocks, block, 0, s>>>(a);
  return cudaGetLastError();
}

template <int N1, int NCOL>
cudaError_t dispatch_src(const hx_axlocal_args& a, cudaStream_t s) {
  const bool helm = a.equation == HX_HELMHOLTZ;
  switch (a.factor_source) {
    case HX_STORED:
      return helm ? launch<N1, NCOL, HX_STORED, true>(a, s) : launch<N1, NCOL, HX_STORED, false>(a, s);
    case HX_PARALLELEPIPED:
      return helm ? launch<N1, NCOL, HX_PARALLELEPIPED, true>(a, s)
                  : launch<N1, NCOL, HX_PARALLELEPIPED, false>(a, s);
    case HX_TRILINEAR:
      return helm ? launch<N1, NCOL, HX_TRILINEAR, true>(a, s) : launch<N1, NCOL, HX_TRILINEAR, false>(a, s);
    case HX_TRILINEAR_MERGED:
      return launch<N1, NCOL, HX_TRILINEAR_MERGED, true>(a, s);
    case HX_TRILINEAR_PARTIAL:
      return launch<N1, NCOL, HX_TRILINEAR_PARTIAL, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace
}  // namespace hx

#define HX_CAT2(a, b) a##b
#define HX_CAT(a, b) HX_CAT2(a, b)

extern "C" cudaError_t HX_CAT(hx_generic_launch_, HX_N1)(const hx_axlocal_args* a, cudaStream_t s) {
  return a->n_col == 3 ? hx::dispatch_src<HX_N1, 3>(*a, s) : hx::dispatch_src<HX_N1, 1>(*a, s);
}

HX_DEFINE_UPLOAD_HOOK(HX_CAT(hx_upload_basis_generic_, HX_N1))
