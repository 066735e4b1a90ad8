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

#ifndef HX_N1
#error "compile with -DHX_N1=<points per direction>"
#endif

namespace hx {
namespace {

template <int N1>
struct GCfg {
  static constexpr int N3 = N1 * N1 * N1;
  static constexpr int TPE = N1 * N1;
  static constexpr int EPB = TPE >= 128 ? 1 : 128 / TPE;
  static constexpr int P = N1 + 1;  // padded slice row
};

template <int N1, int SRC, bool HELM>
struct Factors;

// ---- stored (Nek-style): load 6 (+1) SoA fields (axlocal.py:181-185) ----
template <int N1, bool HELM>
struct Factors<N1, HX_STORED, HELM> {
  const double* g;
  const double* gwj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ void init(const hx_axlocal_args& a, int64_t e, int, int) {
    constexpr int N3 = GCfg<N1>::N3;
    g = a.g + e * 6 * N3;
    gwj = HELM ? a.gwj + e * N3 : nullptr;
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  __device__ NodeFactors at(int node, int, int, int) const {
    constexpr int N3 = GCfg<N1>::N3;
    NodeFactors f;
    f.g0 = __ldg(g + 0 * N3 + node);
    f.g1 = __ldg(g + 1 * N3 + node);
    f.g2 = __ldg(g + 2 * N3 + node);
    f.g3 = __ldg(g + 3 * N3 + node);
    f.g4 = __ldg(g + 4 * N3 + node);
    f.g5 = __ldg(g + 5 * N3 + node);
    if (HELM) {
      f.grad_scale = lam0 ? __ldg(lam0 + node) : l0v;
      f.mass_scale = (lam1 ? __ldg(lam1 + node) : l1v) * __ldg(gwj + node);
    } else {
      f.grad_scale = 1.0;
      f.mass_scale = 0.0;
    }
    return f;
  }
  static constexpr bool kHasGradScale = HELM;
};

// ---- parallelepiped: w (x) h (geometry.py:389-398) ----
template <int N1, bool HELM>
struct Factors<N1, HX_PARALLELEPIPED, HELM> {
  double h[7];
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ void init(const hx_axlocal_args& a, int64_t e, int, int) {
#pragma unroll
    for (int q = 0; q < 7; ++q) h[q] = __ldg(a.h + e * 7 + q);
    constexpr int N3 = GCfg<N1>::N3;
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  __device__ NodeFactors at(int node, int i, int j, int k) const {
    const double w = cW<N1>(k) * cW<N1>(j) * cW<N1>(i);
    NodeFactors f;
    f.g0 = w * h[0];
    f.g1 = w * h[1];
    f.g2 = w * h[2];
    f.g3 = w * h[3];
    f.g4 = w * h[4];
    f.g5 = w * h[5];
    if (HELM) {
      f.grad_scale = lam0 ? __ldg(lam0 + node) : l0v;
      f.mass_scale = (lam1 ? __ldg(lam1 + node) : l1v) * (w * h[6]);
    } else {
      f.grad_scale = 1.0;
      f.mass_scale = 0.0;
    }
    return f;
  }
  static constexpr bool kHasGradScale = HELM;
};

// ---- trilinear recompute (geometry.py:304-351, axlocal.py:191-201) ----
template <int N1, bool HELM>
struct Factors<N1, HX_TRILINEAR, HELM> {
  TrilinearPencil p;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ void init(const hx_axlocal_args& a, int64_t e, int i, int j) {
    double v[24];
#pragma unroll
    for (int q = 0; q < 24; ++q) v[q] = __ldg(a.verts + e * 24 + q);
    trilinear_pencil(v, cX<N1>(i), cX<N1>(j), p);
    constexpr int N3 = GCfg<N1>::N3;
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  __device__ NodeFactors at(int node, int i, int j, int k) const {
    double g[6], det;
    trilinear_node(p, cX<N1>(k), g, det);
    const double w = cW<N1>(k) * cW<N1>(j) * cW<N1>(i);
    const double lam_geo = 0.125 * w / det;
    NodeFactors f{g[0], g[1], g[2], g[3], g[4], g[5], lam_geo, 0.0};
    if (HELM) {
      const double gwj = 0.015625 * det * det;
      f.grad_scale = (lam0 ? __ldg(lam0 + node) : l0v) * lam_geo;
      f.mass_scale = (lam1 ? __ldg(lam1 + node) : l1v) * (lam_geo * gwj);
    }
    return f;
  }
  static constexpr bool kHasGradScale = true;
};

// ---- trilinear, merged scalars lam2/lam3 (Helmholtz; axlocal.py:202-206) ----
template <int N1, bool HELM>
struct Factors<N1, HX_TRILINEAR_MERGED, HELM> {
  TrilinearPencil p;
  const double* lam2;
  const double* lam3;
  __device__ void init(const hx_axlocal_args& a, int64_t e, int i, int j) {
    double v[24];
#pragma unroll
    for (int q = 0; q < 24; ++q) v[q] = __ldg(a.verts + e * 24 + q);
    trilinear_pencil(v, cX<N1>(i), cX<N1>(j), p);
    constexpr int N3 = GCfg<N1>::N3;
    lam2 = a.lam2 + e * N3;
    lam3 = a.lam3 + e * N3;
  }
  __device__ NodeFactors at(int node, int, int, int k) const {
    double g[6], det;
    trilinear_node(p, cX<N1>(k), g, det);
    (void)det;
    return NodeFactors{g[0], g[1], g[2], g[3], g[4], g[5], __ldg(lam2 + node), __ldg(lam3 + node)};
  }
  static constexpr bool kHasGradScale = true;
};

// ---- trilinear, stored lam_geo (Poisson; axlocal.py:207-211) ----
template <int N1, bool HELM>
struct Factors<N1, HX_TRILINEAR_PARTIAL, HELM> {
  TrilinearPencil p;
  const double* lam_geo;
  __device__ void init(const hx_axlocal_args& a, int64_t e, int i, int j) {
    double v[24];
#pragma unroll
    for (int q = 0; q < 24; ++q) v[q] = __ldg(a.verts + e * 24 + q);
    trilinear_pencil(v, cX<N1>(i), cX<N1>(j), p);
    lam_geo = a.lam_geo + e * GCfg<N1>::N3;
  }
  __device__ NodeFactors at(int node, int, int, int k) const {
    double g[6], det;
    trilinear_node(p, cX<N1>(k), g, det);
    (void)det;
    return NodeFactors{g[0], g[1], g[2], g[3], g[4], g[5], __ldg(lam_geo + node), 0.0};
  }
  static constexpr bool kHasGradScale = true;
};

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
