// Per-node geometric factors of every factor source (axlocal.py:171-211), for
// kernels that evaluate factors node by node: the slice kernel (ax_generic.cu)
// and the element-per-thread low-order kernel (ax_low.cu).  Included inside
// an anonymous namespace of each translation unit.
#pragma once
#include "hx_common.cuh"

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
  __device__ void init_from(const double*, const hx_axlocal_args& a, int64_t e, int i, int j) { init(a, e, i, j); }
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
  __device__ void init_from(const double*, const hx_axlocal_args& a, int64_t e, int i, int j) { init(a, e, i, j); }
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
    init_from(v, a, e, i, j);
  }
  // same, with the element's 24 vertex coordinates already at hand
  __device__ void init_from(const double* v, const hx_axlocal_args& a, int64_t e, int i, int j) {
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
    init_from(v, a, e, i, j);
  }
  // same, with the element's 24 vertex coordinates already at hand
  __device__ void init_from(const double* v, const hx_axlocal_args& a, int64_t e, int i, int j) {
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
    init_from(v, a, e, i, j);
  }
  // same, with the element's 24 vertex coordinates already at hand
  __device__ void init_from(const double* v, const hx_axlocal_args& a, int64_t e, int i, int j) {
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

}  // namespace
}  // namespace hx
