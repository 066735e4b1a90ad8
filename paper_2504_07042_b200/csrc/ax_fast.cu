// Specialised AxLocal kernel for N = 7 (n1 = 8), the north-star order.
//
// One 64-thread CTA per element.  The FP64 pipe (DFMA and DMMA share it on
// B200, tools/ubench_fp64.cu) is the bound, so the design minimises FP64
// operations and keeps shared memory under the pipe time:
//
//  * contractions by even-odd decomposition: D and D^T are centro-
//    antisymmetric on GLL points, so an 8-point contraction is 8 adds +
//    two 4x4 products + 8 adds = 48 ops instead of 64 (the 4x4 blocks sit in
//    __constant__ and are DFMA operands at compile-time offsets);
//  * three pencil ownerships per element (k-fibres, i-rows, j-columns); the
//    element cube moves between them through shared memory with the additive
//    layout a(k,j,i) = Ak[k] + Aj[j] + i, conflict-free for all three access
//    patterns (DESIGN.md derives it);
//  * trilinear geometry (Algorithm 2) as polynomials in the
//    reference coordinate t along each k-fibre: K00, K01, K11 are quadratic,
//    K02, K12 linear, K22 constant, det(JT) quadratic, so a node costs 8 FMAs
//    for K, 12 for adj(K), 2 for det and one reciprocal (MUFU + 3 FMAs)
//    instead of re-evaluating the Jacobian columns;
//  * D, tensor weights and points never touch shared memory.
//
// The arithmetic differs from the reference's operation order, so parity is
// to the 1e-12 relative bar, not bitwise; per-column arithmetic is identical
// for n_col = 1 and 3, so n_col=3 == 3 x n_col=1 bitwise.
#include "hx_common.cuh"

namespace hx {
namespace fast {

constexpr int N1 = 8;
constexpr int N3 = 512;
constexpr int CUBE = 576;  // 575 used, rounded up


__host__ __device__ constexpr int Aj(int j) { return 17 * (j >> 1) + 8 * (j & 1); }
__host__ __device__ constexpr int Ak(int k) { return 144 * (k >> 1) + 72 * (k & 1) + 4 * ((k >> 1) & 1); }

}  // namespace fast
}  // namespace hx

// Even-odd blocks: [0] forward D, [1] transposed D^T; [.][0] = A (even), [.][1] = B (odd);
// A[i][m] = (M[i][m] + M[i][7-m]) / 2, B[i][m] = (M[i][m] - M[i][7-m]) / 2 for M = D or D^T.
static __constant__ double c_EO[2][2][4][4];

namespace hx {
namespace fast {

// out = M v for an 8-point fibre, M = D (T=0) or D^T (T=1).
template <int T>
__device__ __forceinline__ void eo8(const double v[8], double out[8]) {
  double ue[4], uo[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    ue[m] = v[m] + v[7 - m];
    uo[m] = v[m] - v[7 - m];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double p = c_EO[T][0][i][0] * ue[0];
    double q = c_EO[T][1][i][0] * uo[0];
#pragma unroll
    for (int m = 1; m < 4; ++m) {
      p = fma(c_EO[T][0][i][m], ue[m], p);
      q = fma(c_EO[T][1][i][m], uo[m], q);
    }
    out[i] = p + q;
    out[7 - i] = q - p;
  }
}

// 1/d from the MUFU seed and one cubic correction: r (1 + e + e^2), e = 1 - d r.
__device__ __forceinline__ double rcp_fast(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  return fma(fma(e, e, e), r, r);
}

struct Fibre {
  int i, j;  // k-fibre owner
};

// ---------------------------------------------------------------------------
// factor policies: prepare() once per element (after vertices are in smem),
// node(k, x0, x1, x2, &rr, &ss, &tt, &mass_scale) per node of the k-fibre.

// Trilinear recompute (geometry.py:304-351; axlocal.py:191-201), polynomial in t.
template <bool HELM, bool MERGED, bool PARTIAL>
struct TrilinearPoly {
  double k00[3], k11[3], k01[3], k02[2], k12[2], k22, det[3];
  double w_ji;  // w_j * w_i with the k weight applied per node: (w_k w_j) w_i
  double wj, wi;
  const double* lam_a;  // partial: lam_geo; merged: lam2; trilinear-helm: lam0 (or null)
  const double* lam_b;  // merged: lam3; trilinear-helm: lam1 (or null)
  double l0v, l1v;

  __device__ void prepare(const hx_axlocal_args& a, int64_t e, const double* sv, Fibre f) {
    const double xi = cX<N1>(f.i), xj = cX<N1>(f.j);
    TrilinearPencil p;
    trilinear_pencil(sv, xi, xj, p);
    const double* br = p.dr_base;
    const double* sr = p.dr_slope;
    const double* bs = p.ds_base;
    const double* ss = p.ds_slope;
    const double* c = p.dt_col;
    auto dot = [](const double* u, const double* v) { return u[0] * v[0] + u[1] * v[1] + u[2] * v[2]; };
    k00[0] = dot(br, br);
    k00[1] = 2.0 * dot(br, sr);
    k00[2] = dot(sr, sr);
    k11[0] = dot(bs, bs);
    k11[1] = 2.0 * dot(bs, ss);
    k11[2] = dot(ss, ss);
    k01[0] = dot(br, bs);
    k01[1] = dot(br, ss) + dot(sr, bs);
    k01[2] = dot(sr, ss);
    k02[0] = dot(br, c);
    k02[1] = dot(sr, c);
    k12[0] = dot(bs, c);
    k12[1] = dot(ss, c);
    k22 = dot(c, c);
    // det = (br + t sr) . ((bs + t ss) x c)
    const double P[3] = {bs[1] * c[2] - bs[2] * c[1], bs[2] * c[0] - bs[0] * c[2], bs[0] * c[1] - bs[1] * c[0]};
    const double Q[3] = {ss[1] * c[2] - ss[2] * c[1], ss[2] * c[0] - ss[0] * c[2], ss[0] * c[1] - ss[1] * c[0]};
    det[0] = dot(br, P);
    det[1] = dot(br, Q) + dot(sr, P);
    det[2] = dot(sr, Q);
    wj = cW<N1>(f.j);
    wi = cW<N1>(f.i);
    lam_a = lam_b = nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
    if (PARTIAL) {
      lam_a = a.lam_geo + e * N3;
    } else if (MERGED) {
      lam_a = a.lam2 + e * N3;
      lam_b = a.lam3 + e * N3;
    } else if (HELM) {
      lam_a = a.lam0 ? a.lam0 + e * N3 : nullptr;
      lam_b = a.lam1 ? a.lam1 + e * N3 : nullptr;
    }
  }

  template <int K>
  __device__ __forceinline__ void node(int nodeidx, double x0, double x1, double x2, double& rr, double& ss,
                                       double& tt, double& mass) const {
    const double t = cX<N1>(K);
    const double a00 = fma(fma(k00[2], t, k00[1]), t, k00[0]);
    const double a11 = fma(fma(k11[2], t, k11[1]), t, k11[0]);
    const double a01 = fma(fma(k01[2], t, k01[1]), t, k01[0]);
    const double a02 = fma(k02[1], t, k02[0]);
    const double a12 = fma(k12[1], t, k12[0]);
    const double g0 = fma(a11, k22, -a12 * a12);
    const double g1 = fma(a02, a12, -a01 * k22);
    const double g2 = fma(a01, a12, -a02 * a11);
    const double g3 = fma(a00, k22, -a02 * a02);
    const double g4 = fma(a01, a02, -a00 * a12);
    const double g5 = fma(a00, a11, -a01 * a01);
    double scale;
    mass = 0.0;
    if (MERGED) {
      scale = __ldg(lam_a + nodeidx);
      mass = __ldg(lam_b + nodeidx);
    } else if (PARTIAL) {
      scale = __ldg(lam_a + nodeidx);
    } else {
      const double dt = fma(fma(det[2], t, det[1]), t, det[0]);
      const double lam_geo = (0.125 * ((cW<N1>(K) * wj) * wi)) * rcp_fast(dt);
      if (HELM) {
        const double l0 = lam_a ? __ldg(lam_a + nodeidx) : l0v;
        const double l1 = lam_b ? __ldg(lam_b + nodeidx) : l1v;
        scale = l0 * lam_geo;
        mass = l1 * (lam_geo * (0.015625 * dt * dt));
      } else {
        scale = lam_geo;
      }
    }
    const double s0 = scale * x0, s1 = scale * x1, s2 = scale * x2;
    rr = fma(g0, s0, fma(g1, s1, g2 * s2));
    ss = fma(g1, s0, fma(g3, s1, g4 * s2));
    tt = fma(g2, s0, fma(g4, s1, g5 * s2));
  }
};

// Stored (Nek-style) factors: 6 (+gwj) SoA loads per node (axlocal.py:181-185).
template <bool HELM>
struct StoredLoad {
  const double* g;
  const double* gwj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ void prepare(const hx_axlocal_args& a, int64_t e, const double*, Fibre) {
    g = a.g + e * 6 * N3;
    gwj = HELM ? a.gwj + e * N3 : nullptr;
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  template <int K>
  __device__ __forceinline__ void node(int n, double x0, double x1, double x2, double& rr, double& ss, double& tt,
                                       double& mass) const {
    const double g0 = __ldg(g + 0 * N3 + n), g1 = __ldg(g + 1 * N3 + n), g2 = __ldg(g + 2 * N3 + n);
    const double g3 = __ldg(g + 3 * N3 + n), g4 = __ldg(g + 4 * N3 + n), g5 = __ldg(g + 5 * N3 + n);
    rr = fma(g0, x0, fma(g1, x1, g2 * x2));
    ss = fma(g1, x0, fma(g3, x1, g4 * x2));
    tt = fma(g2, x0, fma(g4, x1, g5 * x2));
    mass = 0.0;
    if (HELM) {
      const double l0 = lam0 ? __ldg(lam0 + n) : l0v;
      rr *= l0;
      ss *= l0;
      tt *= l0;
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * __ldg(gwj + n);
    }
  }
};

// Parallelepiped: w (x) h (geometry.py:389-398).
template <bool HELM>
struct Ppd {
  double h[7];
  double wj, wi;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ void prepare(const hx_axlocal_args& a, int64_t e, const double*, Fibre f) {
#pragma unroll
    for (int q = 0; q < 7; ++q) h[q] = __ldg(a.h + e * 7 + q);
    wj = cW<N1>(f.j);
    wi = cW<N1>(f.i);
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  template <int K>
  __device__ __forceinline__ void node(int n, double x0, double x1, double x2, double& rr, double& ss, double& tt,
                                       double& mass) const {
    const double w = (cW<N1>(K) * wj) * wi;
    const double s0 = w * x0, s1 = w * x1, s2 = w * x2;
    rr = fma(h[0], s0, fma(h[1], s1, h[2] * s2));
    ss = fma(h[1], s0, fma(h[3], s1, h[4] * s2));
    tt = fma(h[2], s0, fma(h[4], s1, h[5] * s2));
    mass = 0.0;
    if (HELM) {
      const double l0 = lam0 ? __ldg(lam0 + n) : l0v;
      rr *= l0;
      ss *= l0;
      tt *= l0;
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * (w * h[6]);
    }
  }
};

template <typename F, int NCOL, bool HELM, bool NEED_VERTS, int MINB>
__global__ void __launch_bounds__(64, MINB) ax8(const hx_axlocal_args a) {
  __shared__ double sX[CUBE];
  __shared__ double sA[CUBE];
  __shared__ double sB[CUBE];
  __shared__ double sV[24];
  const int t = threadIdx.x;
  const int64_t e = blockIdx.x;
  // k-fibre (i, j); i-row (j = t&7, k = t>>3); j-column (i = t&7, k = t>>3)
  const int fi = t & 7, fj = t >> 3;
  const int kp = Aj(fj) + fi;                  // + Ak(k)
  const int rb = Ak(t >> 3) + Aj(t & 7);       // + n
  const int cb = Ak(t >> 3) + (t & 7);         // + Aj(n)
  if (NEED_VERTS && t < 24) sV[t] = __ldg(a.verts + e * 24 + t);

#pragma unroll 1
  for (int c = 0; c < NCOL; ++c) {
    double xk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) xk[k] = __ldg(a.x + (e * N3 + k * 64 + fj * 8 + fi) * NCOL + c);
#pragma unroll
    for (int k = 0; k < 8; ++k) sX[Ak(k) + kp] = xk[k];
    __syncthreads();

    F fac;
    fac.prepare(a, e, sV, Fibre{fi, fj});

    // forward: x2 on the k-fibre; x0 on the i-row; x1 on the j-column
    double x2[8];
    eo8<0>(xk, x2);
    {
      double v[8], o[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sX[rb + n];
      eo8<0>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sA[rb + n] = o[n];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sX[cb + Aj(n)];
      eo8<0>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sB[cb + Aj(n)] = o[n];
    }
    __syncthreads();

    // nodewise factor stage on the k-fibre, in place (each address owned by one thread)
    double tt[8], yk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int adr = Ak(k) + kp;
      const double x0 = sA[adr], x1 = sB[adr];
      double rr, ss, mass;
      switch (k) {
#define HX_NODE(K) \
  case K:          \
    fac.template node<K>(K * 64 + fj * 8 + fi, x0, x1, x2[K], rr, ss, tt[K], mass); \
    break;
        HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
      }
      sA[adr] = rr;
      sB[adr] = ss;
      yk[k] = HELM ? mass * xk[k] : 0.0;
    }
    double yt[8];
    eo8<1>(tt, yt);
    __syncthreads();

    // transposed: D^T rr on the i-row, D^T ss on the j-column, in place
    {
      double v[8], o[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sA[rb + n];
      eo8<1>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sA[rb + n] = o[n];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sB[cb + Aj(n)];
      eo8<1>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sB[cb + Aj(n)] = o[n];
    }
    __syncthreads();

#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int adr = Ak(k) + kp;
      const double y = (sA[adr] + sB[adr]) + yt[k] + yk[k];
      a.y[(e * N3 + k * 64 + fj * 8 + fi) * NCOL + c] = y;
    }
  }
}

// MINB = resident CTAs per SM the register budget is sized for (64 threads
// each): 6 -> <= 168 registers, 8 -> <= 128.
template <typename F, bool HELM, bool NEED_VERTS, int MINB = 6>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  if (a.n_elements > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)a.n_elements;
  if (a.n_col == 3)
    ax8<F, 3, HELM, NEED_VERTS, MINB><<<grid, 64, 0, s>>>(a);
  else
    ax8<F, 1, HELM, NEED_VERTS, MINB><<<grid, 64, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fast
}  // namespace hx

extern "C" cudaError_t hx_fast_launch(const hx_axlocal_args* a, cudaStream_t s) {
  using namespace hx::fast;
  if (a->order != 7) return cudaErrorNotSupported;
  const bool helm = a->equation == HX_HELMHOLTZ;
  switch (a->factor_source) {
    case HX_TRILINEAR:
      if (helm) return launch<TrilinearPoly<true, false, false>, true, true>(*a, s);
      // tuning hook (reserved != 0): alternative register budgets
      switch (a->reserved) {
        case 4: return launch<TrilinearPoly<false, false, false>, false, true, 4>(*a, s);
        case 5: return launch<TrilinearPoly<false, false, false>, false, true, 5>(*a, s);
        case 8: return launch<TrilinearPoly<false, false, false>, false, true, 8>(*a, s);
        default: return launch<TrilinearPoly<false, false, false>, false, true>(*a, s);
      }
    case HX_TRILINEAR_PARTIAL:
      return launch<TrilinearPoly<false, false, true>, false, true>(*a, s);
    case HX_TRILINEAR_MERGED:
      return launch<TrilinearPoly<true, true, false>, true, true>(*a, s);
    case HX_STORED:
      return helm ? launch<StoredLoad<true>, true, false>(*a, s) : launch<StoredLoad<false>, false, false>(*a, s);
    case HX_PARALLELEPIPED:
      return helm ? launch<Ppd<true>, true, false>(*a, s) : launch<Ppd<false>, false, false>(*a, s);
  }
  return cudaErrorNotSupported;
}

// Basis upload hook: the common constants plus, for n1 = 8, the even-odd blocks.
extern "C" cudaError_t hx_upload_basis_fast(int n1, const double* pts, const double* w, const double* d) {
  cudaError_t err = hx_upload_basis_local(n1, pts, w, d);
  if (err != cudaSuccess || n1 != 8) return err;
  double eo[2][2][4][4];
  for (int T = 0; T < 2; ++T)
    for (int i = 0; i < 4; ++i)
      for (int m = 0; m < 4; ++m) {
        const double a = T ? d[m * 8 + i] : d[i * 8 + m];            // M[i][m]
        const double b = T ? d[(7 - m) * 8 + i] : d[i * 8 + 7 - m];  // M[i][7-m]
        eo[T][0][i][m] = 0.5 * (a + b);
        eo[T][1][i][m] = 0.5 * (a - b);
      }
  return cudaMemcpyToSymbol(c_EO, eo, sizeof(eo));
}
