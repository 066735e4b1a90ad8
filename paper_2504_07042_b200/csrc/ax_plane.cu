// AxLocal at orders 2 and 3 (n1 = 3, 4; compiled once per n1 with -DHX_N1=n1):
// one thread per j-plane of an element, the element in registers.
//
// The order-generic kernel (ax_fastn.cu) moves the element through three
// shared cubes and is bound by shared-memory wavefronts at small orders (ncu at
// N = 4: l1tex 86 %, FP64 54 %, 241 wavefronts per element); an element of
// order 2 or 3 is small enough to live in the registers of n1 threads instead.
// Thread j of an element (n1 consecutive lanes) owns the n1^2 nodes (i, j, k):
//   * r direction (over i) and t direction (over k): inside the thread, D and
//     D^T with compile-time indices (constant-bank operands);
//   * s direction (over j): across the element's n1 lanes by warp shuffles of
//     64-bit values, n1 - 1 per node and direction, with the thread's own row /
//     column of D in registers;
//   * geometry (Algorithm 2) fibre by fibre: the thread's n1
//     k-fibres (i = 0..n1-1, j) as polynomials in t, one fibre's coefficients
//     live at a time.
// 32 / n1 elements per warp (n1 = 3: lanes 30, 31 idle), no shared memory, no
// barriers.  n_col = 3 runs each column in its own CTA row (blockIdx.y) with the
// n_col = 1 arithmetic, so n_col = 3 == 3 x n_col = 1 bitwise.  At n1 = 5 the 25
// nodes per thread exhaust the register file (parallelepiped 138 vs 181 GDOF/s
// for the order-generic kernel, measured); orders 4 and up stay there.
#include "hx_common.cuh"

#ifndef HX_N1
#error "compile with -DHX_N1=<points per direction>"
#endif

#define HX_CAT2(a, b) a##b
#define HX_CAT(a, b) HX_CAT2(a, b)

// D (row-major [i][m]) for lane-dependent indices (the thread's own row / column
// for the shuffled s direction); loaded once per thread through L1.
static __device__ double g_Dp[HX_N1 * HX_N1];
static __device__ double g_Xp[HX_N1];
static __device__ double g_Wp[HX_N1];

namespace hx {
namespace plane {
namespace {

constexpr int N1 = HX_N1;
constexpr int N2 = N1 * N1;
constexpr int N3 = N1 * N2;
constexpr int EPW = 32 / N1;  // elements per warp
constexpr int WPB = 4;        // warps per CTA
constexpr int EPB = EPW * WPB;

__device__ __forceinline__ double dot3(const double* u, const double* v) {
  return fma(u[2], v[2], fma(u[1], v[1], u[0] * v[0]));
}

// out = M v along a fibre in registers, M = D (TR = false) or D^T (TR = true)
template <bool TR>
__device__ __forceinline__ void contract(const double v[N1], double out[N1]) {
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double s = (TR ? cD<N1>(0, i) : cD<N1>(i, 0)) * v[0];
#pragma unroll
    for (int m = 1; m < N1; ++m) s = fma(TR ? cD<N1>(m, i) : cD<N1>(i, m), v[m], s);
    out[i] = s;
  }
}

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// Lane context: element e, plane j, first lane of the element's group.
struct Lane {
  int64_t e;
  int j, base;
  bool valid;
};

// (rr, ss, tt) = G (s x0, s x1, s x2), G symmetric (the reference's row order)
__device__ __forceinline__ void symv(const double g[6], double s, double x0, double x1, double x2, double& rr,
                                     double& ss, double& tt) {
  const double s0 = s * x0, s1 = s * x1, s2 = s * x2;
  rr = fma(g[0], s0, fma(g[1], s1, g[2] * s2));
  ss = fma(g[1], s0, fma(g[3], s1, g[4] * s2));
  tt = fma(g[2], s0, fma(g[4], s1, g[5] * s2));
}

__device__ __forceinline__ double div_fast(double w, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  const double wr = w * r;
  return fma(fma(e, e, e), wr, wr);
}

// ---------------------------------------------------------------------------
// Factor policies (axlocal.py:171-211).  elem() once per thread; fibre<I>() before
// the nodes of k-fibre (I, j); node<K, I>() per node.

// Trilinear recompute (geometry.py:135-184, 304-351) as polynomials in t per fibre;
// HELM: lam0 / lam1 scale and mass; PARTIAL: stored lam_geo; MERGED: stored lam2 / lam3.
template <bool HELM, bool PARTIAL, bool MERGED>
struct Tri {
  static constexpr bool kVerts = true;
  // element terms (this thread's j): j-side base / slope, dt-column U / V, K00 poly,
  // and the vertex differences the i-side terms need
  double br[3], sr[3], U[3], V[3], k00[3], dq[12], xj, wj;
  // the current fibre
  double k01[3], k02[2], k12[2], k22, det[3], k11[3], wji8;
  const double* pa;
  const double* pb;
  double l0v, l1v;
  __device__ __forceinline__ void elem(const hx_axlocal_args& a, const Lane& L, const double* v) {
    xj = g_Xp[L.j];
    wj = g_Wp[L.j];
    const double a0 = 1.0 - xj, a1 = 1.0 + xj;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double lo = fma(a1, v[9 + c] - v[6 + c], a0 * (v[3 + c] - v[c]));      // a0 (v1-v0) + a1 (v3-v2)
      const double hi = fma(a1, v[21 + c] - v[18 + c], a0 * (v[15 + c] - v[12 + c]));  // a0 (v5-v4) + a1 (v7-v6)
      br[c] = lo + hi;
      sr[c] = hi - lo;
      const double l = fma(a1, v[18 + c] - v[6 + c], a0 * (v[12 + c] - v[c]));     // a0 (v4-v0) + a1 (v6-v2)
      const double r = fma(a1, v[21 + c] - v[9 + c], a0 * (v[15 + c] - v[3 + c]));  // a0 (v5-v1) + a1 (v7-v3)
      U[c] = l + r;
      V[c] = r - l;
      dq[c] = v[6 + c] - v[c];             // v2 - v0
      dq[3 + c] = v[9 + c] - v[3 + c];     // v3 - v1
      dq[6 + c] = v[18 + c] - v[12 + c];   // v6 - v4
      dq[9 + c] = v[21 + c] - v[15 + c];   // v7 - v5
    }
    k00[0] = dot3(br, br);
    k00[1] = 2.0 * dot3(br, sr);
    k00[2] = dot3(sr, sr);
    pa = pb = nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
    if (PARTIAL) {
      pa = a.lam_geo + L.e * N3;
    } else if (MERGED) {
      pa = a.lam2 + L.e * N3;
      pb = a.lam3 + L.e * N3;
    } else if (HELM) {
      pa = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
      pb = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
    }
  }
  template <int I>
  __device__ __forceinline__ void fibre() {
    const double xi = cX<N1>(I), a0 = 1.0 - xi, a1 = 1.0 + xi;
    double bs[3], ss[3], c[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double lo = fma(a1, dq[3 + q], a0 * dq[q]);      // a0 (v2-v0) + a1 (v3-v1)
      const double hi = fma(a1, dq[9 + q], a0 * dq[6 + q]);  // a0 (v6-v4) + a1 (v7-v5)
      bs[q] = lo + hi;
      ss[q] = hi - lo;
      c[q] = fma(xi, V[q], U[q]);
    }
    k11[0] = dot3(bs, bs);
    k11[1] = 2.0 * dot3(bs, ss);
    k11[2] = dot3(ss, ss);
    k01[0] = dot3(br, bs);
    k01[1] = dot3(br, ss) + dot3(sr, bs);
    k01[2] = dot3(sr, ss);
    k02[0] = dot3(br, c);
    k02[1] = dot3(sr, c);
    k12[0] = dot3(bs, c);
    k12[1] = dot3(ss, c);
    k22 = dot3(c, c);
    if (!PARTIAL && !MERGED) {
      const double P[3] = {fma(bs[1], c[2], -(bs[2] * c[1])), fma(bs[2], c[0], -(bs[0] * c[2])),
                           fma(bs[0], c[1], -(bs[1] * c[0]))};
      const double Q[3] = {fma(ss[1], c[2], -(ss[2] * c[1])), fma(ss[2], c[0], -(ss[0] * c[2])),
                           fma(ss[0], c[1], -(ss[1] * c[0]))};
      det[0] = dot3(br, P);
      det[1] = dot3(br, Q) + dot3(sr, P);
      det[2] = dot3(sr, Q);
      wji8 = 0.125 * (wj * cW<N1>(I));
    }
  }
  template <int K, int I>
  __device__ __forceinline__ void node(const Lane& L, double x0, double x1, double x2, double& rr, double& ss,
                                       double& tt, double& mass) const {
    const double t = cX<N1>(K);
    const double a00 = fma(fma(k00[2], t, k00[1]), t, k00[0]);
    const double a11 = fma(fma(k11[2], t, k11[1]), t, k11[0]);
    const double a01 = fma(fma(k01[2], t, k01[1]), t, k01[0]);
    const double a02 = fma(k02[1], t, k02[0]);
    const double a12 = fma(k12[1], t, k12[0]);
    double g[6];
    g[0] = fma(a11, k22, -a12 * a12);
    g[1] = fma(a02, a12, -a01 * k22);
    g[2] = fma(a01, a12, -a02 * a11);
    g[3] = fma(a00, k22, -a02 * a02);
    g[4] = fma(a01, a02, -a00 * a12);
    g[5] = fma(a00, a11, -a01 * a01);
    const int n = K * N2 + L.j * N1 + I;
    double scale;
    mass = 0.0;
    if (MERGED) {
      scale = __ldg(pa + n);
      mass = __ldg(pb + n);
    } else if (PARTIAL) {
      scale = __ldg(pa + n);
    } else {
      const double dt = fma(fma(det[2], t, det[1]), t, det[0]);
      const double lam = div_fast(cW<N1>(K) * wji8, dt);  // 0.125 w / det(JT)
      if (HELM) {
        const double l0 = pa ? __ldg(pa + n) : l0v;
        const double l1 = pb ? __ldg(pb + n) : l1v;
        scale = l0 * lam;
        mass = l1 * (lam * (0.015625 * (dt * dt)));
      } else {
        scale = lam;
      }
    }
    symv(g, scale, x0, x1, x2, rr, ss, tt);
  }
};

// Stored (Nek-style) factors: 6 (+gwj) SoA loads per node (axlocal.py:181-185).
template <bool HELM>
struct Stored {
  static constexpr bool kVerts = false;
  const double* gp;
  const double* gwj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void elem(const hx_axlocal_args& a, const Lane& L, const double*) {
    gp = a.g + L.e * 6 * N3;
    gwj = HELM ? a.gwj + L.e * N3 : nullptr;
    lam0 = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  template <int I>
  __device__ __forceinline__ void fibre() {}
  template <int K, int I>
  __device__ __forceinline__ void node(const Lane& L, double x0, double x1, double x2, double& rr, double& ss,
                                       double& tt, double& mass) const {
    const int n = K * N2 + L.j * N1 + I;
    double g[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) g[q] = __ldg(gp + q * N3 + n);
    rr = fma(g[0], x0, fma(g[1], x1, g[2] * x2));
    ss = fma(g[1], x0, fma(g[3], x1, g[4] * x2));
    tt = fma(g[2], x0, fma(g[4], x1, g[5] * x2));
    mass = 0.0;
    if (HELM) {
      const double l0 = lam0 ? __ldg(lam0 + n) : l0v;
      rr = __dmul_rn(rr, l0);
      ss = __dmul_rn(ss, l0);
      tt = __dmul_rn(tt, l0);
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * __ldg(gwj + n);
    }
  }
};

// Parallelepiped: g = w (x) h (geometry.py:389-398).
template <bool HELM>
struct Ppd {
  static constexpr bool kVerts = false;
  double h[7], wj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void elem(const hx_axlocal_args& a, const Lane& L, const double*) {
#pragma unroll
    for (int q = 0; q < 7; ++q) h[q] = __ldg(a.h + L.e * 7 + q);
    wj = g_Wp[L.j];
    lam0 = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  template <int I>
  __device__ __forceinline__ void fibre() {}
  template <int K, int I>
  __device__ __forceinline__ void node(const Lane& L, double x0, double x1, double x2, double& rr, double& ss,
                                       double& tt, double& mass) const {
    const double w = (cW<N1>(K) * wj) * cW<N1>(I);
    symv(h, w, x0, x1, x2, rr, ss, tt);
    mass = 0.0;
    if (HELM) {
      const int n = K * N2 + L.j * N1 + I;
      const double l0 = lam0 ? __ldg(lam0 + n) : l0v;
      rr = __dmul_rn(rr, l0);
      ss = __dmul_rn(ss, l0);
      tt = __dmul_rn(tt, l0);
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * (w * h[6]);
    }
  }
};

// compile-time loops over the thread's nodes: fibre I (outer), k = K (inner)
template <typename F, int I, int K>
struct Nodes {
  __device__ __forceinline__ static void run(F& fac, const Lane& L, double (*x0)[N1], double (*x1)[N1],
                                             double (*x2)[N1], const double (*xk)[N1], double (*ms)[N1]) {
    if constexpr (K == 0) fac.template fibre<I>();
    double rr, ss, tt, mass;
    fac.template node<K, I>(L, x0[K][I], x1[K][I], x2[K][I], rr, ss, tt, mass);
    x0[K][I] = rr;
    x1[K][I] = ss;
    x2[K][I] = tt;
    ms[K][I] = __dmul_rn(mass, xk[K][I]);
    if constexpr (K + 1 < N1)
      Nodes<F, I, K + 1>::run(fac, L, x0, x1, x2, xk, ms);
    else if constexpr (I + 1 < N1)
      Nodes<F, I + 1, 0>::run(fac, L, x0, x1, x2, xk, ms);
  }
};

// MINB: resident CTAs of 128 threads per SM the register budget is sized for
// (1: up to 255 registers; 3: 168).  Measured per order and source (A/B in
// profiles/r02_plane_ab.txt): the N = 3 trilinear sources keep 255 registers,
// everything else runs faster at 168.
template <typename F, int NCOL, bool HELM, int MINB>
__global__ void __launch_bounds__(32 * WPB, MINB) axp(const __grid_constant__ hx_axlocal_args a) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int slot = lane / N1;
  Lane L;
  L.j = lane - slot * N1;
  L.base = lane - L.j;
  const int64_t e_raw = ((int64_t)blockIdx.x * WPB + w) * EPW + slot;
  L.valid = slot < EPW && e_raw < a.n_elements;
  L.e = L.valid ? e_raw : 0;
  const int c = NCOL > 1 ? (int)blockIdx.y : 0;
  const int j = L.j;

  // x of the plane: [k][i]
  double xk[N1][N1];
#pragma unroll
  for (int k = 0; k < N1; ++k)
#pragma unroll
    for (int i = 0; i < N1; ++i) xk[k][i] = __ldg(a.x + (L.e * N3 + k * N2 + j * N1 + i) * NCOL + c);
  // the thread's row and column of D for the shuffled s direction, by lane offset d:
  // partner plane (j + d) mod n1
  double Drow[N1], Dcol[N1];
#pragma unroll
  for (int d = 0; d < N1; ++d) {
    const int m = (j + d) % N1;
    Drow[d] = g_Dp[j * N1 + m];  // D[j][m]
    Dcol[d] = g_Dp[m * N1 + j];  // D[m][j]
  }
  F fac;
  double vtx[24];
  if constexpr (F::kVerts) {
#pragma unroll
    for (int q = 0; q < 12; ++q) {
      const double2 p = __ldg(reinterpret_cast<const double2*>(a.verts + L.e * 24) + q);
      vtx[2 * q] = p.x;
      vtx[2 * q + 1] = p.y;
    }
  }
  fac.elem(a, L, vtx);

  // forward: x1 = D_s x (shuffles over the element's lanes), x0 = D_r x, x2 = D_t x
  double x0[N1][N1], x1[N1][N1], x2[N1][N1];
#pragma unroll
  for (int k = 0; k < N1; ++k)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double s = Drow[0] * xk[k][i];
#pragma unroll
      for (int d = 1; d < N1; ++d) s = fma(Drow[d], shfl(xk[k][i], L.base + (j + d) % N1), s);
      x1[k][i] = s;
    }
#pragma unroll
  for (int k = 0; k < N1; ++k) contract<false>(xk[k], x0[k]);
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double v[N1], o[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) v[k] = xk[k][i];
    contract<false>(v, o);
#pragma unroll
    for (int k = 0; k < N1; ++k) x2[k][i] = o[k];
  }
  // node stage, fibre by fibre (rr, ss, tt overwrite x0, x1, x2)
  double ms[N1][N1];
  Nodes<F, 0, 0>::run(fac, L, x0, x1, x2, xk, ms);

  // transposed: y = (D_r^T rr + D_s^T ss) + D_t^T tt [+ mass x]
  double y[N1][N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) contract<true>(x0[k], y[k]);
#pragma unroll
  for (int k = 0; k < N1; ++k)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double s = Dcol[0] * x1[k][i];
#pragma unroll
      for (int d = 1; d < N1; ++d) s = fma(Dcol[d], shfl(x1[k][i], L.base + (j + d) % N1), s);
      y[k][i] = y[k][i] + s;
    }
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double v[N1], o[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) v[k] = x2[k][i];
    contract<true>(v, o);
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double r = y[k][i] + o[k];
      if (HELM) r = __dadd_rn(r, ms[k][i]);
      y[k][i] = r;
    }
  }
  if (L.valid) {
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int i = 0; i < N1; ++i) a.y[(L.e * N3 + k * N2 + j * N1 + i) * NCOL + c] = y[k][i];
  }
}

#ifndef HX_PLANE_MINB_TRI4
#define HX_PLANE_MINB_TRI4 1
#endif
template <typename F, bool HELM>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  constexpr int MINB = (F::kVerts && N1 == 4) ? HX_PLANE_MINB_TRI4 : 3;
  const int64_t blocks = (a.n_elements + EPB - 1) / EPB;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)blocks, a.n_col);
  if (a.n_col == 3)
    axp<F, 3, HELM, MINB><<<grid, 32 * WPB, 0, s>>>(a);
  else
    axp<F, 1, HELM, MINB><<<grid, 32 * WPB, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace
}  // namespace plane
}  // namespace hx

// Every (equation, factor source, n_col) at order HX_N1 - 1, element-local x.
extern "C" cudaError_t HX_CAT(hx_plane_launch_, HX_N1)(const hx_axlocal_args* a, cudaStream_t s) {
  using namespace hx::plane;
  if (a->order + 1 != N1 || a->gather) return cudaErrorNotSupported;
  const bool helm = a->equation == HX_HELMHOLTZ;
  switch (a->factor_source) {
    case HX_TRILINEAR:
    case HX_TRILINEAR_PARTIAL:
    case HX_TRILINEAR_MERGED:
      if constexpr (N1 <= 4) {
        if (a->factor_source == HX_TRILINEAR_PARTIAL) return launch<Tri<false, true, false>, false>(*a, s);
        if (a->factor_source == HX_TRILINEAR_MERGED) return launch<Tri<true, false, true>, true>(*a, s);
        return helm ? launch<Tri<true, false, false>, true>(*a, s) : launch<Tri<false, false, false>, false>(*a, s);
      }
      return cudaErrorNotSupported;
    case HX_STORED:
      return helm ? launch<Stored<true>, true>(*a, s) : launch<Stored<false>, false>(*a, s);
    case HX_PARALLELEPIPED:
      return helm ? launch<Ppd<true>, true>(*a, s) : launch<Ppd<false>, false>(*a, s);
  }
  return cudaErrorNotSupported;
}

extern "C" cudaError_t HX_CAT(hx_upload_basis_plane_, HX_N1)(int n1, const double* pts, const double* w,
                                                            const double* d) {
  cudaError_t err = hx_upload_basis_local(n1, pts, w, d);
  if (err != cudaSuccess || n1 != HX_N1) return err;
  err = cudaMemcpyToSymbol(g_Dp, d, sizeof(double) * HX_N1 * HX_N1);
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(g_Xp, pts, sizeof(double) * HX_N1);
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(g_Wp, w, sizeof(double) * HX_N1);
  return err;
}
