// Specialised AxLocal kernel for N = 7 (n1 = 8), the north-star order.
//
// Persistent 64-thread CTAs, one element at a time, the next element's x (and
// vertices) prefetched by a 1-D bulk async copy (TMA, cp.async.bulk) into a
// double-buffered landing zone tracked by mbarriers.  The FP64 pipe (DFMA and
// DMMA share it on B200, tools/ubench_fp64.cu) is the bound, so the design
// minimises FP64 operations and keeps shared memory below the pipe time:
//
//  * contractions by even-odd decomposition: D and D^T are centro-
//    antisymmetric on GLL points, so an 8-point contraction is 8 adds + two
//    4x4 products + 8 adds = 48 ops instead of 64, the 4x4 blocks read as
//    __constant__ operands at compile-time offsets;
//  * three fibre ownerships per element (k-fibres, i-rows, j-columns); the
//    cube moves between them through shared memory laid out as
//    a(k,j,i) = Ak[k] + Aj[j] + i with lane->fibre maps chosen so every
//    64-bit access of every phase hits 16 distinct bank pairs per half-warp
//    (no conflicts; DESIGN.md derives it) — including the k-fibre read of the
//    linear TMA landing buffer;
//  * trilinear geometry (Algorithm 2) as polynomials in the
//    reference coordinate t along each k-fibre: K00, K01, K11 quadratic, K02,
//    K12 linear, K22 constant and det(JT) quadratic, so a node costs 8 FMAs
//    for K, 12 for adj(K), 2 for det and a MUFU reciprocal with one cubic
//    correction; the per-element pieces that depend on j only or i only are
//    computed once per element and shared through shared memory.
//
// The arithmetic differs from the reference's operation order, so parity is
// to the 1e-12 relative bar, not bitwise; per-column arithmetic is identical
// for n_col = 1 and 3, so n_col=3 == 3 x n_col=1 bitwise.
#include "n7_common.cuh"

namespace hx {
namespace fast {

constexpr int CUBE = 544;  // 543 used
#ifndef HX_PREFETCH_AHEAD
#define HX_PREFETCH_AHEAD 2368
#endif
constexpr int64_t kPrefetchAhead = HX_PREFETCH_AHEAD;  // ~1.6-2 waves of resident CTAs

__host__ __device__ constexpr int Aj(int j) { return 17 * (j >> 1) + 8 * (j & 1); }
__host__ __device__ constexpr int Ak(int k) { return 68 * k; }

// lane -> fibre maps
struct Roles {
  int fi, fj;  // k-fibre (i, j)
  int rj, rk;  // i-row (j, k)
  int ci, ck;  // j-column (i, k)
};

__device__ __forceinline__ Roles roles(int t) {
  const int w = t >> 5, l = t & 31, h = l >> 4, p = (l >> 3) & 1, q = l & 15;
  Roles r;
  r.fi = l & 7;
  r.fj = 4 * w + 2 * h + p;
  r.rj = 2 * (q & 3) + h;
  r.rk = 4 * w + (q >> 2);
  r.ci = l & 7;
  r.ck = 4 * w + h + 2 * p;
  return r;
}

// ---------------------------------------------------------------------------
// factor policies: prepare() once per element (after TriShared is written),
// node<K>(...) per node of the k-fibre.

// Trilinear recompute (geometry.py:304-351; axlocal.py:191-211), polynomial in t.
template <bool HELM, bool MERGED, bool PARTIAL, bool SHARED = true, bool LAMFIRST = false, bool TTSMEM = false,
          bool TAB = false>
struct TrilinearPoly {
  static constexpr bool kStageA = SHARED;
  static constexpr bool kScaleFirst = LAMFIRST;
  static constexpr bool kTtSmem = TTSMEM;
  // TAB: K00(j,k) and K11(i,k) are evaluated once per element into shared
  // tables (each thread fills one entry of each) instead of per fibre node.
  double k00[3], k11[3], k01[3], k02[2], k12[2], k22, det[3];
  const double* tab00;  // &t00[fj][0]
  const double* tab11;  // &t11[fi][0]
  double wji8;
  const double* lam_a;  // partial: lam_geo; merged: lam2; trilinear-helm: lam0 (or null)
  const double* lam_b;  // merged: lam3; trilinear-helm: lam1 (or null)
  double l0v, l1v;

  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, int64_t e, const TriShared& s,
                                          const double* sv, int fi, int fj) {
    double br[3], sr[3], bs[3], ss[3], c[3];
    tab00 = s.t00[fj];
    tab11 = s.t11[fi];
    if (SHARED) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        br[q] = s.j[fj][q];
        sr[q] = s.j[fj][3 + q];
        bs[q] = s.i[fi][q];
        ss[q] = s.i[fi][3 + q];
      }
    } else {
      TrilinearPencil p;
      trilinear_pencil(sv, xr(fi), xr(fj), p);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        br[q] = p.dr_base[q];
        sr[q] = p.dr_slope[q];
        bs[q] = p.ds_base[q];
        ss[q] = p.ds_slope[q];
      }
    }
    if (TAB) {
      // this thread's entries: K00(j = fj, k = fi) and K11(i = fi, k = fj)
      TriShared& w = const_cast<TriShared&>(s);
      const double tk = SHARED ? s.xs[fi] : xr(fi), tj = SHARED ? s.xs[fj] : xr(fj);
      double cr[3], cs[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        cr[q] = br[q] + tk * sr[q];
        cs[q] = bs[q] + tj * ss[q];
      }
      w.t00[fj][fi] = dot3(cr, cr);
      w.t11[fi][fj] = dot3(cs, cs);
    } else {
      k00[0] = dot3(br, br);
      k00[1] = 2.0 * dot3(br, sr);
      k00[2] = dot3(sr, sr);
      k11[0] = dot3(bs, bs);
      k11[1] = 2.0 * dot3(bs, ss);
      k11[2] = dot3(ss, ss);
    }
    if (SHARED) {
      const double xj = s.xs[fj], xi = s.xs[fi];
      const double a0j = 1.0 - xj, a1j = 1.0 + xj, a0i = 1.0 - xi, a1i = 1.0 + xi;
      const double w00 = a0j * a0i, w01 = a0j * a1i, w10 = a1j * a0i, w11 = a1j * a1i;
#pragma unroll
      for (int q = 0; q < 3; ++q) c[q] = w00 * s.d[q] + w01 * s.d[3 + q] + w11 * s.d[6 + q] + w10 * s.d[9 + q];
    } else {
      const double xj = xr(fj), xi = xr(fi);
      const double a0j = 1.0 - xj, a1j = 1.0 + xj, a0i = 1.0 - xi, a1i = 1.0 + xi;
      const double w00 = a0j * a0i, w01 = a0j * a1i, w10 = a1j * a0i, w11 = a1j * a1i;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        c[q] = w00 * (sv[12 + q] - sv[q]) + w01 * (sv[15 + q] - sv[3 + q]) + w11 * (sv[21 + q] - sv[9 + q]) +
               w10 * (sv[18 + q] - sv[6 + q]);
    }
    k01[0] = dot3(br, bs);
    k01[1] = dot3(br, ss) + dot3(sr, bs);
    k01[2] = dot3(sr, ss);
    k02[0] = dot3(br, c);
    k02[1] = dot3(sr, c);
    k12[0] = dot3(bs, c);
    k12[1] = dot3(ss, c);
    k22 = dot3(c, c);
    // det(JT) = (br + t sr) . ((bs + t ss) x c)
    const double P[3] = {bs[1] * c[2] - bs[2] * c[1], bs[2] * c[0] - bs[0] * c[2], bs[0] * c[1] - bs[1] * c[0]};
    const double Q[3] = {ss[1] * c[2] - ss[2] * c[1], ss[2] * c[0] - ss[0] * c[2], ss[0] * c[1] - ss[1] * c[0]};
    det[0] = dot3(br, P);
    det[1] = dot3(br, Q) + dot3(sr, P);
    det[2] = dot3(sr, Q);
    wji8 = SHARED ? 0.125 * (s.ws[fj] * s.ws[fi]) : 0.125 * (wr(fj) * wr(fi));
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

  // Per-node scale (grad_scale) and mass coefficient; independent of x.
  template <int K>
  __device__ __forceinline__ void scale_at(int n, double& scale, double& mass) const {
    const double t = cX<N1>(K);
    mass = 0.0;
    if (MERGED) {
      scale = __ldg(lam_a + n);
      mass = __ldg(lam_b + n);
    } else if (PARTIAL) {
      scale = __ldg(lam_a + n);
    } else {
      const double dt = fma(fma(det[2], t, det[1]), t, det[0]);
      const double lam_geo = div_fast(cW<N1>(K) * wji8, dt);  // 0.125 w / det(JT)
      if (HELM) {
        const double l0 = lam_a ? __ldg(lam_a + n) : l0v;
        const double l1 = lam_b ? __ldg(lam_b + n) : l1v;
        scale = l0 * lam_geo;
        mass = l1 * (lam_geo * (0.015625 * dt * dt));
      } else {
        scale = lam_geo;
      }
    }
  }

  // adj(K(t_K)) entries (unscaled g of geometry.py:329-339).
  template <int K>
  __device__ __forceinline__ void adj_at(double g[6]) const {
    const double t = cX<N1>(K);
    const double a00 = TAB ? tab00[K] : fma(fma(k00[2], t, k00[1]), t, k00[0]);
    const double a11 = TAB ? tab11[K] : fma(fma(k11[2], t, k11[1]), t, k11[0]);
    const double a01 = fma(fma(k01[2], t, k01[1]), t, k01[0]);
    const double a02 = fma(k02[1], t, k02[0]);
    const double a12 = fma(k12[1], t, k12[0]);
    g[0] = fma(a11, k22, -a12 * a12);
    g[1] = fma(a02, a12, -a01 * k22);
    g[2] = fma(a01, a12, -a02 * a11);
    g[3] = fma(a00, k22, -a02 * a02);
    g[4] = fma(a01, a02, -a00 * a12);
    g[5] = fma(a00, a11, -a01 * a01);
  }

  // Factors of one node for multi-column application (see apply_factors):
  // rr = g . (sin x) [* sout], the same operation order as node().
  static constexpr bool kIn = true, kOut = false;
  template <int K>
  __device__ __forceinline__ void factors(int n, double g[6], double& sin, double& sout, double& mass) const {
    adj_at<K>(g);
    scale_at<K>(n, sin, mass);
    sout = 1.0;
  }

  // rr, ss, tt = scale * adj(K(t_K)) (x0, x1, x2).
  template <int K>
  __device__ __forceinline__ void apply_at(double scale, double x0, double x1, double x2, double& rr, double& ss,
                                           double& tt) const {
    const double t = cX<N1>(K);
    const double a00 = TAB ? tab00[K] : fma(fma(k00[2], t, k00[1]), t, k00[0]);
    const double a11 = TAB ? tab11[K] : fma(fma(k11[2], t, k11[1]), t, k11[0]);
    const double a01 = fma(fma(k01[2], t, k01[1]), t, k01[0]);
    const double a02 = fma(k02[1], t, k02[0]);
    const double a12 = fma(k12[1], t, k12[0]);
    const double g0 = fma(a11, k22, -a12 * a12);
    const double g1 = fma(a02, a12, -a01 * k22);
    const double g2 = fma(a01, a12, -a02 * a11);
    const double g3 = fma(a00, k22, -a02 * a02);
    const double g4 = fma(a01, a02, -a00 * a12);
    const double g5 = fma(a00, a11, -a01 * a01);
    const double s0 = scale * x0, s1 = scale * x1, s2 = scale * x2;
    rr = fma(g0, s0, fma(g1, s1, g2 * s2));
    ss = fma(g1, s0, fma(g3, s1, g4 * s2));
    tt = fma(g2, s0, fma(g4, s1, g5 * s2));
  }

  template <int K>
  __device__ __forceinline__ void node(int n, double x0, double x1, double x2, double& rr, double& ss, double& tt,
                                       double& mass) const {
    double scale;
    scale_at<K>(n, scale, mass);
    apply_at<K>(scale, x0, x1, x2, rr, ss, tt);
  }
};

// Stored (Nek-style) factors: 6 (+gwj) SoA loads per node (axlocal.py:181-185).
template <bool HELM>
struct StoredLoad {
  static constexpr bool kStageA = false;
  static constexpr bool kScaleFirst = false;
  static constexpr bool kTtSmem = false;
  const double* g;
  const double* gwj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, int64_t e, const TriShared&, const double*, int,
                                          int) {
    g = a.g + e * 6 * N3;
    gwj = HELM ? a.gwj + e * N3 : nullptr;
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  static constexpr bool kIn = false, kOut = HELM;  // rr = (g . x) * lam0 (axlocal.py:221-227 order)
  template <int K>
  __device__ __forceinline__ void factors(int n, double gg[6], double& sin, double& sout, double& mass) const {
#pragma unroll
    for (int q = 0; q < 6; ++q) gg[q] = __ldg(g + q * N3 + n);
    sin = sout = 1.0;
    mass = 0.0;
    if (HELM) {
      sout = lam0 ? __ldg(lam0 + n) : l0v;
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * __ldg(gwj + n);
    }
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
      // __dmul_rn: ptxas must not fuse tt * l0 into the next even-odd add (it can
      // where tt stays in registers, not where it is parked in shared memory)
      const double l0 = lam0 ? __ldg(lam0 + n) : l0v;
      rr = __dmul_rn(rr, l0);
      ss = __dmul_rn(ss, l0);
      tt = __dmul_rn(tt, l0);
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * __ldg(gwj + n);
    }
  }
};

// Parallelepiped: w (x) h (geometry.py:389-398).
template <bool HELM>
struct Ppd {
  static constexpr bool kStageA = false;
  static constexpr bool kScaleFirst = false;
  static constexpr bool kTtSmem = false;
  double h[7];
  double wj, wi;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, int64_t e, const TriShared&, const double*,
                                          int fi, int fj) {
#pragma unroll
    for (int q = 0; q < 7; ++q) h[q] = __ldg(a.h + e * 7 + q);
    wj = wr(fj);
    wi = wr(fi);
    lam0 = a.lam0 ? a.lam0 + e * N3 : nullptr;
    lam1 = a.lam1 ? a.lam1 + e * N3 : nullptr;
    l0v = a.lam0_value;
    l1v = a.lam1_value;
  }
  static constexpr bool kIn = true, kOut = HELM;  // x scaled by w before h (node order), then lam0
  template <int K>
  __device__ __forceinline__ void factors(int n, double gg[6], double& sin, double& sout, double& mass) const {
    const double w = (cW<N1>(K) * wj) * wi;
#pragma unroll
    for (int q = 0; q < 6; ++q) gg[q] = h[q];
    sin = w;
    sout = 1.0;
    mass = 0.0;
    if (HELM) {
      sout = lam0 ? __ldg(lam0 + n) : l0v;
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * (w * h[6]);
    }
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
      // __dmul_rn: ptxas must not fuse tt * l0 into the next even-odd add (it can
      // where tt stays in registers, not where it is parked in shared memory)
      const double l0 = lam0 ? __ldg(lam0 + n) : l0v;
      rr = __dmul_rn(rr, l0);
      ss = __dmul_rn(ss, l0);
      tt = __dmul_rn(tt, l0);
      mass = (lam1 ? __ldg(lam1 + n) : l1v) * (w * h[6]);
    }
  }
};

template <typename F, int K>
__device__ __forceinline__ void node_at(const F& fac, int n, double x0, double x1, double x2, double& rr,
                                        double& ss, double& tt, double& mass) {
#if defined(HX_ABLATE) && HX_ABLATE == 1
  // timing experiment only (tools/build_variant.sh abl1 "-DHX_ABLATE=1" ax_fast; wrong
  // results): the skeleton without per-node geometry, profiles/r01_ablation_n7.txt
  rr = x0 * 1.0000001;
  ss = x1 * 1.0000001;
  tt = x2 * 1.0000001;
  mass = 0.0;
#else
  fac.template node<K>(n, x0, x1, x2, rr, ss, tt, mass);
#endif
}

// Shared memory lives at file scope so that the per-element body can be a
// separate (non-inlined) function: inlined into the persistent loop, NVVM
// hoists every __constant__ operand out of the loop into registers and spills.
// TMA landing zones for x (linear, as in HBM), one per column count
static __shared__ __align__(128) double s_land1[2][N3];
static __shared__ __align__(128) double s_land3[2][N3 * 3];
static __shared__ __align__(128) double s_land1_one[N3];
static __shared__ __align__(128) double s_land3_one[N3 * 3];
template <int NCOL>
__device__ __forceinline__ double* landing_one() {
  if constexpr (NCOL == 1)
    return s_land1_one;
  else
    return s_land3_one;
}
template <int NCOL>
__device__ __forceinline__ double* landing(int b) {
  if constexpr (NCOL == 1)
    return s_land1[b];
  else
    return s_land3[b];
}
static __shared__ __align__(16) double s_verts[2][24];  // TMA landing zone for the vertices
static __shared__ double s_cubeX[CUBE];
static __shared__ double s_cubeA[CUBE];
static __shared__ double s_cubeB[CUBE];
static __shared__ TriShared s_tri;
static __shared__ __align__(8) uint64_t s_mbar[2];

template <typename F, int NCOL, bool HELM, bool TRI>
__device__ __noinline__ void element(const hx_axlocal_args* __restrict__ ap, int64_t e, int b) {
  const hx_axlocal_args& a = *ap;
  double* sX = s_cubeX;
  double* sA = s_cubeA;
  double* sB = s_cubeB;
  const int t = threadIdx.x;
  const Roles r = roles(t);
  const int kp = Aj(r.fj) + r.fi;      // k-fibre base (+ Ak(k))
  const int rb = Ak(r.rk) + Aj(r.rj);  // i-row base (+ n)
  const int cb = Ak(r.ck) + r.ci;      // j-column base (+ Aj(n))
  const int lin = r.fj * 8 + r.fi;     // k-fibre offset in the linear element (+ 64 k)
  const double* sL = landing<NCOL>(b);

#pragma unroll 1
  for (int c = 0; c < NCOL; ++c) {
    double xk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) xk[k] = sL[(k * 64 + lin) * NCOL + c];
#pragma unroll
    for (int k = 0; k < 8; ++k) sX[Ak(k) + kp] = xk[k];
    if (TRI && F::kStageA && c == 0) tri_stage_a(t, s_verts[b], s_tri);
    __syncthreads();

    F fac;
    fac.prepare(a, e, s_tri, s_verts[b], r.fi, r.fj);

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
    if constexpr (F::kScaleFirst) {
      // all eight reciprocals first: eight independent chains for the scheduler
      double sc[8], ms[8];
#define HX_SCALE(K) fac.template scale_at<K>(K * 64 + lin, sc[K], ms[K]);
      HX_SCALE(0) HX_SCALE(1) HX_SCALE(2) HX_SCALE(3) HX_SCALE(4) HX_SCALE(5) HX_SCALE(6) HX_SCALE(7)
#undef HX_SCALE
#define HX_NODE(K)                                                          \
  {                                                                         \
    const int adr = Ak(K) + kp;                                             \
    double rr, ss;                                                          \
    fac.template apply_at<K>(sc[K], sA[adr], sB[adr], x2[K], rr, ss, tt[K]); \
    sA[adr] = rr;                                                           \
    sB[adr] = ss;                                                           \
    if (HELM) yk[K] = __dmul_rn(ms[K], xk[K]);                              \
  }
      HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
    } else {
#define HX_NODE(K)                                                                  \
  {                                                                                 \
    const int adr = Ak(K) + kp;                                                     \
    double rr, ss, mass;                                                            \
    node_at<F, K>(fac, K * 64 + lin, sA[adr], sB[adr], x2[K], rr, ss, tt[K], mass); \
    sA[adr] = rr;                                                                   \
    sB[adr] = ss;                                                                   \
    if (HELM) yk[K] = __dmul_rn(mass, xk[K]);                                       \
  }
      HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
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

    double* yout = a.y + e * N3 * NCOL;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int adr = Ak(k) + kp;
      double y = (sA[adr] + sB[adr]) + yt[k];
      if (HELM) y = __dadd_rn(y, yk[k]);  // pinned rounding: n_col=3 == 3 x n_col=1 bitwise
      yout[(k * 64 + lin) * NCOL + c] = y;
    }
  }
}

// COPY selects the copy of the D blocks (so two bodies in one kernel do not
// share constants); XLAND reads x from the single-element TMA landing buffer.
template <typename F, int NCOL, bool HELM, bool TRI, int COPY = 0, bool XLAND = false, bool VGLOBAL = false,
          bool CGP = false>
__device__ __forceinline__ void element_direct(const hx_axlocal_args* __restrict__ ap, int64_t e, int b = 0) {
  const hx_axlocal_args& a = *ap;
  double* sX = s_cubeX;
  double* sA = s_cubeA;
  double* sB = s_cubeB;
  const int t = threadIdx.x;
  const Roles r = roles(t);
  const int kp = Aj(r.fj) + r.fi;      // k-fibre base (+ Ak(k))
  const int rb = Ak(r.rk) + Aj(r.rj);  // i-row base (+ n)
  const int cb = Ak(r.ck) + r.ci;      // j-column base (+ Aj(n))
  const int lin = r.fj * 8 + r.fi;     // k-fibre offset in the linear element (+ 64 k)
  // VGLOBAL: stage A reads the 24 vertex coordinates straight from global memory (L1),
  // so the CTA needs no vertex staging barrier
  const double* vsrc = VGLOBAL ? a.verts + e * 24 : s_verts[b];

  // element-local x, or (fused BP5 gather) the slab lattice: node (i,j,k) of
  // element (cx,cy,cz) is lattice point (cx N + i, cy N + j, cz N + k)
  int64_t xoff = (e * N3 + lin) * NCOL, xstr = 64 * NCOL;
  if (!XLAND && a.gather) {
    const hx_box& bx = a.gather_box;
    const int64_t nx = (int64_t)bx.ex * 7 + 1, ny = (int64_t)bx.ey * 7 + 1;
    const unsigned e32 = (unsigned)e, exu = (unsigned)bx.ex, exy = exu * (unsigned)bx.ey;  // 32-bit division
    const unsigned cz = e32 / exy, rem = e32 - cz * exy, cy = rem / exu, cx = rem - cy * exu;
    xoff = ((int64_t)(cz * 7) * ny + cy * 7 + r.fj) * nx + cx * 7 + r.fi;
    xstr = nx * ny;
  }
#pragma unroll 1
  for (int c = 0; c < NCOL; ++c) {
    double xk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      xk[k] = XLAND ? landing_one<NCOL>()[(k * 64 + lin) * NCOL + c] : __ldg(a.x + xoff + k * xstr + c);
    if constexpr (CGP) {
      // fused CG direction update on the lattice: p = r + beta p_old (solver.py:170, the
      // rounding of cg_p_kernel); every element writes its nodes (shared nodes get the
      // same value from each of their elements)
      const double beta = a.cg_scal[2] / a.cg_scal[0];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t g = xoff + k * xstr;
        xk[k] = __dadd_rn(__ldg(a.cg_r + g), __dmul_rn(beta, xk[k]));
        a.cg_p_out[g] = xk[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) sX[Ak(k) + kp] = xk[k];
    if (TRI && F::kStageA && c == 0) tri_stage_a(t, vsrc, s_tri);
    __syncthreads();

    F fac;
    fac.prepare(a, e, s_tri, vsrc, r.fi, r.fj);

    // forward: x2 on the k-fibre; x0 on the i-row; x1 on the j-column
    double x2[8];
    eo8<0, COPY>(xk, x2);
    {
      double v[8], o[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sX[rb + n];
      eo8<0, COPY>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sA[rb + n] = o[n];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sX[cb + Aj(n)];
      eo8<0, COPY>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sB[cb + Aj(n)] = o[n];
    }
    __syncthreads();

    // nodewise factor stage on the k-fibre, in place (each address owned by one thread)
    double tt[8], yk[8];
    if constexpr (F::kScaleFirst) {
      // all eight reciprocals first: eight independent chains for the scheduler
      double sc[8], ms[8];
#define HX_SCALE(K) fac.template scale_at<K>(K * 64 + lin, sc[K], ms[K]);
      HX_SCALE(0) HX_SCALE(1) HX_SCALE(2) HX_SCALE(3) HX_SCALE(4) HX_SCALE(5) HX_SCALE(6) HX_SCALE(7)
#undef HX_SCALE
#define HX_NODE(K)                                                          \
  {                                                                         \
    const int adr = Ak(K) + kp;                                             \
    double rr, ss;                                                          \
    fac.template apply_at<K>(sc[K], sA[adr], sB[adr], x2[K], rr, ss, tt[K]); \
    sA[adr] = rr;                                                           \
    sB[adr] = ss;                                                           \
    if (HELM) yk[K] = __dmul_rn(ms[K], xk[K]);                              \
  }
      HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
    } else if constexpr (F::kTtSmem && !HELM) {
      // park each tt in the (consumed) x cube instead of holding 8 registers
#define HX_NODE(K)                                                                   \
  {                                                                                  \
    const int adr = Ak(K) + kp;                                                      \
    double rr, ss, t_, mass;                                                         \
    node_at<F, K>(fac, K * 64 + lin, sA[adr], sB[adr], x2[K], rr, ss, t_, mass);     \
    sA[adr] = rr;                                                                    \
    sB[adr] = ss;                                                                    \
    sX[adr] = t_;                                                                    \
  }
      HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
#pragma unroll
      for (int k = 0; k < 8; ++k) tt[k] = sX[Ak(k) + kp];
    } else {
#define HX_NODE(K)                                                                  \
  {                                                                                 \
    const int adr = Ak(K) + kp;                                                     \
    double rr, ss, mass;                                                            \
    node_at<F, K>(fac, K * 64 + lin, sA[adr], sB[adr], x2[K], rr, ss, tt[K], mass); \
    sA[adr] = rr;                                                                   \
    sB[adr] = ss;                                                                   \
    if (HELM) yk[K] = __dmul_rn(mass, xk[K]);                                       \
  }
      HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
    }
    double yt[8];
    eo8<1, COPY>(tt, yt);
    __syncthreads();

    // transposed: D^T rr on the i-row, D^T ss on the j-column, in place
    {
      double v[8], o[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sA[rb + n];
      eo8<1, COPY>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sA[rb + n] = o[n];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = sB[cb + Aj(n)];
      eo8<1, COPY>(v, o);
#pragma unroll
      for (int n = 0; n < 8; ++n) sB[cb + Aj(n)] = o[n];
    }
    __syncthreads();

    double* yout = a.y + e * N3 * NCOL;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int adr = Ak(k) + kp;
      double y = (sA[adr] + sB[adr]) + yt[k];
      if (HELM) y = __dadd_rn(y, yk[k]);  // pinned rounding: n_col=3 == 3 x n_col=1 bitwise
      yout[(k * 64 + lin) * NCOL + c] = y;
    }
  }
}


// One CTA per element (no persistent loop): the body inlines into the kernel
// and D's even-odd blocks stay __constant__ operands.
template <typename F, int NCOL, bool HELM, bool TRI, int MINB, bool VG = false, bool CGP = false>
__global__ void __launch_bounds__(64, MINB) ax8s(const __grid_constant__ hx_axlocal_args a) {
  const int64_t e = blockIdx.x;
  // CTAs start in blockIdx order, ~148 x 8 resident at a time: warm L2 for the
  // element two waves ahead so its CTA's loads do not wait on HBM latency.
  if (a.reserved != 3) {
    // 1.25 waves of resident CTAs ahead (the stored kernel streams 28 KB per element and
    // prefers the shorter distance: 109 vs 105 GDOF/s at 2 waves; trilinear is insensitive)
    const int64_t ahead = e + (a.reserved == 8 ? kPrefetchAhead : 148 * MINB * 5 / 4);
    if (ahead < a.n_elements) {
      if (a.gather) {
        // fused BP5 gather: x is the slab lattice; warm the 64 lattice rows (64 B each)
        // of the element two waves ahead, one row per thread
        const hx_box& bx = a.gather_box;
        const int64_t nx = (int64_t)bx.ex * 7 + 1, ny = (int64_t)bx.ey * 7 + 1;
        const unsigned e32 = (unsigned)ahead, exu = (unsigned)bx.ex, exy = exu * (unsigned)bx.ey;
        const unsigned cz = e32 / exy, rem = e32 - cz * exy, cy = rem / exu, cx = rem - cy * exu;
        const int j = threadIdx.x & 7, k = threadIdx.x >> 3;
        const int64_t off = ((int64_t)(cz * 7 + k) * ny + cy * 7 + j) * nx + cx * 7;
        prefetch_l2(a.x + off);
        prefetch_l2(a.x + off + 7);
        if (CGP) {
          prefetch_l2(a.cg_r + off);
          prefetch_l2(a.cg_r + off + 7);
        }
      } else if (threadIdx.x == 0) {
        bulk_prefetch_l2(a.x + ahead * N3 * NCOL, 4096u * NCOL);
      }
      if (TRI && threadIdx.x == 0) bulk_prefetch_l2(a.verts + ahead * 24, 192u);
      // per-node scalar fields of the partial / merged / Helmholtz variants
      if (threadIdx.x == 1) {
        if (a.lam_geo) bulk_prefetch_l2(a.lam_geo + ahead * N3, 4096u);
        if (a.lam2) bulk_prefetch_l2(a.lam2 + ahead * N3, 4096u);
        if (a.lam3) bulk_prefetch_l2(a.lam3 + ahead * N3, 4096u);
        if (a.lam0) bulk_prefetch_l2(a.lam0 + ahead * N3, 4096u);
        if (a.lam1) bulk_prefetch_l2(a.lam1 + ahead * N3, 4096u);
      }
    }
  }
  if (!VG) {
    if (TRI && threadIdx.x < 24) s_verts[0][threadIdx.x] = __ldg(a.verts + e * 24 + threadIdx.x);
    if (TRI) __syncthreads();
  }
  element_direct<F, NCOL, HELM, TRI, 0, false, VG, CGP>(&a, e);
}

// Two elements per CTA in straight-line code: the second element's x and
// vertices arrive by TMA bulk copy while the first is computed, so half of the
// CTA-start load latency disappears without a loop (a loop lets NVVM hoist the
// D-block constants into registers; see element()).
template <typename F, int NCOL, bool HELM, bool TRI, int MINB>
__global__ void __launch_bounds__(64, MINB) ax8d(const __grid_constant__ hx_axlocal_args a) {
  const int64_t e0 = 2 * (int64_t)blockIdx.x, e1 = e0 + 1;
  const bool has1 = e1 < a.n_elements;
  const int t = threadIdx.x;
  if (t == 0) {
    mbar_init(&s_mbar[1], 1);
    fence_mbar_init();
  }
  if (TRI && t < 24) s_verts[0][t] = __ldg(a.verts + e0 * 24 + t);
  __syncthreads();
  if (t == 0 && has1) {
    mbar_arrive_expect_tx(&s_mbar[1], 4096u * NCOL + (TRI ? 192u : 0u));
    bulk_g2s(landing_one<NCOL>(), a.x + e1 * N3 * NCOL, 4096u * NCOL, &s_mbar[1]);
    if (TRI) bulk_g2s(s_verts[1], a.verts + e1 * 24, 192u, &s_mbar[1]);
  }
  element_direct<F, NCOL, HELM, TRI, 0, false>(&a, e0, 0);
  if (has1) {
    mbar_wait(&s_mbar[1], 0);
    element_direct<F, NCOL, HELM, TRI, 1, true>(&a, e1, 1);
  }
}

template <typename F, bool HELM, bool TRI, int MINB>
cudaError_t launch_double(const hx_axlocal_args& a, cudaStream_t s) {
  const int64_t blocks = (a.n_elements + 1) / 2;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  if (a.n_col == 3)
    ax8d<F, 3, HELM, TRI, MINB><<<(unsigned)blocks, 64, 0, s>>>(a);
  else
    ax8d<F, 1, HELM, TRI, MINB><<<(unsigned)blocks, 64, 0, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// n_col = 3 with factor reuse (the paper's loop swap, §4.1): all three columns
// go through every phase together, each node's factors are computed once and
// applied to the three columns with exactly the per-column arithmetic of the
// n_col = 1 kernel (so n_col=3 == 3 x n_col=1 bitwise, test_axlocal.py:206-225).
static __shared__ double s_c3X[3][CUBE];
static __shared__ double s_c3A[3][CUBE];
static __shared__ double s_c3B[3][CUBE];

// n_col = 3: keep tt / yt in registers (parallelepiped: +6-12 %; merged at 4 CTAs / SM:
// +6 %) or park them in the x cube (the other sources: registers would spill, -5-13 %;
// A/B in profiles/r01_n7_variants_c4.txt)
template <typename F>
struct C3RegTt {
#ifdef HX_C3_REGTT_ALL  // A/B builds
  static constexpr bool value = true;
#else
  static constexpr bool value = false;
#endif
};
template <bool HELM>
struct C3RegTt<Ppd<HELM>> {
  static constexpr bool value = true;
};
template <>  // merged, with 4 CTAs / SM (255 registers): +6 % (launch_c3 below)
struct C3RegTt<TrilinearPoly<true, true, false, true, false, false, true>> {
  static constexpr bool value = true;
};

template <typename F>
__device__ __forceinline__ void apply_factors(const double g[6], double sin, double sout, double x0, double x1,
                                              double x2, double& rr, double& ss, double& tt) {
  double s0 = x0, s1 = x1, s2 = x2;
  if (F::kIn) {
    s0 = sin * x0;
    s1 = sin * x1;
    s2 = sin * x2;
  }
  rr = fma(g[0], s0, fma(g[1], s1, g[2] * s2));
  ss = fma(g[1], s0, fma(g[3], s1, g[4] * s2));
  tt = fma(g[2], s0, fma(g[4], s1, g[5] * s2));
  if (F::kOut) {
    rr = __dmul_rn(rr, sout);
    ss = __dmul_rn(ss, sout);
    tt = __dmul_rn(tt, sout);
  }
}

template <typename F, bool HELM, bool TRI, int MINB, bool VG = false>
__global__ void __launch_bounds__(64, MINB) ax8c3(const __grid_constant__ hx_axlocal_args a) {
  constexpr int NC = 3;
  const int64_t e = blockIdx.x;
  const int t = threadIdx.x;
  const Roles r = roles(t);
  const int kp = Aj(r.fj) + r.fi;
  const int rb = Ak(r.rk) + Aj(r.rj);
  const int cb = Ak(r.ck) + r.ci;
  const int lin = r.fj * 8 + r.fi;
  // warm L2 with the element two waves ahead (as ax8s): its three columns of x, its
  // vertices and any per-node scalar fields
  if (a.reserved != 7 && t < 2) {
    const int64_t ahead = e + 2 * 148 * MINB;
    if (ahead < a.n_elements) {
      if (t == 0) {
        bulk_prefetch_l2(a.x + ahead * N3 * NC, 4096u * NC);
        if (TRI) bulk_prefetch_l2(a.verts + ahead * 24, 192u);
      } else {
        if (a.lam_geo) bulk_prefetch_l2(a.lam_geo + ahead * N3, 4096u);
        if (a.lam2) bulk_prefetch_l2(a.lam2 + ahead * N3, 4096u);
        if (a.lam3) bulk_prefetch_l2(a.lam3 + ahead * N3, 4096u);
        if (a.lam0) bulk_prefetch_l2(a.lam0 + ahead * N3, 4096u);
        if (a.lam1) bulk_prefetch_l2(a.lam1 + ahead * N3, 4096u);
      }
    }
  }
  // P0: the three columns of the k-fibre (loads issued before the vertex staging
  // barrier); x2 = D_t x in registers
  double x2[NC][8];
#ifndef HX_C3_XLATE
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) x2[c][k] = __ldg(a.x + (e * N3 + k * 64 + lin) * NC + c);
#endif
  // VG: stage A reads the vertices from L1 (no staging barrier)
  const double* vsrc = VG ? a.verts + e * 24 : s_verts[0];
  if (!VG) {
    if (TRI && t < 24) s_verts[0][t] = __ldg(a.verts + e * 24 + t);
    if (TRI) __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double xk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#ifndef HX_C3_XLATE
      xk[k] = x2[c][k];
#else
      xk[k] = __ldg(a.x + (e * N3 + k * 64 + lin) * NC + c);
#endif
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s_c3X[c][Ak(k) + kp] = xk[k];
    eo8<0>(xk, x2[c]);
  }
  if (TRI && F::kStageA) tri_stage_a(t, vsrc, s_tri);
  __syncthreads();

  // P1: forward r (i-rows) and s (j-columns) derivatives of the three columns
  F fac;
  fac.prepare(a, e, s_tri, vsrc, r.fi, r.fj);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double v[8], o[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) v[n] = s_c3X[c][rb + n];
    eo8<0>(v, o);
#pragma unroll
    for (int n = 0; n < 8; ++n) s_c3A[c][rb + n] = o[n];
#pragma unroll
    for (int n = 0; n < 8; ++n) v[n] = s_c3X[c][cb + Aj(n)];
    eo8<0>(v, o);
#pragma unroll
    for (int n = 0; n < 8; ++n) s_c3B[c][cb + Aj(n)] = o[n];
  }
  __syncthreads();

  // P2: factors once per node, applied to the three columns
#define HX_NODE3(K, TT)                                                                   \
  {                                                                                       \
    const int adr = Ak(K) + kp;                                                           \
    double g[6], sin, sout;                                                               \
    fac.template factors<K>(K * 64 + lin, g, sin, sout, mass[K]);                         \
    _Pragma("unroll") for (int c = 0; c < NC; ++c) {                                      \
      double rr, ss, tt;                                                                  \
      apply_factors<F>(g, sin, sout, s_c3A[c][adr], s_c3B[c][adr], x2[c][K], rr, ss, tt); \
      s_c3A[c][adr] = rr;                                                                 \
      s_c3B[c][adr] = ss;                                                                 \
      TT = tt;                                                                            \
    }                                                                                     \
  }
  double mass[8], yt[NC][8];
  if constexpr (C3RegTt<F>::value) {
    // tt in registers (x2[c][K] dies as tt[c][K] is born), then D_t^T tt with the
    // n_col = 1 kernel's even-odd arithmetic (n_col=3 == 3 x n_col=1 bitwise): saves
    // the 4 shared accesses per node and column of parking tt / yt in the x cube
    double tt3[NC][8];
    HX_NODE3(0, tt3[c][0]) HX_NODE3(1, tt3[c][1]) HX_NODE3(2, tt3[c][2]) HX_NODE3(3, tt3[c][3])
    HX_NODE3(4, tt3[c][4]) HX_NODE3(5, tt3[c][5]) HX_NODE3(6, tt3[c][6]) HX_NODE3(7, tt3[c][7])
#pragma unroll
    for (int c = 0; c < NC; ++c) eo8<1>(tt3[c], yt[c]);
  } else {
    // tt parked in the (consumed) x cube at this thread's own fibre positions
    HX_NODE3(0, s_c3X[c][adr]) HX_NODE3(1, s_c3X[c][adr]) HX_NODE3(2, s_c3X[c][adr]) HX_NODE3(3, s_c3X[c][adr])
    HX_NODE3(4, s_c3X[c][adr]) HX_NODE3(5, s_c3X[c][adr]) HX_NODE3(6, s_c3X[c][adr]) HX_NODE3(7, s_c3X[c][adr])
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double tt[8], yc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) tt[k] = s_c3X[c][Ak(k) + kp];
      eo8<1>(tt, yc);
#pragma unroll
      for (int k = 0; k < 8; ++k) s_c3X[c][Ak(k) + kp] = yc[k];
    }
  }
#undef HX_NODE3
  __syncthreads();

  // P3: transposed r and s contractions, in place
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double v[8], o[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) v[n] = s_c3A[c][rb + n];
    eo8<1>(v, o);
#pragma unroll
    for (int n = 0; n < 8; ++n) s_c3A[c][rb + n] = o[n];
#pragma unroll
    for (int n = 0; n < 8; ++n) v[n] = s_c3B[c][cb + Aj(n)];
    eo8<1>(v, o);
#pragma unroll
    for (int n = 0; n < 8; ++n) s_c3B[c][cb + Aj(n)] = o[n];
  }
  __syncthreads();

  // P4: y = D_r^T rr + D_s^T ss + D_t^T tt [+ mass x] (n_col = 1 order)
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int adr = Ak(k) + kp;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double y = (s_c3A[c][adr] + s_c3B[c][adr]) + (C3RegTt<F>::value ? yt[c][k] : s_c3X[c][adr]);
      if (HELM) y = __dadd_rn(y, __dmul_rn(mass[k], __ldg(a.x + (e * N3 + k * 64 + lin) * NC + c)));
      a.y[(e * N3 + k * 64 + lin) * NC + c] = y;
    }
  }
}

#ifndef HX_C3_MINB
#define HX_C3_MINB 5
#endif
template <typename F, bool HELM, bool TRI, int MINB = HX_C3_MINB>
cudaError_t launch_c3(const hx_axlocal_args& a, cudaStream_t s) {
  if (a.n_elements > 0x7fffffffLL) return cudaErrorInvalidValue;
  if (TRI && a.reserved == 6)  // vertices from L1: 7 % slower here (profiles/r01_sweep_variants.txt)
    ax8c3<F, HELM, TRI, MINB, true><<<(unsigned)a.n_elements, 64, 0, s>>>(a);
  else
    ax8c3<F, HELM, TRI, MINB><<<(unsigned)a.n_elements, 64, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename F, int NCOL, bool HELM, bool TRI, int MINB>
__global__ void __launch_bounds__(64, MINB) ax8(const __grid_constant__ hx_axlocal_args a) {
  const int t = threadIdx.x;
  const int64_t E = a.n_elements;
  constexpr uint32_t kBytes = 4096u * NCOL + (TRI ? 192u : 0u);

  if (t == 0) {
    mbar_init(&s_mbar[0], 1);
    mbar_init(&s_mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t e = blockIdx.x;
  if (t == 0 && e < E) {
    mbar_arrive_expect_tx(&s_mbar[0], kBytes);
    bulk_g2s(landing<NCOL>(0), a.x + e * N3 * NCOL, 4096u * NCOL, &s_mbar[0]);
    if (TRI) bulk_g2s(s_verts[0], a.verts + e * 24, 192u, &s_mbar[0]);
  }
  for (int it = 0; e < E; e += gridDim.x, ++it) {
    const int b = it & 1;
    const int64_t en = e + gridDim.x;
    if (t == 0 && en < E) {
      // buffer b^1 was last read before the barriers of this CTA's previous element
      fence_proxy_async();
      mbar_arrive_expect_tx(&s_mbar[b ^ 1], kBytes);
      bulk_g2s(landing<NCOL>(b ^ 1), a.x + en * N3 * NCOL, 4096u * NCOL, &s_mbar[b ^ 1]);
      if (TRI) bulk_g2s(s_verts[b ^ 1], a.verts + en * 24, 192u, &s_mbar[b ^ 1]);
    }
    mbar_wait(&s_mbar[b], (it >> 1) & 1);
    element<F, NCOL, HELM, TRI>(&a, e, b);
  }
}

// One element per WARP (32-thread CTA): each lane plays two fibre roles
// (t = lane and t = 32 + lane of the 64-role maps above), phases are separated
// by __syncwarp only, and no register state crosses a phase: x2 is recomputed
// from the x fibre in the node phase and the t-transpose result is parked in
// place of x in the X cube.  The node phase of one role is an out-of-line
// function so that the two roles cannot share (and keep live) constants.
template <typename F, bool HELM, int COPY>
__device__ __noinline__ void warp_node_phase(const hx_axlocal_args* __restrict__ ap, int64_t e, int role) {
  const hx_axlocal_args& a = *ap;
  double* sX = s_cubeX;
  double* sA = s_cubeA;
  double* sB = s_cubeB;
  const Roles r = roles(role);
  const int kp = Aj(r.fj) + r.fi, lin = r.fj * 8 + r.fi;
  F fac;
  fac.prepare(a, e, s_tri, s_verts[0], r.fi, r.fj);
  double xk[8], x2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) xk[k] = sX[Ak(k) + kp];
  eo8<0, COPY>(xk, x2);
  double tt[8], yk[8];
#define HX_NODE(K)                                                                  \
  {                                                                                 \
    const int adr = Ak(K) + kp;                                                     \
    double rr, ss, mass;                                                            \
    node_at<F, K>(fac, K * 64 + lin, sA[adr], sB[adr], x2[K], rr, ss, tt[K], mass); \
    sA[adr] = rr;                                                                   \
    sB[adr] = ss;                                                                   \
    if (HELM) yk[K] = __dmul_rn(mass, xk[K]);                                       \
  }
  HX_NODE(0) HX_NODE(1) HX_NODE(2) HX_NODE(3) HX_NODE(4) HX_NODE(5) HX_NODE(6) HX_NODE(7)
#undef HX_NODE
  double yt[8];
  eo8<1, COPY>(tt, yt);
#pragma unroll
  for (int k = 0; k < 8; ++k) sX[Ak(k) + kp] = HELM ? yt[k] + yk[k] : yt[k];
}

template <int T, int COPY>
__device__ __forceinline__ void warp_rowcol(int role, double* sR, double* sC, const double* srcR,
                                            const double* srcC) {
  const Roles r = roles(role);
  const int rb = Ak(r.rk) + Aj(r.rj), cb = Ak(r.ck) + r.ci;
  double v[8], o[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) v[n] = srcR[rb + n];
  eo8<T, COPY>(v, o);
#pragma unroll
  for (int n = 0; n < 8; ++n) sR[rb + n] = o[n];
#pragma unroll
  for (int n = 0; n < 8; ++n) v[n] = srcC[cb + Aj(n)];
  eo8<T, COPY>(v, o);
#pragma unroll
  for (int n = 0; n < 8; ++n) sC[cb + Aj(n)] = o[n];
}

template <typename F, int NCOL, bool HELM, bool TRI, int MINB>
__global__ void __launch_bounds__(32, MINB) ax8w(const __grid_constant__ hx_axlocal_args a) {
  double* sX = s_cubeX;
  double* sA = s_cubeA;
  double* sB = s_cubeB;
  const int lane = threadIdx.x;
  const int64_t e = blockIdx.x;
  if (TRI && lane < 24) s_verts[0][lane] = __ldg(a.verts + e * 24 + lane);
  if (TRI) __syncwarp();

#pragma unroll 1
  for (int c = 0; c < NCOL; ++c) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const Roles r = roles(32 * p + lane);
      const int kp = Aj(r.fj) + r.fi, lin = r.fj * 8 + r.fi;
      double xk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) xk[k] = __ldg(a.x + (e * N3 + k * 64 + lin) * NCOL + c);
#pragma unroll
      for (int k = 0; k < 8; ++k) sX[Ak(k) + kp] = xk[k];
    }
    if (TRI && F::kStageA && c == 0) {
      tri_stage_a(lane, s_verts[0], s_tri);
      tri_stage_a(lane + 32, s_verts[0], s_tri);
    }
    __syncwarp();
    warp_rowcol<0, 0>(lane, sA, sB, sX, sX);
    warp_rowcol<0, 1>(32 + lane, sA, sB, sX, sX);
    __syncwarp();
    warp_node_phase<F, HELM, 0>(&a, e, lane);
    warp_node_phase<F, HELM, 1>(&a, e, 32 + lane);
    __syncwarp();
    warp_rowcol<1, 0>(lane, sA, sB, sA, sB);
    warp_rowcol<1, 1>(32 + lane, sA, sB, sA, sB);
    __syncwarp();
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const Roles r = roles(32 * p + lane);
      const int kp = Aj(r.fj) + r.fi, lin = r.fj * 8 + r.fi;
      double* yout = a.y + e * N3 * NCOL;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int adr = Ak(k) + kp;
        yout[(k * 64 + lin) * NCOL + c] = (sA[adr] + sB[adr]) + sX[adr];
      }
    }
    __syncwarp();
  }
}

template <typename F, bool HELM, bool TRI, int MINB>
cudaError_t launch_warp(const hx_axlocal_args& a, cudaStream_t s) {
  if (a.n_elements > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)a.n_elements;
  if (a.n_col == 3)
    ax8w<F, 3, HELM, TRI, MINB><<<grid, 32, 0, s>>>(a);
  else
    ax8w<F, 1, HELM, TRI, MINB><<<grid, 32, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename F, int NCOL, bool HELM, bool TRI, int MINB>
cudaError_t launch_n(const hx_axlocal_args& a, cudaStream_t s) {
  static int grid_cap = 0;  // persistent grid: SMs x resident CTAs (per instantiation)
  if (grid_cap == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess)
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ax8<F, NCOL, HELM, TRI, MINB>, 64, 0);
    if (err != cudaSuccess) return err;
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t grid = a.n_elements < grid_cap ? a.n_elements : grid_cap;
  ax8<F, NCOL, HELM, TRI, MINB><<<(unsigned)grid, 64, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename F, bool HELM, bool TRI, int MINB, bool VG = false>
cudaError_t launch_single(const hx_axlocal_args& a, cudaStream_t s) {
  if (a.n_elements > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)a.n_elements;
  if (a.cg_r) {  // fused CG direction update (gather mode, n_col = 1; checked by the caller)
    ax8s<F, 1, HELM, TRI, MINB, VG, true><<<grid, 64, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (a.n_col == 3)
    ax8s<F, 3, HELM, TRI, MINB, VG><<<grid, 64, 0, s>>>(a);
  else
    ax8s<F, 1, HELM, TRI, MINB, VG><<<grid, 64, 0, s>>>(a);
  return cudaGetLastError();
}

// MINB = resident 64-thread CTAs per SM the register budget is sized for
// (8 -> <= 128 registers, 6 -> <= 168).
template <typename F, bool HELM, bool TRI, int MINB = 8>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  if (a.n_col == 3) return launch_n<F, 3, HELM, TRI, MINB>(a, s);
  return launch_n<F, 1, HELM, TRI, MINB>(a, s);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace fast
}  // namespace hx

// Kernel choice per variant (measured on B200, tools/sweep.py, profiles/):
//  * trilinear family (FP64-bound): one CTA per element (ax8s), shared
//    per-element setup incl. the K00(j,k)/K11(i,k) tables, 10 CTAs/SM
//    (96 registers, no spills);
//  * stored / parallelepiped (HBM-bound): also one CTA per element — with
//    8 CTAs/SM the plain coalesced loads reach 7.0 TB/s, ahead of the
//    persistent TMA-prefetch pipeline (ax8, hook 1: 6.6 TB/s).
// `reserved` is a tuning hook used by tools/sweep.py to time the alternatives.
extern "C" cudaError_t hx_fast_launch(const hx_axlocal_args* a, cudaStream_t s) {
  using namespace hx::fast;
  if (a->order != 7) return cudaErrorNotSupported;
  // the bulk copies need 16-byte aligned sources
  if (!aligned16(a->x) || (a->verts && !aligned16(a->verts))) return cudaErrorNotSupported;
  const bool helm = a->equation == HX_HELMHOLTZ;
  const int hook = a->gather ? 0 : a->reserved;  // fused gather lives in the single-shot kernels
  if (a->n_col == 3 && hook != 4) {
    switch (a->factor_source) {
      case HX_TRILINEAR:
        return helm ? launch_c3<TrilinearPoly<true, false, false, true, false, false, true>, true, true>(*a, s)
                    : launch_c3<TrilinearPoly<false, false, false, true, false, false, true>, false, true>(*a, s);
      case HX_TRILINEAR_PARTIAL:
        return launch_c3<TrilinearPoly<false, false, true, true, false, false, true>, false, true>(*a, s);
      case HX_TRILINEAR_MERGED:
        return launch_c3<TrilinearPoly<true, true, false, true, false, false, true>, true, true, 4>(*a, s);
      case HX_STORED:
        return helm ? launch_c3<StoredLoad<true>, true, false>(*a, s) : launch_c3<StoredLoad<false>, false, false>(*a, s);
      case HX_PARALLELEPIPED:
        return helm ? launch_c3<Ppd<true>, true, false>(*a, s) : launch_c3<Ppd<false>, false, false>(*a, s);
    }
    return cudaErrorNotSupported;
  }
  switch (a->factor_source) {
    case HX_TRILINEAR:
      if (helm) {
        if (hook == 1) return launch<TrilinearPoly<true, false, false>, true, true>(*a, s);
        if (hook == 2) return launch_single<TrilinearPoly<true, false, false, true, false, false, true>, true, true, 10>(*a, s);
        if (hook == 3) return launch_single<TrilinearPoly<true, false, false>, true, true, 8, true>(*a, s);
        // default: K00/K11 tables, vertices from L1, 8 CTAs/SM (10 would spill): +1.4 % over no tables
        return launch_single<TrilinearPoly<true, false, false, true, false, false, true>, true, true, 8, true>(*a, s);
      }
      switch (hook) {
        case 1: return launch<TrilinearPoly<false, false, false>, false, true>(*a, s);
        case 2: return launch_single<TrilinearPoly<false, false, false, true>, false, true, 8>(*a, s);
        case 6: return launch<TrilinearPoly<false, false, false>, false, true, 6>(*a, s);
        case 9: return launch<TrilinearPoly<false, false, false, false>, false, true, 6>(*a, s);
        case 10: return launch_single<TrilinearPoly<false, false, false, true>, false, true, 6>(*a, s);
        case 11: return launch_single<TrilinearPoly<false, false, false, false>, false, true, 6>(*a, s);
        case 13: return launch_single<TrilinearPoly<false, false, false, false>, false, true, 8>(*a, s);
        case 14: return launch_single<TrilinearPoly<false, false, false, true, true>, false, true, 8>(*a, s);
        case 16: return launch_single<TrilinearPoly<false, false, false, true, false, true>, false, true, 8>(*a, s);
        case 19: return launch_single<TrilinearPoly<false, false, false, true, false, false>, false, true, 10>(*a, s);
        case 20: return launch_warp<TrilinearPoly<false, false, false, true>, false, true, 15>(*a, s);
        case 25: return launch_single<TrilinearPoly<false, false, false, true, false, false, true>, false, true, 8>(*a, s);
        case 27: return launch_double<TrilinearPoly<false, false, false, true, false, false, true>, false, true, 8>(*a, s);
        case 30: return launch_single<TrilinearPoly<false, false, false, true, false, false, true>, false, true, 10>(*a, s);
        // default: vertices read by stage A from L1 (no staging barrier; +1 % under bench conditions)
        default: return launch_single<TrilinearPoly<false, false, false, true, false, false, true>, false, true, 10, true>(*a, s);
      }
    case HX_TRILINEAR_PARTIAL:
      if (hook == 1) return launch<TrilinearPoly<false, false, true>, false, true>(*a, s);
      if (hook == 2) return launch_single<TrilinearPoly<false, false, true>, false, true, 8>(*a, s);
      return launch_single<TrilinearPoly<false, false, true, true, false, false, true>, false, true, 10, true>(*a, s);
    case HX_TRILINEAR_MERGED:
      if (hook == 1) return launch<TrilinearPoly<true, true, false>, true, true>(*a, s);
      if (hook == 2) return launch_single<TrilinearPoly<true, true, false>, true, true, 8>(*a, s);
      if (hook == 3) return launch_single<TrilinearPoly<true, true, false, true, false, false, true>, true, true, 8, true>(*a, s);
      return launch_single<TrilinearPoly<true, true, false, true, false, false, true>, true, true, 10, true>(*a, s);
    case HX_STORED:
      if (hook == 1)
        return helm ? launch<StoredLoad<true>, true, false>(*a, s) : launch<StoredLoad<false>, false, false>(*a, s);
      return helm ? launch_single<StoredLoad<true>, true, false, 8>(*a, s)
                  : launch_single<StoredLoad<false>, false, false, 8>(*a, s);
    case HX_PARALLELEPIPED:
      if (hook == 1)
        return helm ? launch<Ppd<true>, true, false>(*a, s) : launch<Ppd<false>, false, false>(*a, s);
      return helm ? launch_single<Ppd<true>, true, false, 8>(*a, s) : launch_single<Ppd<false>, false, false, 8>(*a, s);
  }
  return cudaErrorNotSupported;
}

// Basis upload hook: the common constants plus, for n1 = 8, the even-odd blocks.
extern "C" cudaError_t hx_upload_basis_fast(int n1, const double* pts, const double* w, const double* d) {
  cudaError_t err = hx_upload_basis_local(n1, pts, w, d);
  if (err != cudaSuccess || n1 != 8) return err;
  return hx::fast::n7_upload_eo(d);
}
