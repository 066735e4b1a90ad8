// AxLocal at N = 7 (n1 = 8) with the r- and s-direction contractions on the
// FP64 tensor path: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), the paper's
// Algorithm 5 re-derived for the sm_100a fragment layout.
//
// One warp per element.  Lane l = 4g + q owns the 16 nodes (i = 2q + b, j = g, k)
// for b in {0, 1} and every k: for each k-slice that is exactly the m8n8k4
// accumulator layout (row g, columns 2q and 2q + 1).  Per slice k (X_k = the
// 8 x 8 slice [j][i]):
//   Xr = X_k D^T   A = X_k, whose fragment [g][q] at k-step s is taken as
//                  X_k[g][2q + s] (the contraction index enumerated 2q + s):
//                  the thread's own two values.  B = D^T: constant D[g][2q + s].
//   Xs = D X_k     A = D: constant D[g][q + 4s].  B = X_k rows: x[k][q + 4s][g],
//                  a reload of the element's x (L1 hit).
//   node stage     rr, ss, tt at the thread's two nodes of the slice (x2 = Xt
//                  from registers).
//   Y  = rr D      A = rr: own values (enumeration 2q + s); B = D[2q + s][g].
//      + D^T ss    A = D[q + 4s][g]; B = ss rows [q + 4s][g] through a 64-double
//                  warp tile (the one transpose of the scheme); both products,
//                  and the Helmholtz mass term, accumulate in one fragment.
// The t direction is thread-local: a thread owns two whole k-fibres and
// applies D and D^T to them in registers with the even-odd form.
//
// Weight folding (sources whose factors are w (x) something: trilinear,
// parallelepiped): the node stage runs without the GLL weight w_k of the node's
// k index, and w_k enters at the end, y_k = w_k (D_r^T rr + D_s^T ss)_k +
// (D_t^T (w .* tt))_k -- an FMA on the DMMA accumulator, and w folded into the
// columns of the transposed even-odd blocks (c_EOW; w_m = w_{7-m}).  For the
// trilinear sources the per-fibre det polynomial is divided by 0.125 w_j w_i
// once, so a node needs 1/det' and no weight products at all.  The dt column of
// JT is bilinear, c(i,j) = U_j + xi_i V_j, with U/V per j from stage A.
//
// Shared traffic per element: 2 x 512 B for the ss transposes plus the
// per-element geometry tables, against ~60 KB for the three-ownership ax8s.
// FP64 work: a DMMA.8x8x4 holds the FP64 pipe for 256 FMAs (the same pipe and
// rate as DFMA on B200), so the r/s contractions cost 64 FMA per fibre instead
// of the even-odd 48, and DMMA mixed with DFMA costs ~5.6 pipe cycles per DMMA
// (profiles/r02_ubench_mix.txt); DESIGN.md §4.1a has the budget and the A/B.
//
// Per-node fields (Helmholtz lam0 / lam1, the stored scale of partial, lam2 /
// lam3 of merged) reach the node stage through shared memory: one bulk copy
// (cp.async.bulk + mbarrier) per array per element, issued before the geometry
// prologue, so no registers hold them and no load latency sits in the slices.
//
// n_col = 3 (every column bitwise an n_col = 1 apply, test_axlocal.py:180-199):
// one CTA of three warps per element, warp c on column c; the element's
// interleaved x arrives by one bulk copy and y leaves through a shared tile as
// contiguous 16-byte stores. Either each warp runs the n_col = 1 column pass
// (ax8m with CTA3), or (ax8m3) warps 0 / 1 first evaluate the per-node factors
// once into shared memory and every warp's column pass reads them back.
//
// Fused BP5 gather (every policy): x read straight from the slab lattice, the
// CG direction update p = r + beta p optionally applied on the fly.
#include "n7_common.cuh"
#include <type_traits>

// D (row-major [i][m]) for the per-lane fragments (lane-dependent indices: a
// global array read once per warp through L1, not a divergent constant load).
static __device__ double g_D8[64];
// GLL points and inverse weights for lane-dependent indices (one L1 load each,
// instead of the select chains of fast::pick8)
static __device__ double g_X8[8];
static __device__ double g_W8[8];
static __device__ double g_IW8[8];

namespace hx {
namespace mma {

using fast::N1;
using fast::N3;

static __constant__ double c_EOW[2][4][4];  // D^T even-odd blocks, column m scaled by w_m

// D = A B + C, m8n8k4 f64: A [g][q], B [q][g], C/D [g][2q], [g][2q+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Per-warp shared state.
struct ElemGeo {
  double jb[8][6];   // dr_base[3], dr_slope[3] per j (common_terms, geometry.py:135-184)
  double ib[8][6];   // ds_base[3], ds_slope[3] per i
  double uv[8][6];   // U[3], V[3] per j: dt column c(i,j) = U_j + xi_i V_j
  double xs[8];      // GLL points
  double iw[8];      // 1 / w
  double t00[8][8];  // K00 [k][j]
  double t11[8][8];  // K11 [k][i]
  double tile[2][64];
};

// Stage A of the trilinear geometry: 72 short tasks (one coordinate of a j-side
// or i-side base/slope pair, or of a U/V pair) plus the point / weight copies.
__device__ __forceinline__ void stage_a(int t, const double* __restrict__ v, ElemGeo& s) {
  if (t < 72) {
    const int side = t / 24, task = t - 24 * side, idx = task / 3, c = task % 3;
    const double xi = g_X8[idx];
    const double a0 = 1.0 - xi, a1 = 1.0 + xi;
    // j side: a0 (v1-v0) + a1 (v3-v2) | a0 (v5-v4) + a1 (v7-v6)   (geometry.py:152-167)
    // i side: a0 (v2-v0) + a1 (v3-v1) | a0 (v6-v4) + a1 (v7-v5)
    // dt col: a0 (v4-v0) + a1 (v6-v2) | a0 (v5-v1) + a1 (v7-v3)   (L | R with a = 1 -/+ xj)
    const int p0 = side == 0 ? 1 : side == 1 ? 2 : 4, q0 = 0;
    const int p1 = side == 0 ? 3 : side == 1 ? 3 : 6, q1 = side == 0 ? 2 : side == 1 ? 1 : 2;
    const int p2 = side == 0 ? 5 : side == 1 ? 6 : 5, q2 = side == 2 ? 1 : 4;
    const int p3 = 7, q3 = side == 0 ? 6 : side == 1 ? 5 : 3;
    const double lo = fma(a1, v[p1 * 3 + c] - v[q1 * 3 + c], a0 * (v[p0 * 3 + c] - v[q0 * 3 + c]));
    const double hi = fma(a1, v[p3 * 3 + c] - v[q3 * 3 + c], a0 * (v[p2 * 3 + c] - v[q2 * 3 + c]));
    double* out = side == 0 ? s.jb[idx] : side == 1 ? s.ib[idx] : s.uv[idx];
    out[c] = lo + hi;
    out[3 + c] = hi - lo;
  } else if (t < 80) {
    s.xs[t - 72] = g_X8[t - 72];
    s.iw[t - 72] = g_IW8[t - 72];
  }
}

// w .* v, then D^T: the transposed even-odd contraction with c_EOW.
__device__ __forceinline__ void eo8w(const double v[8], double out[8]) {
  double ue[4], uo[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    ue[m] = v[m] + v[7 - m];
    uo[m] = v[m] - v[7 - m];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double p = c_EOW[0][i][0] * ue[0];
    double q = c_EOW[1][i][0] * uo[0];
#pragma unroll
    for (int m = 1; m < 4; ++m) {
      p = fma(c_EOW[0][i][m], ue[m], p);
      q = fma(c_EOW[1][i][m], uo[m], q);
    }
    out[i] = p + q;
    out[7 - i] = q - p;
  }
}

// Lane context handed to the factor policies.
struct Lane {
  int g, q;
  int64_t e;
};

__device__ __forceinline__ double2 ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// (rr, ss, tt) = G (s x0, s x1, s x2) with G symmetric, the reference's row order.
__device__ __forceinline__ void symv(double g0, double g1, double g2, double g3, double g4, double g5, double s,
                                     double x0, double x1, double x2, double& rr, double& ss, double& tt) {
  const double s0 = s * x0, s1 = s * x1, s2 = s * x2;
  rr = fma(g0, s0, fma(g1, s1, g2 * s2));
  ss = fma(g1, s0, fma(g3, s1, g4 * s2));
  tt = fma(g2, s0, fma(g4, s1, g5 * s2));
}

// ---------------------------------------------------------------------------
// Factor policies (axlocal.py:171-211).  prepare() once per element after
// stage A; slice<K>() for the thread's two nodes of slice K: inputs the three
// derivatives (and x for the mass term), outputs rr, ss, tt and the mass term
// to add to y (all in the weight-folded domain when kWFold).

// Explicit FMAs (and -fmad=false for this unit, Makefile): every kernel built
// from these templates rounds identically, which the bitwise n_col = 3 ==
// 3 x n_col = 1 contract needs (contraction choices otherwise vary per instantiation).
__device__ __forceinline__ double dot3(const double* u, const double* v) {
  return fma(u[2], v[2], fma(u[1], v[1], u[0] * v[0]));
}
__device__ __forceinline__ void cross(const double* u, const double* v, double* w) {
  w[0] = fma(u[1], v[2], -(u[2] * v[1]));
  w[1] = fma(u[2], v[0], -(u[0] * v[2]));
  w[2] = fma(u[0], v[1], -(u[1] * v[0]));
}

// Polynomial-in-t trilinear geometry of one k-fibre (j = g, i); det' = det / (0.125 w_j w_i).
struct TriFibre {
  double k01[3], k02[2], k12[2], k22, det[3];
};

template <bool DET>
__device__ __forceinline__ void tri_fibre(const ElemGeo& s, const double br[3], const double sr[3],
                                          const double U[3], const double V[3], double aj, int ii, TriFibre& f) {
  double bs[3], ss[3], c[3];
  const double xi = s.xs[ii];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    bs[q] = s.ib[ii][q];
    ss[q] = s.ib[ii][3 + q];
    c[q] = fma(xi, V[q], U[q]);
  }
  f.k01[0] = dot3(br, bs);
  f.k01[1] = dot3(br, ss) + dot3(sr, bs);
  f.k01[2] = dot3(sr, ss);
  f.k02[0] = dot3(br, c);
  f.k02[1] = dot3(sr, c);
  f.k12[0] = dot3(bs, c);
  f.k12[1] = dot3(ss, c);
  f.k22 = dot3(c, c);
  if (DET) {
    // det(JT) = (br + t sr) . ((bs + t ss) x c)
    double P[3], Q[3];
    cross(bs, c, P);
    cross(ss, c, Q);
    const double gam = aj * s.iw[ii];  // 8 / (w_j w_i)
    f.det[0] = gam * dot3(br, P);
    f.det[1] = gam * (dot3(br, Q) + dot3(sr, P));
    f.det[2] = gam * dot3(sr, Q);
  }
}

// adj(K(t_K)) (unscaled g of geometry.py:329-339) of a fibre.
template <int K>
__device__ __forceinline__ void tri_adj(const TriFibre& f, double a00, double a11, double g[6]) {
  const double t = cX<N1>(K);
  const double a01 = fma(fma(f.k01[2], t, f.k01[1]), t, f.k01[0]);
  const double a02 = fma(f.k02[1], t, f.k02[0]);
  const double a12 = fma(f.k12[1], t, f.k12[0]);
  g[0] = fma(a11, f.k22, -a12 * a12);
  g[1] = fma(a02, a12, -a01 * f.k22);
  g[2] = fma(a01, a12, -a02 * a11);
  g[3] = fma(a00, f.k22, -a02 * a02);
  g[4] = fma(a01, a02, -a00 * a12);
  g[5] = fma(a00, a11, -a01 * a01);
}

// 1 / det'(t_K): MUFU seed r, e = 1 - d r, r (1 + e + e^2)  (error ~ e^3).
template <int K>
__device__ __forceinline__ double tri_rdet(const TriFibre& f, double& dt) {
  const double t = cX<N1>(K);
  dt = fma(fma(f.det[2], t, f.det[1]), t, f.det[0]);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(dt));
  const double e = fma(-dt, r, 1.0);
  return fma(fma(e, e, e), r, r);
}

// K00(j = jj, k = kk) and K11(i = jj, k = kk) table entries.
__device__ __forceinline__ void tri_tables(ElemGeo& S, int jj, int kk) {
  const double tk = S.xs[kk];
  double cr[3], cs[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    cr[c] = fma(tk, S.jb[jj][3 + c], S.jb[jj][c]);
    cs[c] = fma(tk, S.ib[jj][3 + c], S.ib[jj][c]);
  }
  S.t00[kk][jj] = dot3(cr, cr);
  S.t11[kk][jj] = dot3(cs, cs);
}

// Fibre (j = g, i = 2q + b).
template <bool DET>
__device__ __forceinline__ void tri_fibre_of(const ElemGeo& S, const Lane& L, int b, TriFibre& f) {
  double br[3], sr[3], U[3], V[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    br[c] = S.jb[L.g][c];
    sr[c] = S.jb[L.g][3 + c];
    U[c] = S.uv[L.g][c];
    V[c] = S.uv[L.g][3 + c];
  }
  tri_fibre<DET>(S, br, sr, U, V, 8.0 * S.iw[L.g], 2 * L.q + b, f);
}

// Shared by the trilinear policies: the K00 / K11 tables and the two fibres.
template <bool DET>
__device__ __forceinline__ void tri_prepare(ElemGeo& S, const Lane& L, TriFibre f[2]) {
  tri_tables(S, L.g, 2 * L.q);
  tri_tables(S, L.g, 2 * L.q + 1);
  tri_fibre_of<DET>(S, L, 0, f[0]);
  tri_fibre_of<DET>(S, L, 1, f[1]);
}

// Trilinear recompute, Poisson or Helmholtz (axlocal.py:191-201).
template <bool HELM>
struct Tri {
  static constexpr bool kTri = true, kWFold = true, kGather = true, kFields = HELM;
  TriFibre f[2];
  const double* lam0;  // (E, n3) fields or null (scalars)
  const double* lam1;
  double l0v, l1v, cm[2];
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, ElemGeo& S, const Lane& L) {
    tri_prepare<true>(S, L, f);
    if (HELM) {
      lam0 = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
      lam1 = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
      l0v = a.lam0_value;
      l1v = a.lam1_value;
      // mass = lam1 lam_geo det^2 / 64 = w_k lam1 det' (0.125 w_j w_i)^2 / 64
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const double wji8 = 0.125 * (g_W8[L.g] * g_W8[2 * L.q + b]);
        cm[b] = 0.015625 * (wji8 * wji8);
      }
    }
  }
  // lam0 / lam1 fields staged in shared memory by the kernel (bulk copy per element)
  static constexpr int kStage = HELM ? 2 : 0;
  __device__ __forceinline__ static const double* stage_base(const hx_axlocal_args& a, int f) {
    return f == 0 ? a.lam0 : a.lam1;
  }
  const double* sf;
  struct Fld {
    double2 l0, l1;
  };
  template <int K>
  __device__ __forceinline__ void load(const Lane& L, Fld& fl) const {
    if (HELM) {
      const int n = K * 64 + L.g * 8 + 2 * L.q;
      fl.l0 = lam0 ? *reinterpret_cast<const double2*>(sf + n) : make_double2(l0v, l0v);
      fl.l1 = lam1 ? *reinterpret_cast<const double2*>(sf + N3 + n) : make_double2(l1v, l1v);
    }
  }
  template <int K>
  __device__ __forceinline__ void slice(const ElemGeo& S, const Lane& L, const double x0[2], const double x1[2],
                                        const double x2[2], const double xk[2], double rr[2], double ss[2],
                                        double tt[2], double ms[2], const Fld& fl) const {
    const double a00 = S.t00[K][L.g];
    const double2 a11 = *reinterpret_cast<const double2*>(&S.t11[K][2 * L.q]);
    const double2 l0 = fl.l0, l1 = fl.l1;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      double g[6], dt;
      tri_adj<K>(f[b], a00, b ? a11.y : a11.x, g);
      double sc = tri_rdet<K>(f[b], dt);
      if (HELM) {
        ms[b] = ((b ? l1.y : l1.x) * (dt * cm[b])) * xk[b];
        sc = (b ? l0.y : l0.x) * sc;
      }
      symv(g[0], g[1], g[2], g[3], g[4], g[5], sc, x0[b], x1[b], x2[b], rr[b], ss[b], tt[b]);
    }
  }

  // n_col = 3 factor reuse (ax8m3): the same arithmetic split into the per-node
  // factors (g, scale[, mass coefficient]) and their application to one column.
  static constexpr int kNF = HELM ? 8 : 7;
  // n_col = 3 through ax8m3's factor reuse (Poisson 159 vs 148, Helmholtz 133 vs 128
  // GDOF/s per-column; profiles/r02_mma3_xstage_ab.txt)
  static constexpr bool kReuse3 = true;
  __device__ __forceinline__ void prepare_one(const hx_axlocal_args& a, const ElemGeo& S, const Lane& L, int b) {
    tri_fibre_of<true>(S, L, b, f[b]);
    if (HELM) {
      lam0 = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
      lam1 = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
      l0v = a.lam0_value;
      l1v = a.lam1_value;
      const double wji8 = 0.125 * (g_W8[L.g] * g_W8[2 * L.q + b]);
      cm[b] = 0.015625 * (wji8 * wji8);
    }
  }
  template <int K>
  __device__ __forceinline__ void node_factors(const ElemGeo& S, const Lane& L, int b, double v[kNF]) const {
    double dt;
    tri_adj<K>(f[b], S.t00[K][L.g], S.t11[K][2 * L.q + b], v);
    double sc = tri_rdet<K>(f[b], dt);
    if (HELM) {
      const int n = K * 64 + L.g * 8 + 2 * L.q + b;
      const double l0 = lam0 ? (sf ? sf[n] : __ldg(lam0 + n)) : l0v;
      const double l1 = lam1 ? (sf ? sf[N3 + n] : __ldg(lam1 + n)) : l1v;
      v[7] = l1 * (dt * cm[b]);
      sc = l0 * sc;
    }
    v[6] = sc;
  }
  __device__ __forceinline__ static void apply(const double v[kNF], double x0, double x1, double x2, double xk,
                                               double& rr, double& ss, double& tt, double& ms) {
    if (HELM) ms = v[7] * xk;
    symv(v[0], v[1], v[2], v[3], v[4], v[5], v[6], x0, x1, x2, rr, ss, tt);
  }
};

// Trilinear with a stored per-node scale: partial (Poisson, lam_geo) or
// merged (Helmholtz, lam2 / lam3) -- the stored scales carry w_k (no folding).
template <bool MERGED>
struct TriStoredScale {
  static constexpr bool kTri = true, kWFold = false, kGather = true, kFields = true;
  TriFibre f[2];
  const double* sa;  // lam_geo or lam2
  const double* sb;  // lam3
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, ElemGeo& S, const Lane& L) {
    tri_prepare<false>(S, L, f);
    sa = (MERGED ? a.lam2 : a.lam_geo) + L.e * N3;
    sb = MERGED ? a.lam3 + L.e * N3 : nullptr;
  }
  // the stored scale(s) staged in shared memory by the kernel (bulk copy per element)
  static constexpr int kStage = MERGED ? 2 : 1;
  __device__ __forceinline__ static const double* stage_base(const hx_axlocal_args& a, int f) {
    return MERGED ? (f == 0 ? a.lam2 : a.lam3) : a.lam_geo;
  }
  const double* sf;
  struct Fld {
    double2 s2, m2;
  };
  template <int K>
  __device__ __forceinline__ void load(const Lane& L, Fld& fl) const {
    const int n = K * 64 + L.g * 8 + 2 * L.q;
    fl.s2 = *reinterpret_cast<const double2*>(sf + n);
    fl.m2 = MERGED ? *reinterpret_cast<const double2*>(sf + N3 + n) : make_double2(0.0, 0.0);
  }
  template <int K>
  __device__ __forceinline__ void slice(const ElemGeo& S, const Lane& L, const double x0[2], const double x1[2],
                                        const double x2[2], const double xk[2], double rr[2], double ss[2],
                                        double tt[2], double ms[2], const Fld& fl) const {
    const double a00 = S.t00[K][L.g];
    const double2 a11 = *reinterpret_cast<const double2*>(&S.t11[K][2 * L.q]);
    const double2 s2 = fl.s2, m2 = fl.m2;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      double g[6];
      tri_adj<K>(f[b], a00, b ? a11.y : a11.x, g);
      symv(g[0], g[1], g[2], g[3], g[4], g[5], b ? s2.y : s2.x, x0[b], x1[b], x2[b], rr[b], ss[b], tt[b]);
      if (MERGED) ms[b] = (b ? m2.y : m2.x) * xk[b];
    }
  }

  static constexpr int kNF = MERGED ? 8 : 7;
  // n_col = 3: partial through ax8m3's factor reuse (161 vs 151 GDOF/s per-column),
  // merged as per-column warps (148 vs 143; profiles/r02_mma3_xstage_ab.txt)
  static constexpr bool kReuse3 = !MERGED;
  __device__ __forceinline__ void prepare_one(const hx_axlocal_args& a, const ElemGeo& S, const Lane& L, int b) {
    tri_fibre_of<false>(S, L, b, f[b]);
    sa = (MERGED ? a.lam2 : a.lam_geo) + L.e * N3;
    sb = MERGED ? a.lam3 + L.e * N3 : nullptr;
  }
  template <int K>
  __device__ __forceinline__ void node_factors(const ElemGeo& S, const Lane& L, int b, double v[kNF]) const {
    tri_adj<K>(f[b], S.t00[K][L.g], S.t11[K][2 * L.q + b], v);
    const int n = K * 64 + L.g * 8 + 2 * L.q + b;
    v[6] = sf ? sf[n] : __ldg(sa + n);
    if (MERGED) v[7] = sf ? sf[N3 + n] : __ldg(sb + n);
  }
  __device__ __forceinline__ static void apply(const double v[kNF], double x0, double x1, double x2, double xk,
                                               double& rr, double& ss, double& tt, double& ms) {
    symv(v[0], v[1], v[2], v[3], v[4], v[5], v[6], x0, x1, x2, rr, ss, tt);
    if (MERGED) ms = v[7] * xk;
  }
};

// The per-node factors of a trilinear policy read back from shared memory
// (ax8m3's column pass): [slice][factor][lane] pairs for the lane's two fibres.
template <typename F>
struct FacLoaded {
  static constexpr bool kTri = true, kWFold = F::kWFold;
  const double2 (*fac)[F::kNF][32];
  static constexpr int kStage = 0;
  __device__ __forceinline__ static const double* stage_base(const hx_axlocal_args&, int) { return nullptr; }
  const double* sf;
  struct Fld {};  // loads stay in the slice
  template <int K>
  __device__ __forceinline__ void load(const Lane&, Fld&) const {}
  template <int K>
  __device__ __forceinline__ void slice(const ElemGeo&, const Lane& L, const double x0[2], const double x1[2],
                                        const double x2[2], const double xk[2], double rr[2], double ss[2],
                                        double tt[2], double ms[2], const Fld& fl) const {
    const int lane = L.g * 4 + L.q;
    double v0[F::kNF], v1[F::kNF];
#pragma unroll
    for (int c = 0; c < F::kNF; ++c) {
      const double2 p = fac[K][c][lane];
      v0[c] = p.x;
      v1[c] = p.y;
    }
    F::apply(v0, x0[0], x1[0], x2[0], xk[0], rr[0], ss[0], tt[0], ms[0]);
    F::apply(v1, x0[1], x1[1], x2[1], xk[1], rr[1], ss[1], tt[1], ms[1]);
  }
};

// Parallelepiped: g = w (x) h (geometry.py:389-398), w_j w_i per fibre, w_k folded.
template <bool HELM>
struct Ppd {
  static constexpr bool kTri = false, kWFold = true, kGather = true, kFields = HELM;
  double h[7], wji[2];
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, ElemGeo&, const Lane& L) {
#pragma unroll
    for (int c = 0; c < 7; ++c) h[c] = __ldg(a.h + L.e * 7 + c);
    wji[0] = g_W8[L.g] * g_W8[2 * L.q];
    wji[1] = g_W8[L.g] * g_W8[2 * L.q + 1];
    if (HELM) {
      lam0 = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
      lam1 = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
      l0v = a.lam0_value;
      l1v = a.lam1_value;
    }
  }
  // lam0 / lam1 fields staged in shared memory by the kernel (bulk copy per element)
  static constexpr int kStage = HELM ? 2 : 0;
  __device__ __forceinline__ static const double* stage_base(const hx_axlocal_args& a, int f) {
    return f == 0 ? a.lam0 : a.lam1;
  }
  const double* sf;
  struct Fld {
    double2 l0, l1;
  };
  template <int K>
  __device__ __forceinline__ void load(const Lane& L, Fld& fl) const {
    if (HELM) {
      const int n = K * 64 + L.g * 8 + 2 * L.q;
      fl.l0 = lam0 ? *reinterpret_cast<const double2*>(sf + n) : make_double2(l0v, l0v);
      fl.l1 = lam1 ? *reinterpret_cast<const double2*>(sf + N3 + n) : make_double2(l1v, l1v);
    }
  }
  template <int K>
  __device__ __forceinline__ void slice(const ElemGeo&, const Lane& L, const double x0[2], const double x1[2],
                                        const double x2[2], const double xk[2], double rr[2], double ss[2],
                                        double tt[2], double ms[2], const Fld& fl) const {
    const double2 l0 = fl.l0, l1 = fl.l1;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      symv(h[0], h[1], h[2], h[3], h[4], h[5], wji[b], x0[b], x1[b], x2[b], rr[b], ss[b], tt[b]);
      if (HELM) {
        const double l = b ? l0.y : l0.x;
        rr[b] *= l;
        ss[b] *= l;
        tt[b] *= l;
        ms[b] = ((b ? l1.y : l1.x) * (wji[b] * h[6])) * xk[b];
      }
    }
  }
};

// Stored (Nek-style) factors: 6 (+gwj) SoA loads per node (axlocal.py:181-185).
template <bool HELM>
struct Stored {
  static constexpr bool kTri = false, kWFold = false, kGather = true, kFields = HELM;
  const double* gp;
  const double* gwj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, ElemGeo&, const Lane& L) {
    gp = a.g + L.e * 6 * N3;
    if (HELM) {
      gwj = a.gwj + L.e * N3;
      lam0 = a.lam0 ? a.lam0 + L.e * N3 : nullptr;
      lam1 = a.lam1 ? a.lam1 + L.e * N3 : nullptr;
      l0v = a.lam0_value;
      l1v = a.lam1_value;
    }
  }
  static constexpr int kStage = 0;
  __device__ __forceinline__ static const double* stage_base(const hx_axlocal_args&, int) { return nullptr; }
  const double* sf;
  struct Fld {};  // loads stay in the slice
  template <int K>
  __device__ __forceinline__ void load(const Lane&, Fld&) const {}
  template <int K>
  __device__ __forceinline__ void slice(const ElemGeo&, const Lane& L, const double x0[2], const double x1[2],
                                        const double x2[2], const double xk[2], double rr[2], double ss[2],
                                        double tt[2], double ms[2], const Fld& fl) const {
    const int n = K * 64 + L.g * 8 + 2 * L.q;
    double2 gg[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) gg[c] = ld2(gp + c * N3 + n);
    double2 l0 = make_double2(l0v, l0v), l1 = make_double2(l1v, l1v), gw = make_double2(0.0, 0.0);
    if (HELM) {
      if (lam0) l0 = ld2(lam0 + n);
      if (lam1) l1 = ld2(lam1 + n);
      gw = ld2(gwj + n);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double g0 = b ? gg[0].y : gg[0].x, g1 = b ? gg[1].y : gg[1].x, g2 = b ? gg[2].y : gg[2].x;
      const double g3 = b ? gg[3].y : gg[3].x, g4 = b ? gg[4].y : gg[4].x, g5 = b ? gg[5].y : gg[5].x;
      rr[b] = fma(g0, x0[b], fma(g1, x1[b], g2 * x2[b]));
      ss[b] = fma(g1, x0[b], fma(g3, x1[b], g4 * x2[b]));
      tt[b] = fma(g2, x0[b], fma(g4, x1[b], g5 * x2[b]));
      if (HELM) {
        const double l = b ? l0.y : l0.x;
        rr[b] *= l;
        ss[b] *= l;
        tt[b] *= l;
        ms[b] = ((b ? l1.y : l1.x) * (b ? gw.y : gw.x)) * xk[b];
      }
    }
  }
};

#ifndef HX_MMA3_NREG
#define HX_MMA3_NREG 168  // ax8m3: 4 CTAs (12 warps) / SM; 150 vs 145 GDOF/s at 128 (profiles/r02_mma_c3_ab.txt)
#endif
#ifndef HX_MMA_AHEAD_WAVES4
#define HX_MMA_AHEAD_WAVES4 5  // L2 prefetch distance in quarter waves of resident warps
#endif

// Where a column's x comes from: element-local (E, n1^3, NCOL), or (GATHER)
// the slab lattice of the fused BP5 gather -- node (i,j,k) of element (cx,cy,cz)
// is lattice point (7 cx + i, 7 cy + j, 7 cz + k), the index computed, not
// loaded -- optionally (CGP) with the CG direction update p = r + beta p_old
// applied on the fly (the rounding of cg_p_kernel, solver.py:170) and the
// thread's own nodes of p written to cg_p_out.
template <int NCOL, bool GATHER, bool CGP>
struct XSrc {
  const double* x;
  const double* r;
  double* pout;
  int64_t sk, sj;  // strides of k and j (i stride: NCOL, or 1 on the lattice)
  double beta;
  __device__ __forceinline__ XSrc(const hx_axlocal_args& a, const Lane& L, int col) {
    if (GATHER) {
      const hx_box& bx = a.gather_box;
      const int64_t nx = (int64_t)bx.ex * 7 + 1, ny = (int64_t)bx.ey * 7 + 1;
      const unsigned e32 = (unsigned)L.e, exu = (unsigned)bx.ex, exy = exu * (unsigned)bx.ey;
      const unsigned cz = e32 / exy, rem = e32 - cz * exy, cy = rem / exu, cx = rem - cy * exu;
      const int64_t base = ((int64_t)(cz * 7) * ny + cy * 7) * nx + cx * 7;
      x = a.x + base;
      sk = nx * ny;
      sj = nx;
      if (CGP) {
        r = a.cg_r + base;
        pout = a.cg_p_out + base;
        beta = a.cg_scal[2] / a.cg_scal[0];
      }
    } else {
      x = a.x + L.e * N3 * NCOL + col;
      sk = 64 * NCOL;
      sj = 8 * NCOL;
    }
  }
  __device__ __forceinline__ int64_t off(int k, int j, int i) const {
    return k * sk + j * sj + (GATHER ? i : i * NCOL);
  }
  __device__ __forceinline__ double at(int k, int j, int i) const {
    const int64_t o = off(k, j, i);
    if (CGP) return __dadd_rn(__ldg(r + o), __dmul_rn(beta, __ldg(x + o)));
    return __ldg(x + o);
  }
  // the thread's pair of nodes (k, j, i), (k, j, i + 1)
  __device__ __forceinline__ void pair(int k, int j, int i, double& v0, double& v1) const {
    if (NCOL == 1 && !GATHER) {
      const double2 v = ld2(x + off(k, j, i));
      v0 = v.x;
      v1 = v.y;
    } else {
      v0 = at(k, j, i);
      v1 = at(k, j, i + 1);
      if (CGP) {
        const int64_t o = off(k, j, i);
        pout[o] = v0;
        pout[o + 1] = v1;
      }
    }
  }
};

// n_col = 3 in a 3-warp CTA: the element's interleaved x (n1^3 x 3) staged in
// shared memory, warp col reading its column (stride 3 doubles: conflict-free)
struct XStaged3 {
  const double* x;
  __device__ __forceinline__ XStaged3(const double* xs, int col) : x(xs + col) {}
  __device__ __forceinline__ double at(int k, int j, int i) const { return x[(k * 64 + j * 8 + i) * 3]; }
  __device__ __forceinline__ void pair(int k, int j, int i, double& v0, double& v1) const {
    v0 = at(k, j, i);
    v1 = at(k, j, i + 1);
  }
};

template <typename XS, int NCOL, bool GATHER, bool CGP>
__device__ __forceinline__ XS make_xs(const hx_axlocal_args& a, const Lane& L, int col, const double* sx) {
  if constexpr (std::is_same<XS, XStaged3>::value)
    return XStaged3(sx, col);
  else
    return XSrc<NCOL, GATHER, CGP>(a, L, col);
}

// The element's y from a column-major shared tile [3][512] to the interleaved
// (512 x 3) rows in global memory: thread v takes nodes 2v, 2v+1, reads their
// three columns (16-byte, conflict-free) and writes 48 contiguous bytes. (The
// row-major tile written by the column warps had 4-way bank conflicts:
// profiles/r02_ncu_mma_ncol3.txt.)
__device__ __forceinline__ void store_y_tile3(const double* __restrict__ sy, double* __restrict__ y) {
  for (int v = threadIdx.x; v < N3 / 2; v += 96) {
    const double2 c0 = *reinterpret_cast<const double2*>(sy + 2 * v);
    const double2 c1 = *reinterpret_cast<const double2*>(sy + N3 + 2 * v);
    const double2 c2 = *reinterpret_cast<const double2*>(sy + 2 * N3 + 2 * v);
    double2* d = reinterpret_cast<double2*>(y + 6 * v);
    d[0] = make_double2(c0.x, c1.x);
    d[1] = make_double2(c2.x, c0.y);
    d[2] = make_double2(c1.y, c2.y);
  }
}

// One column of one element: x -> y, with the geometry prepared.
// The transposed r / s products of a slice, accumulated into (y0, y1) from
// the mass term ms: one order for every kernel built from these templates
// (the bitwise n_col contract).
#if !defined(HX_MMA_YR_FIRST)  // D_s^T ss first: +1 % over D_r^T rr first (profiles/r02_mma_sched_ab.txt)
#define HX_MMA_Y(K)                                          \
  dmma(y0, y1, Dy[0], tl[q * 8 + g], ms[0], ms[1]);          \
  dmma(y0, y1, Dy[1], tl[(q + 4) * 8 + g], y0, y1);          \
  dmma(y0, y1, rr[0], Dt[0], y0, y1);                        \
  dmma(y0, y1, rr[1], Dt[1], y0, y1);
#else
#define HX_MMA_Y(K)                                          \
  dmma(y0, y1, rr[0], Dt[0], ms[0], ms[1]);                  \
  dmma(y0, y1, rr[1], Dt[1], y0, y1);                        \
  dmma(y0, y1, Dy[0], tl[q * 8 + g], y0, y1);                \
  dmma(y0, y1, Dy[1], tl[(q + 4) * 8 + g], y0, y1);
#endif

// xa / xb: the thread's two k-fibres of x, loaded by the caller before the
// geometry prologue so that their latency hides behind it.
// X: XSrc (global / lattice) or XStaged3 (shared).  Where y goes (YOut): to
// global memory, into the element's (512 x 3) y tile ysh in shared memory
// (written back by the CTA), or back to the caller in xa / xb.
enum class YOut { kGlobal, kTile, kRegs };
template <typename F, int NCOL, typename XS, YOut YO = YOut::kGlobal>
__device__ __forceinline__ void column(const hx_axlocal_args& a, ElemGeo& S, double (*tiles)[64], const F& fac,
                                       const Lane& L, const XS& X, double xa[8], double xb[8], const double Dr[2],
                                       const double Ds[2], const double Dt[2], const double Dy[2], int col,
                                       double* ysh = nullptr) {
  const int g = L.g, q = L.q;
  double ta[8], tb[8];
  fast::eo8<0>(xa, ta);
  fast::eo8<0>(xb, tb);


  // forward r / s derivatives of slice K (two chained DMMAs each)
#define HX_FWD(K, X0, X1)                                               \
  double X0[2], X1[2];                                                  \
  typename F::Fld X0##_fl;                                              \
  fac.template load<K>(L, X0##_fl); /* fields one pipeline step ahead */ \
  {                                                                     \
    dmma(X0[0], X0[1], xa[K], Dr[0], 0.0, 0.0);                         \
    dmma(X0[0], X0[1], xb[K], Dr[1], X0[0], X0[1]);                     \
    const double bx0 = X.at(K, q, g), bx1 = X.at(K, q + 4, g);          \
    dmma(X1[0], X1[1], Ds[0], bx0, 0.0, 0.0);                           \
    dmma(X1[0], X1[1], Ds[1], bx1, X1[0], X1[1]);                       \
  }
  // node stage and transposed r / s of slice K, from its forward derivatives
#define HX_BWD(K, X0, X1)                                                                \
  {                                                                                      \
    double x2[2] = {ta[K], tb[K]}, xk[2] = {xa[K], xb[K]};                               \
    double rr[2], ss[2], tt[2], ms[2] = {0.0, 0.0};                                      \
    fac.template slice<K>(S, L, X0, X1, x2, xk, rr, ss, tt, ms, X0##_fl);               \
    ta[K] = tt[0];                                                                       \
    tb[K] = tt[1];                                                                       \
    double* tl = tiles[K & 1];                                                           \
    *reinterpret_cast<double2*>(tl + g * 8 + 2 * q) = make_double2(ss[0], ss[1]);        \
    __syncwarp();                                                                        \
    double y0, y1;                                                                       \
    HX_MMA_Y(K)                                                                          \
    xa[K] = y0;                                                                          \
    xb[K] = y1;                                                                          \
  }
#if !defined(HX_MMA_NO_PIPE) && !defined(HX_MMA_PIPE2)
  // software pipeline (+2 % with Ys first, profiles/r02_mma_sched_ab.txt): slice K+1's forward DMMAs are issued ahead of slice K's node stage
  HX_FWD(0, f0a, f0b)
  HX_FWD(1, f1a, f1b) HX_BWD(0, f0a, f0b)
  HX_FWD(2, f2a, f2b) HX_BWD(1, f1a, f1b)
  HX_FWD(3, f3a, f3b) HX_BWD(2, f2a, f2b)
  HX_FWD(4, f4a, f4b) HX_BWD(3, f3a, f3b)
  HX_FWD(5, f5a, f5b) HX_BWD(4, f4a, f4b)
  HX_FWD(6, f6a, f6b) HX_BWD(5, f5a, f5b)
  HX_FWD(7, f7a, f7b) HX_BWD(6, f6a, f6b)
  HX_BWD(7, f7a, f7b)
#elif defined(HX_MMA_PIPE2)
  HX_FWD(0, f0a, f0b) HX_FWD(1, f1a, f1b)
  HX_FWD(2, f2a, f2b) HX_BWD(0, f0a, f0b)
  HX_FWD(3, f3a, f3b) HX_BWD(1, f1a, f1b)
  HX_FWD(4, f4a, f4b) HX_BWD(2, f2a, f2b)
  HX_FWD(5, f5a, f5b) HX_BWD(3, f3a, f3b)
  HX_FWD(6, f6a, f6b) HX_BWD(4, f4a, f4b)
  HX_FWD(7, f7a, f7b) HX_BWD(5, f5a, f5b)
  HX_BWD(6, f6a, f6b) HX_BWD(7, f7a, f7b)
#else
#define HX_SLICE(K, A, B) { HX_FWD(K, A, B) HX_BWD(K, A, B) }
  HX_SLICE(0, f0a, f0b) HX_SLICE(1, f1a, f1b) HX_SLICE(2, f2a, f2b) HX_SLICE(3, f3a, f3b)
  HX_SLICE(4, f4a, f4b) HX_SLICE(5, f5a, f5b) HX_SLICE(6, f6a, f6b) HX_SLICE(7, f7a, f7b)
#undef HX_SLICE
#endif
#undef HX_FWD
#undef HX_BWD

  double ya[8], yb[8];
  if (F::kWFold) {
    eo8w(ta, ya);
    eo8w(tb, yb);
  } else {
    fast::eo8<1>(ta, ya);
    fast::eo8<1>(tb, yb);
  }
  double* ye = a.y + L.e * N3 * NCOL + col;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double y0, y1;
    if (F::kWFold) {
      const double wk = cW<N1>(k);
      y0 = fma(wk, xa[k], ya[k]);
      y1 = fma(wk, xb[k], yb[k]);
    } else {
      y0 = xa[k] + ya[k];
      y1 = xb[k] + yb[k];
    }
    const int n = k * 64 + g * 8 + 2 * q;
    if constexpr (YO == YOut::kRegs) {
      xa[k] = y0;
      xb[k] = y1;
    } else if constexpr (YO == YOut::kTile) {
      *reinterpret_cast<double2*>(ysh + col * N3 + n) = make_double2(y0, y1);  // column-major tile
    } else if constexpr (NCOL == 1) {
      *reinterpret_cast<double2*>(ye + n) = make_double2(y0, y1);
    } else {
      ye[n * NCOL] = y0;
      ye[(n + 1) * NCOL] = y1;
    }
  }
}

// NREG: register cap (__maxnreg__); 65536 / (32 NREG) warps per SM are resident.
// n_col = 3: one warp per (element, column), each the n_col = 1 arithmetic;
// CTA3: the element's three column warps in one CTA (one SM, so the strided
// column loads of x share L1 lines), else one CTA per (element, column).
template <typename F, int NCOL, int NREG, bool GATHER = false, bool CGP = false, bool CTA3 = false>
#ifdef HX_MMA_LAUNCH_BOUNDS  // register budget as launch bounds instead of a cap (A/B: +0.2 %, within noise)
__global__ void __launch_bounds__(CTA3 ? 96 : 32, 65536 / (32 * NREG) / (CTA3 ? 3 : 1))
#else
__global__ void __maxnreg__(NREG)
#endif
ax8m(const __grid_constant__ hx_axlocal_args a) {
  constexpr int MINB = 65536 / (32 * NREG);
  __shared__ ElemGeo S_[CTA3 ? NCOL : 1];
  const int lane = threadIdx.x & 31;
  const int col = NCOL == 1 ? 0 : CTA3 ? (int)(threadIdx.x >> 5) : (int)(blockIdx.x % NCOL);
  ElemGeo& S = S_[CTA3 ? col : 0];
  Lane L;
  L.e = NCOL == 1 || CTA3 ? (int64_t)blockIdx.x : (int64_t)(blockIdx.x / NCOL);
  L.g = lane >> 2;
  L.q = lane & 3;

  // the element's per-node field arrays (F::kStage of them: Helmholtz lam0 /
  // lam1, the stored scales of partial / merged) land in shared memory by one
  // bulk copy each, issued first and waited for after the geometry prologue:
  // no registers held for them and no load latency inside the slices
  // (one copy per CTA: the CTA3 column warps share it)
  // XST (n_col = 3 in one CTA): the element's interleaved x staged the same way, and
  // y written back from a shared tile as contiguous 16-byte stores (the strided
  // per-column accesses otherwise stall on store drain and the LSU queue)
  constexpr int NS = F::kStage;
  constexpr bool XST = CTA3 && NCOL == 3 && !GATHER;
  __shared__ alignas(128) double sf[NS > 0 ? NS * N3 : 2];
  __shared__ alignas(128) double sxy[XST ? 2 * 3 * N3 : 2];  // x tile, y tile
  __shared__ uint64_t bar[1];
  bool staged = XST;
  if constexpr (NS > 0 || XST) {
#pragma unroll
    for (int f = 0; f < NS; ++f) staged |= F::stage_base(a, f) != nullptr;
    if (staged && threadIdx.x == 0) {
      uint32_t bytes = XST ? 8u * 3 * N3 : 0u;
#pragma unroll
      for (int f = 0; f < NS; ++f) bytes += F::stage_base(a, f) ? 8u * N3 : 0u;
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, bytes);
      if (XST) bulk_g2s(sxy, a.x + L.e * 3 * N3, 8u * 3 * N3, bar);
#pragma unroll
      for (int f = 0; f < NS; ++f)
        if (const double* src = F::stage_base(a, f)) bulk_g2s(sf + f * N3, src + L.e * N3, 8u * N3, bar);
    }
  }

  // warm L2 with the element ~1.25 waves of resident warps ahead: x, vertices,
  // and the per-node fields of the variants that stream them
  if (lane < 2 && col == 0) {
    const int64_t ahead = L.e + (int64_t)148 * MINB * HX_MMA_AHEAD_WAVES4 / 4 / NCOL;
    if (ahead < a.n_elements) {
      if (lane == 0) {
        if (!GATHER) bulk_prefetch_l2(a.x + ahead * N3 * NCOL, 4096u * NCOL);
        if (F::kTri) bulk_prefetch_l2(a.verts + ahead * 24, 192u);
      } else if (F::kFields) {
        if (a.lam_geo) bulk_prefetch_l2(a.lam_geo + ahead * N3, 4096u);
        if (a.lam2) bulk_prefetch_l2(a.lam2 + ahead * N3, 4096u);
        if (a.lam3) bulk_prefetch_l2(a.lam3 + ahead * N3, 4096u);
        if (a.lam0) bulk_prefetch_l2(a.lam0 + ahead * N3, 4096u);
        if (a.lam1) bulk_prefetch_l2(a.lam1 + ahead * N3, 4096u);
      }
    }
  }
  if (GATHER) {
    // fused gather: warm the 64 lattice rows (64 B each) of the element ahead, two per lane
    const int64_t ahead = L.e + (int64_t)148 * MINB * HX_MMA_AHEAD_WAVES4 / 4;
    if (ahead < a.n_elements) {
      Lane La = L;
      La.e = ahead;
      const XSrc<1, true, false> Xa(a, La, 0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = 2 * lane + h;
        prefetch_l2(Xa.x + Xa.off(row >> 3, row & 7, 0));
        if (CGP) prefetch_l2(a.cg_r + (Xa.x - a.x) + Xa.off(row >> 3, row & 7, 0));
      }
    }
  }
  using XS = typename std::conditional<XST, XStaged3, XSrc<NCOL, GATHER, CGP>>::type;
  const XS X = make_xs<XS, NCOL, GATHER, CGP>(a, L, col, sxy);
  double xa[8], xb[8];
  if constexpr (!XST) {  // staged x is read after the barrier wait
#pragma unroll
    for (int k = 0; k < 8; ++k) X.pair(k, L.g, 2 * L.q, xa[k], xb[k]);
  }
  double Dr[2], Ds[2], Dt[2], Dy[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    Dr[s] = g_D8[L.g * 8 + 2 * L.q + s];
    Ds[s] = g_D8[L.g * 8 + L.q + 4 * s];
    Dt[s] = g_D8[(2 * L.q + s) * 8 + L.g];
    Dy[s] = g_D8[(L.q + 4 * s) * 8 + L.g];
  }
  if (F::kTri) {
    const double* vg = a.verts + L.e * 24;
    stage_a(lane, vg, S);
    stage_a(lane + 32, vg, S);
    stage_a(lane + 64, vg, S);
    __syncwarp();
  }
  F fac;
  fac.prepare(a, S, L);
  fac.sf = sf;
  if (F::kTri || NS > 0 || XST) __syncwarp();
  if constexpr (CTA3 && (NS > 0 || XST)) __syncthreads();  // the barrier's init, for the other warps
  if ((NS > 0 || XST) && staged) mbar_wait(bar, 0);
  if constexpr (XST) {
#pragma unroll
    for (int k = 0; k < 8; ++k) X.pair(k, L.g, 2 * L.q, xa[k], xb[k]);
  }
  column<F, NCOL, XS, XST ? YOut::kTile : YOut::kGlobal>(a, S, S.tile, fac, L, X, xa, xb, Dr, Ds, Dt, Dy, col,
                                                        XST ? sxy + 3 * N3 : nullptr);
  if constexpr (XST) {  // the y tile out as contiguous 16-byte stores
    __syncthreads();
    store_y_tile3(sxy + 3 * N3, a.y + L.e * 3 * N3);
  }
}

// fields staged by ax8m3: none by default -- the factor phase reads them from
// global memory, so the Helmholtz CTA fits 4 per SM instead of 3 (145 vs 121
// GDOF/s same box, profiles/r02_mma3_xstage_ab.txt); HX_MMA3_STAGE stages them (A/B)
template <typename F>
constexpr int kStage3() {
#ifdef HX_MMA3_STAGE
  return F::kStage;
#else
  return 0;
#endif
}

// n_col = 3 with factor reuse, trilinear sources: one CTA of three warps per
// element, warp c owning column c.  Stage A by the whole CTA; then warps 0 / 1
// prepare fibre b = 0 / 1 of their lanes and evaluate its per-node factors
// (adj(K), scale[, mass coefficient]) for all eight slices into shared memory
// while warp 2 fills the K00 / K11 tables; then every warp runs the n_col = 1
// column pass with the factors read back (FacLoaded), so each column is
// bitwise an n_col = 1 apply (the factors are the same roundings, stored).
template <typename F, int NREG>
__global__ void __maxnreg__(NREG) ax8m3(const __grid_constant__ hx_axlocal_args a) {
  constexpr int MINB = 65536 / (32 * NREG);
  constexpr int NS = kStage3<F>();
  __shared__ ElemGeo S;
  __shared__ double s_tile[2][2][64];  // warps 1, 2 (warp 0 uses S.tile)
  __shared__ uint64_t bar[1];
  // dynamic: the per-node factors [8][kNF][32] (then the y tile), the element's
  // interleaved x (512 x 3), the per-node fields of the factor phase
  extern __shared__ __align__(128) double dsm[];
  double2(*s_fac)[F::kNF][32] = reinterpret_cast<double2(*)[F::kNF][32]>(dsm);
  double* const sx = dsm + 2 * 8 * F::kNF * 32;
  double* const sf = sx + 3 * N3;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Lane L;
  L.e = blockIdx.x;
  L.g = lane >> 2;
  L.q = lane & 3;
  // x and the fields staged as in ax8m (one barrier for all copies)
  if (threadIdx.x == 0) {
    uint32_t bytes = 8u * 3 * N3;
#pragma unroll
    for (int f = 0; f < NS; ++f) bytes += F::stage_base(a, f) ? 8u * N3 : 0u;
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(sx, a.x + L.e * 3 * N3, 8u * 3 * N3, bar);
#pragma unroll
    for (int f = 0; f < NS; ++f)
      if (const double* src = F::stage_base(a, f)) bulk_g2s(sf + f * N3, src + L.e * N3, 8u * N3, bar);
  }
  if (threadIdx.x < 2) {
    const int64_t ahead = L.e + (int64_t)148 * MINB * HX_MMA_AHEAD_WAVES4 / 4 / 3;
    if (ahead < a.n_elements) {
      if (threadIdx.x == 0) {
        bulk_prefetch_l2(a.x + ahead * N3 * 3, 4096u * 3);
        bulk_prefetch_l2(a.verts + ahead * 24, 192u);
      } else {
        if (a.lam_geo) bulk_prefetch_l2(a.lam_geo + ahead * N3, 4096u);
        if (a.lam2) bulk_prefetch_l2(a.lam2 + ahead * N3, 4096u);
        if (a.lam3) bulk_prefetch_l2(a.lam3 + ahead * N3, 4096u);
        if (a.lam0) bulk_prefetch_l2(a.lam0 + ahead * N3, 4096u);
        if (a.lam1) bulk_prefetch_l2(a.lam1 + ahead * N3, 4096u);
      }
    }
  }
  const XStaged3 X(sx, w);
  double xa[8], xb[8];
  double Dr[2], Ds[2], Dt[2], Dy[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    Dr[s] = g_D8[L.g * 8 + 2 * L.q + s];
    Ds[s] = g_D8[L.g * 8 + L.q + 4 * s];
    Dt[s] = g_D8[(2 * L.q + s) * 8 + L.g];
    Dy[s] = g_D8[(L.q + 4 * s) * 8 + L.g];
  }
  stage_a(threadIdx.x, a.verts + L.e * 24, S);
  __syncthreads();
  {
    F fac;
    fac.sf = NS > 0 ? sf : nullptr;  // null: the factor phase reads the fields from global memory
#ifdef HX_MMA3_FIBRE_SPLIT  // warps 0 / 1 one fibre each, all slices (A/B: -3 %)
    if (w < 2) {
      fac.prepare_one(a, S, L, w);
    } else {
      tri_tables(S, lane & 7, lane >> 3);
      tri_tables(S, lane & 7, 4 + (lane >> 3));
    }
    __syncthreads();
    if (w < 2) mbar_wait(bar, 0);  // the fields (and x)
    if (w < 2) {
      double* dst = reinterpret_cast<double*>(&s_fac[0][0][lane]) + w;
#define HX_FAC(K)                                                        \
  {                                                                      \
    double v[F::kNF];                                                    \
    fac.template node_factors<K>(S, L, w, v);                            \
    _Pragma("unroll") for (int c = 0; c < F::kNF; ++c) dst[((K)*F::kNF + c) * 64] = v[c]; \
  }
      HX_FAC(0) HX_FAC(1) HX_FAC(2) HX_FAC(3) HX_FAC(4) HX_FAC(5) HX_FAC(6) HX_FAC(7)
#undef HX_FAC
    }
#else
    // warps 0 / 1: both fibres of the lane, slices 0-3 / 4-7 (double2 stores)
    if (w < 2) {
      fac.prepare_one(a, S, L, 0);
      fac.prepare_one(a, S, L, 1);
    } else {
      tri_tables(S, lane & 7, lane >> 3);
      tri_tables(S, lane & 7, 4 + (lane >> 3));
    }
    __syncthreads();
    if (w < 2) mbar_wait(bar, 0);  // the fields (and x)
#define HX_FAC(K)                                                        \
  {                                                                      \
    double v0[F::kNF], v1[F::kNF];                                       \
    fac.template node_factors<K>(S, L, 0, v0);                           \
    fac.template node_factors<K>(S, L, 1, v1);                           \
    _Pragma("unroll") for (int c = 0; c < F::kNF; ++c) s_fac[K][c][lane] = make_double2(v0[c], v1[c]); \
  }
    if (w == 0) {
      HX_FAC(0) HX_FAC(1) HX_FAC(2) HX_FAC(3)
    } else if (w == 1) {
      HX_FAC(4) HX_FAC(5) HX_FAC(6) HX_FAC(7)
    }
#undef HX_FAC
#endif
  }
  __syncthreads();
  if (w == 2) mbar_wait(bar, 0);  // x
#pragma unroll
  for (int k = 0; k < 8; ++k) X.pair(k, L.g, 2 * L.q, xa[k], xb[k]);
  FacLoaded<F> fl;
  fl.fac = s_fac;
  // each warp transposes through its own tile pair; y comes back in xa / xb
  column<FacLoaded<F>, 3, XStaged3, YOut::kRegs>(a, S, w == 0 ? S.tile : s_tile[w - 1], fl, L, X, xa, xb, Dr, Ds,
                                                 Dt, Dy, w);
  // the y tile in the factor buffer once every warp is done with the factors,
  // then out as contiguous 16-byte stores
  __syncthreads();
  double* const sy = dsm;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int n = k * 64 + L.g * 8 + 2 * L.q;
    *reinterpret_cast<double2*>(sy + w * N3 + n) = make_double2(xa[k], xb[k]);  // column-major
  }
  __syncthreads();
  store_y_tile3(sy, a.y + L.e * 3 * N3);
}

// dynamic shared memory of ax8m3<F>: factors (>= the y tile), x, staged fields
template <typename F>
constexpr size_t ax8m3_dsmem() {
  return sizeof(double) * (2 * 8 * F::kNF * 32 + 3 * N3 + kStage3<F>() * N3);
}


#ifndef HX_MMA_NREG
#define HX_MMA_NREG 168
#endif
template <typename F, int NREG = HX_MMA_NREG>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  if (a.n_elements * a.n_col > 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)(a.n_elements * a.n_col);
  if (a.gather) {  // n_col = 1 (checked by hx_axlocal)
    if constexpr (F::kGather) {
      if (a.cg_r)
        ax8m<F, 1, NREG, true, true><<<grid, 32, 0, s>>>(a);
      else
        ax8m<F, 1, NREG, true><<<grid, 32, 0, s>>>(a);
    } else {
      return cudaErrorNotSupported;
    }
  } else if (a.n_col == 3) {
    if constexpr (F::kTri) {
      // factor reuse (ax8m3) where it measures faster (F::kReuse3); else the
      // per-column 3-warp CTA below. Hooks: 71 per-column, 73 reuse (A/B)
      if (a.reserved == 73 || (F::kReuse3 && a.reserved != 71)) {
        constexpr size_t dsm = ax8m3_dsmem<F>();
        // the opt-in above 48 KB is per device: set it on every launch (~1 us host call)
        const cudaError_t e = cudaFuncSetAttribute(ax8m3<F, HX_MMA3_NREG>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
        if (e != cudaSuccess) return e;
        ax8m3<F, HX_MMA3_NREG><<<(unsigned)a.n_elements, 96, dsm, s>>>(a);
        return cudaGetLastError();
      }
    }
    if (a.reserved == 72)  // 72: one CTA per (element, column) (A/B)
      ax8m<F, 3, NREG><<<grid, 32, 0, s>>>(a);
    else
      ax8m<F, 3, NREG, false, false, true><<<(unsigned)a.n_elements, 96, 0, s>>>(a);
  }
  else
    ax8m<F, 1, NREG><<<grid, 32, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace mma
}  // namespace hx

// Every (equation, factor source, n_col) at order 7 with element-local x and
// 16-byte aligned x / y and fields, and the fused lattice gather (+ CG update) for
// every source and equation at n_col = 1; cudaErrorNotSupported otherwise.
extern "C" cudaError_t hx_mma_launch(const hx_axlocal_args* a, cudaStream_t s) {
  using namespace hx::mma;
  if (a->order != 7) return cudaErrorNotSupported;
  if (((reinterpret_cast<uintptr_t>(a->x) | reinterpret_cast<uintptr_t>(a->y)) & (a->gather ? 7u : 15u)) != 0)
    return cudaErrorNotSupported;
  // per-node fields: double2 loads and 16-byte bulk copies; vertices: the 16-byte
  // aligned L2 bulk prefetch
  const uintptr_t fields = reinterpret_cast<uintptr_t>(a->verts) |
                           reinterpret_cast<uintptr_t>(a->lam0) | reinterpret_cast<uintptr_t>(a->lam1) |
                           reinterpret_cast<uintptr_t>(a->lam2) | reinterpret_cast<uintptr_t>(a->lam3) |
                           reinterpret_cast<uintptr_t>(a->lam_geo) | reinterpret_cast<uintptr_t>(a->g) |
                           reinterpret_cast<uintptr_t>(a->gwj);
  if ((fields & 15u) != 0) return cudaErrorNotSupported;
  const bool helm = a->equation == HX_HELMHOLTZ;
  switch (a->factor_source) {
    case HX_TRILINEAR:
      if (helm) {
        // coefficient fields: 232 registers (8 warps / SM), +1.5 %; scalars: 168 (232: -0.7 %);
        // 184 / 200: -6 / -2 %. The register budget does not change the rounding (explicit
        // fma, -fmad=false), so n_col = 1 stays bitwise the ax8m3 n_col = 3 columns.
        // Hooks: 65 forces 232, 66 forces 168 (A/B)
        if (a->reserved == 65) return launch<Tri<true>, 232>(*a, s);
        if (a->reserved != 66 && (a->lam0 || a->lam1)) return launch<Tri<true>, 232>(*a, s);
        return launch<Tri<true>>(*a, s);
      }
      switch (a->reserved) {  // register-cap A/B (tools/kernel_ab.py)
        case 61: return launch<Tri<false>, 160>(*a, s);
        case 62: return launch<Tri<false>, 152>(*a, s);
        case 63: return launch<Tri<false>, 144>(*a, s);
        default: return launch<Tri<false>>(*a, s);
      }
    case HX_TRILINEAR_PARTIAL:
      return launch<TriStoredScale<false>>(*a, s);
    case HX_TRILINEAR_MERGED:
      return launch<TriStoredScale<true>>(*a, s);
    case HX_PARALLELEPIPED:
      return helm ? launch<Ppd<true>>(*a, s) : launch<Ppd<false>>(*a, s);
    case HX_STORED:
      return helm ? launch<Stored<true>>(*a, s) : launch<Stored<false>>(*a, s);
  }
  return cudaErrorNotSupported;
}

extern "C" cudaError_t hx_upload_basis_mma(int n1, const double* pts, const double* w, const double* d) {
  cudaError_t err = hx_upload_basis_local(n1, pts, w, d);
  if (err != cudaSuccess || n1 != 8) return err;
  err = hx::fast::n7_upload_eo(d);
  if (err != cudaSuccess) return err;
  double eow[2][4][4], iw[8];
  for (int i = 0; i < 4; ++i)
    for (int m = 0; m < 4; ++m) {
      const double x = d[m * 8 + i], y = d[(7 - m) * 8 + i];  // D^T[i][m], D^T[i][7-m]
      eow[0][i][m] = 0.5 * (x + y) * w[m];
      eow[1][i][m] = 0.5 * (x - y) * w[m];
    }
  for (int m = 0; m < 8; ++m) iw[m] = 1.0 / w[m];
  err = cudaMemcpyToSymbol(hx::mma::c_EOW, eow, sizeof(eow));
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(g_IW8, iw, sizeof(iw));
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(g_X8, pts, 8 * sizeof(double));
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(g_W8, w, 8 * sizeof(double));
  if (err != cudaSuccess) return err;
  return cudaMemcpyToSymbol(g_D8, d, 64 * sizeof(double));
}
