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
//                  from registers), exactly the ax8s arithmetic.
//   Y  = rr D      A = rr: own values (enumeration 2q + s); B = D[2q + s][g].
//      + D^T ss    A = D[q + 4s][g]; B = ss rows [q + 4s][g] through a 64-double
//                  warp tile (the one transpose of the scheme); both products
//                  accumulate in the same fragment.
// The t direction is thread-local: a thread owns two whole k-fibres and
// applies D and D^T to them in registers with the even-odd form.
//
// Shared traffic per element: 2 x 512 B for the ss transposes plus the
// per-element geometry tables, against ~60 KB for the three-ownership ax8s.
// FP64 work: a DMMA.8x8x4 holds the FP64 pipe for 256 FMAs (the same pipe and
// rate as DFMA on B200, profiles/r01_ubench_fp64.txt), so the r/s contractions
// cost 64 FMA per fibre instead of the even-odd 48; DESIGN.md §4.1a has the
// instruction budget and the measured A/B.
#include "n7_common.cuh"

// D (row-major [i][m]) for the per-lane fragments (lane-dependent indices: a
// global array read once per warp through L1, not a divergent constant load).
static __device__ double g_D8[64];

namespace hx {
namespace mma {

using fast::N1;
using fast::N3;

// D = A B + C, m8n8k4 f64: A [g][q], B [q][g], C/D [g][2q], [g][2q+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Per-warp shared state: stage-A terms, K00(j,k) / K11(i,k) tables, ss tiles.
struct WarpShared {
  fast::TriShared tri;  // j/i/d/xs/ws used; its own tables unused here
  double t00[8][8];     // [k][j]
  double t11[8][8];     // [k][i]
  double tile[2][64];   // ss slice [j][i], ping-pong
};

// Polynomial-in-t geometry of one k-fibre (j = g, i), TrilinearPoly::prepare.
struct Fibre {
  double k01[3], k02[2], k12[2], k22, det[3], wji8;
};

__device__ __forceinline__ void prepare_fibre(const fast::TriShared& s, int jj, int ii, Fibre& f) {
  double br[3], sr[3], bs[3], ss[3], c[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    br[q] = s.j[jj][q];
    sr[q] = s.j[jj][3 + q];
    bs[q] = s.i[ii][q];
    ss[q] = s.i[ii][3 + q];
  }
  const double xj = s.xs[jj], xi = s.xs[ii];
  const double a0j = 1.0 - xj, a1j = 1.0 + xj, a0i = 1.0 - xi, a1i = 1.0 + xi;
  const double w00 = a0j * a0i, w01 = a0j * a1i, w10 = a1j * a0i, w11 = a1j * a1i;
#pragma unroll
  for (int q = 0; q < 3; ++q) c[q] = w00 * s.d[q] + w01 * s.d[3 + q] + w11 * s.d[6 + q] + w10 * s.d[9 + q];
  using fast::dot3;
  f.k01[0] = dot3(br, bs);
  f.k01[1] = dot3(br, ss) + dot3(sr, bs);
  f.k01[2] = dot3(sr, ss);
  f.k02[0] = dot3(br, c);
  f.k02[1] = dot3(sr, c);
  f.k12[0] = dot3(bs, c);
  f.k12[1] = dot3(ss, c);
  f.k22 = dot3(c, c);
  const double P[3] = {bs[1] * c[2] - bs[2] * c[1], bs[2] * c[0] - bs[0] * c[2], bs[0] * c[1] - bs[1] * c[0]};
  const double Q[3] = {ss[1] * c[2] - ss[2] * c[1], ss[2] * c[0] - ss[0] * c[2], ss[0] * c[1] - ss[1] * c[0]};
  f.det[0] = dot3(br, P);
  f.det[1] = dot3(br, Q) + dot3(sr, P);
  f.det[2] = dot3(sr, Q);
  f.wji8 = 0.125 * (s.ws[jj] * s.ws[ii]);
}

// rr, ss, tt at node (k = K) of a fibre: the TrilinearPoly<TAB> apply_at order.
template <int K>
__device__ __forceinline__ void tri_node(const Fibre& f, double a00, double a11, double x0, double x1, double x2,
                                         double& rr, double& ss, double& tt) {
  const double t = cX<N1>(K);
  const double a01 = fma(fma(f.k01[2], t, f.k01[1]), t, f.k01[0]);
  const double a02 = fma(f.k02[1], t, f.k02[0]);
  const double a12 = fma(f.k12[1], t, f.k12[0]);
  const double g0 = fma(a11, f.k22, -a12 * a12);
  const double g1 = fma(a02, a12, -a01 * f.k22);
  const double g2 = fma(a01, a12, -a02 * a11);
  const double g3 = fma(a00, f.k22, -a02 * a02);
  const double g4 = fma(a01, a02, -a00 * a12);
  const double g5 = fma(a00, a11, -a01 * a01);
  const double dt = fma(fma(f.det[2], t, f.det[1]), t, f.det[0]);
  const double scale = fast::div_fast(cW<N1>(K) * f.wji8, dt);  // 0.125 w / det(JT)
  const double s0 = scale * x0, s1 = scale * x1, s2 = scale * x2;
  rr = fma(g0, s0, fma(g1, s1, g2 * s2));
  ss = fma(g1, s0, fma(g3, s1, g4 * s2));
  tt = fma(g2, s0, fma(g4, s1, g5 * s2));
}

#ifndef HX_MMA_AHEAD_WAVES4
#define HX_MMA_AHEAD_WAVES4 5  // L2 prefetch distance in quarter waves of resident warps
#endif

template <int WPB, int MINB>
__global__ void __launch_bounds__(32 * WPB, MINB) ax8m_v1(const __grid_constant__ hx_axlocal_args a) {
  __shared__ WarpShared s_w[WPB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * WPB + w;
  if (e >= a.n_elements) return;  // no block-wide barrier below
  const int g = lane >> 2, q = lane & 3;
  WarpShared& S = s_w[w];

  // warm L2 with the element ~1.25 waves of resident warps ahead
  if (lane == 0) {
    const int64_t ahead = e + (int64_t)148 * WPB * MINB * HX_MMA_AHEAD_WAVES4 / 4;
    if (ahead < a.n_elements) {
      bulk_prefetch_l2(a.x + ahead * N3, 4096u);
      bulk_prefetch_l2(a.verts + ahead * 24, 192u);
    }
  }
  // x in the accumulator layout: x[k][g][2q], x[k][g][2q+1] (16-B loads, 512 B per warp and k)
  const double* xe = a.x + e * N3;
  double xa[8], xb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(xe + k * 64 + g * 8 + 2 * q));
    xa[k] = v.x;
    xb[k] = v.y;
  }
  // fragments of D
  double Dr[2], Ds[2], Dt[2], Dy[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    Dr[s] = g_D8[g * 8 + 2 * q + s];
    Ds[s] = g_D8[g * 8 + q + 4 * s];
    Dt[s] = g_D8[(2 * q + s) * 8 + g];
    Dy[s] = g_D8[(q + 4 * s) * 8 + g];
  }
  // stage A (vertices straight from global / L1), then the K00 / K11 tables
  const double* vg = a.verts + e * 24;
  fast::tri_stage_a(lane, vg, S.tri);
  fast::tri_stage_a(lane + 32, vg, S.tri);
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kk = 2 * q + h;
    const double tk = S.tri.xs[kk];
    double cr[3], cs[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cr[c] = S.tri.j[g][c] + tk * S.tri.j[g][3 + c];
      cs[c] = S.tri.i[g][c] + tk * S.tri.i[g][3 + c];
    }
    S.t00[kk][g] = fast::dot3(cr, cr);
    S.t11[kk][g] = fast::dot3(cs, cs);
  }
  Fibre f0, f1;
  prepare_fibre(S.tri, g, 2 * q, f0);
  prepare_fibre(S.tri, g, 2 * q + 1, f1);
  __syncwarp();

  // t direction forward, in registers
  double ta[8], tb[8];
  fast::eo8<0>(xa, ta);
  fast::eo8<0>(xb, tb);

#define HX_SLICE(K)                                                                                \
  {                                                                                                \
    double r0, r1, s0, s1;                                                                         \
    dmma(r0, r1, xa[K], Dr[0], 0.0, 0.0);                                                          \
    dmma(r0, r1, xb[K], Dr[1], r0, r1);                                                            \
    const double bx0 = __ldg(xe + K * 64 + q * 8 + g), bx1 = __ldg(xe + K * 64 + (q + 4) * 8 + g); \
    dmma(s0, s1, Ds[0], bx0, 0.0, 0.0);                                                            \
    dmma(s0, s1, Ds[1], bx1, s0, s1);                                                              \
    const double a00 = S.t00[K][g];                                                                \
    const double2 a11 = *reinterpret_cast<const double2*>(&S.t11[K][2 * q]);                       \
    double rr0, ss0, rr1, ss1;                                                                     \
    tri_node<K>(f0, a00, a11.x, r0, s0, ta[K], rr0, ss0, ta[K]);                                   \
    tri_node<K>(f1, a00, a11.y, r1, s1, tb[K], rr1, ss1, tb[K]);                                   \
    double* tl = S.tile[K & 1];                                                                    \
    *reinterpret_cast<double2*>(tl + g * 8 + 2 * q) = make_double2(ss0, ss1);                      \
    __syncwarp();                                                                                  \
    double y0, y1;                                                                                 \
    dmma(y0, y1, rr0, Dt[0], 0.0, 0.0);                                                            \
    dmma(y0, y1, rr1, Dt[1], y0, y1);                                                              \
    dmma(y0, y1, Dy[0], tl[q * 8 + g], y0, y1);                                                    \
    dmma(y0, y1, Dy[1], tl[(q + 4) * 8 + g], y0, y1);                                              \
    xa[K] = y0;                                                                                    \
    xb[K] = y1;                                                                                    \
  }
  HX_SLICE(0) HX_SLICE(1) HX_SLICE(2) HX_SLICE(3) HX_SLICE(4) HX_SLICE(5) HX_SLICE(6) HX_SLICE(7)
#undef HX_SLICE

  // t direction transposed, in registers; y = (D_r^T rr + D_s^T ss) + D_t^T tt
  double ya[8], yb[8];
  fast::eo8<1>(ta, ya);
  fast::eo8<1>(tb, yb);
  double* ye = a.y + e * N3;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<double2*>(ye + k * 64 + g * 8 + 2 * q) = make_double2(xa[k] + ya[k], xb[k] + yb[k]);
}


// ---------------------------------------------------------------------------
// v2: the GLL weights and 0.125 w_j w_i leave the per-node work.
//  * lam_geo w_k-free: the node stage uses 1 / det'(t) with det' = det / (0.125 w_j w_i)
//    (the per-fibre det polynomial scaled once), so a node pays no weight products
//    and the reciprocal needs no numerator;
//  * w_k enters at the end: y_k = w_k (D_r^T rr' + D_s^T ss')_k + (D_t^T (w .* tt'))_k,
//    the first term an FMA on the DMMA accumulator, the second with w folded into
//    the columns of the transposed even-odd blocks (c_EOW; w_m = w_{7-m});
//  * the dt column c(i,j) = U_j + xi_i V_j (bilinear), U/V per j from stage A.
static __constant__ double c_EOW[2][4][4];  // D^T even-odd blocks, column m scaled by w_m
static __constant__ double c_IW[8];         // 1 / w_m

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

__device__ __forceinline__ void stage_a2(int t, const double* __restrict__ v, ElemGeo& s) {
  if (t < 72) {
    const int side = t / 24, task = t - 24 * side, idx = task / 3, c = task % 3;
    const double xi = fast::xr(idx);
    const double a0 = 1.0 - xi, a1 = 1.0 + xi;
    // j side: a0 (v1-v0) + a1 (v3-v2) | a0 (v5-v4) + a1 (v7-v6)
    // i side: a0 (v2-v0) + a1 (v3-v1) | a0 (v6-v4) + a1 (v7-v5)
    // dt col: a0 (v4-v0) + a1 (v6-v2) | a0 (v5-v1) + a1 (v7-v3)   (L | R, a = 1 -/+ xj)
    const int p0 = side == 0 ? 1 : side == 1 ? 2 : 4, q0 = 0;
    const int p1 = side == 0 ? 3 : side == 1 ? 3 : 6, q1 = side == 0 ? 2 : side == 1 ? 1 : 2;
    const int p2 = side == 0 ? 5 : side == 1 ? 6 : 5, q2 = side == 2 ? 1 : 4;
    const int p3 = 7, q3 = side == 0 ? 6 : side == 1 ? 5 : 3;
    const double lo = a0 * (v[p0 * 3 + c] - v[q0 * 3 + c]) + a1 * (v[p1 * 3 + c] - v[q1 * 3 + c]);
    const double hi = a0 * (v[p2 * 3 + c] - v[q2 * 3 + c]) + a1 * (v[p3 * 3 + c] - v[q3 * 3 + c]);
    double* out = side == 0 ? s.jb[idx] : side == 1 ? s.ib[idx] : s.uv[idx];
    out[c] = lo + hi;
    out[3 + c] = hi - lo;
  } else if (t < 80) {
    s.xs[t - 72] = fast::xr(t - 72);
    s.iw[t - 72] = fast::pick8(c_IW, t - 72);
  }
}

// w .* tt, then D^T: the transposed even-odd contraction with c_EOW.
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

struct Fibre2 {
  double k01[3], k02[2], k12[2], k22, det[3];  // det' = det(JT) / (0.125 w_j w_i)
};

__device__ __forceinline__ void prepare_fibre2(const ElemGeo& s, const double br[3], const double sr[3],
                                               const double U[3], const double V[3], double aj, int ii,
                                               Fibre2& f) {
  double bs[3], ss[3], c[3];
  const double xi = s.xs[ii];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    bs[q] = s.ib[ii][q];
    ss[q] = s.ib[ii][3 + q];
    c[q] = fma(xi, V[q], U[q]);
  }
  using fast::dot3;
  f.k01[0] = dot3(br, bs);
  f.k01[1] = dot3(br, ss) + dot3(sr, bs);
  f.k01[2] = dot3(sr, ss);
  f.k02[0] = dot3(br, c);
  f.k02[1] = dot3(sr, c);
  f.k12[0] = dot3(bs, c);
  f.k12[1] = dot3(ss, c);
  f.k22 = dot3(c, c);
  const double P[3] = {bs[1] * c[2] - bs[2] * c[1], bs[2] * c[0] - bs[0] * c[2], bs[0] * c[1] - bs[1] * c[0]};
  const double Q[3] = {ss[1] * c[2] - ss[2] * c[1], ss[2] * c[0] - ss[0] * c[2], ss[0] * c[1] - ss[1] * c[0]};
  const double gam = aj * s.iw[ii];  // 8 / (w_j w_i)
  f.det[0] = gam * dot3(br, P);
  f.det[1] = gam * (dot3(br, Q) + dot3(sr, P));
  f.det[2] = gam * dot3(sr, Q);
}

// rr', ss', tt' = (1 / det'(t_K)) adj(K(t_K)) (x0, x1, x2): the weight-free node stage.
template <int K>
__device__ __forceinline__ void tri_node2(const Fibre2& f, double a00, double a11, double x0, double x1,
                                          double x2, double& rr, double& ss, double& tt) {
  const double t = cX<N1>(K);
  const double a01 = fma(fma(f.k01[2], t, f.k01[1]), t, f.k01[0]);
  const double a02 = fma(f.k02[1], t, f.k02[0]);
  const double a12 = fma(f.k12[1], t, f.k12[0]);
  const double g0 = fma(a11, f.k22, -a12 * a12);
  const double g1 = fma(a02, a12, -a01 * f.k22);
  const double g2 = fma(a01, a12, -a02 * a11);
  const double g3 = fma(a00, f.k22, -a02 * a02);
  const double g4 = fma(a01, a02, -a00 * a12);
  const double g5 = fma(a00, a11, -a01 * a01);
  const double dt = fma(fma(f.det[2], t, f.det[1]), t, f.det[0]);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(dt));
  const double e = fma(-dt, r, 1.0);
  const double lam = fma(fma(e, e, e), r, r);  // 1 / det'   (error ~ e^3)
  const double s0 = lam * x0, s1 = lam * x1, s2 = lam * x2;
  rr = fma(g0, s0, fma(g1, s1, g2 * s2));
  ss = fma(g1, s0, fma(g3, s1, g4 * s2));
  tt = fma(g2, s0, fma(g4, s1, g5 * s2));
}

template <int WPB, int MINB>
__global__ void __launch_bounds__(32 * WPB, MINB) ax8m(const __grid_constant__ hx_axlocal_args a) {
  __shared__ ElemGeo s_g[WPB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * WPB + w;
  if (e >= a.n_elements) return;  // no block-wide barrier below
  const int g = lane >> 2, q = lane & 3;
  ElemGeo& S = s_g[w];

  if (lane == 0) {
    const int64_t ahead = e + (int64_t)148 * WPB * MINB * HX_MMA_AHEAD_WAVES4 / 4;
    if (ahead < a.n_elements) {
      bulk_prefetch_l2(a.x + ahead * N3, 4096u);
      bulk_prefetch_l2(a.verts + ahead * 24, 192u);
    }
  }
  const double* xe = a.x + e * N3;
  double xa[8], xb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(xe + k * 64 + g * 8 + 2 * q));
    xa[k] = v.x;
    xb[k] = v.y;
  }
  double Dr[2], Ds[2], Dt[2], Dy[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    Dr[s] = g_D8[g * 8 + 2 * q + s];
    Ds[s] = g_D8[g * 8 + q + 4 * s];
    Dt[s] = g_D8[(2 * q + s) * 8 + g];
    Dy[s] = g_D8[(q + 4 * s) * 8 + g];
  }
  const double* vg = a.verts + e * 24;
  stage_a2(lane, vg, S);
  stage_a2(lane + 32, vg, S);
  stage_a2(lane + 64, vg, S);
  __syncwarp();
  double br[3], sr[3], U[3], V[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    br[c] = S.jb[g][c];
    sr[c] = S.jb[g][3 + c];
    U[c] = S.uv[g][c];
    V[c] = S.uv[g][3 + c];
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int kk = 2 * q + h;
    const double tk = S.xs[kk];
    double cr[3], cs[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      cr[c] = fma(tk, sr[c], br[c]);
      cs[c] = fma(tk, S.ib[g][3 + c], S.ib[g][c]);
    }
    S.t00[kk][g] = fast::dot3(cr, cr);
    S.t11[kk][g] = fast::dot3(cs, cs);
  }
  const double aj = 8.0 * S.iw[g];
  Fibre2 f0, f1;
  prepare_fibre2(S, br, sr, U, V, aj, 2 * q, f0);
  prepare_fibre2(S, br, sr, U, V, aj, 2 * q + 1, f1);
  __syncwarp();

  double ta[8], tb[8];
  fast::eo8<0>(xa, ta);
  fast::eo8<0>(xb, tb);

#define HX_SLICE(K)                                                                                \
  {                                                                                                \
    double r0, r1, s0, s1;                                                                         \
    dmma(r0, r1, xa[K], Dr[0], 0.0, 0.0);                                                          \
    dmma(r0, r1, xb[K], Dr[1], r0, r1);                                                            \
    const double bx0 = __ldg(xe + K * 64 + q * 8 + g), bx1 = __ldg(xe + K * 64 + (q + 4) * 8 + g); \
    dmma(s0, s1, Ds[0], bx0, 0.0, 0.0);                                                            \
    dmma(s0, s1, Ds[1], bx1, s0, s1);                                                              \
    const double a00 = S.t00[K][g];                                                                \
    const double2 a11 = *reinterpret_cast<const double2*>(&S.t11[K][2 * q]);                       \
    double rr0, ss0, rr1, ss1;                                                                     \
    tri_node2<K>(f0, a00, a11.x, r0, s0, ta[K], rr0, ss0, ta[K]);                                  \
    tri_node2<K>(f1, a00, a11.y, r1, s1, tb[K], rr1, ss1, tb[K]);                                  \
    double* tl = S.tile[K & 1];                                                                    \
    *reinterpret_cast<double2*>(tl + g * 8 + 2 * q) = make_double2(ss0, ss1);                      \
    __syncwarp();                                                                                  \
    double y0, y1;                                                                                 \
    dmma(y0, y1, rr0, Dt[0], 0.0, 0.0);                                                            \
    dmma(y0, y1, rr1, Dt[1], y0, y1);                                                              \
    dmma(y0, y1, Dy[0], tl[q * 8 + g], y0, y1);                                                    \
    dmma(y0, y1, Dy[1], tl[(q + 4) * 8 + g], y0, y1);                                              \
    xa[K] = y0;                                                                                    \
    xb[K] = y1;                                                                                    \
  }
  HX_SLICE(0) HX_SLICE(1) HX_SLICE(2) HX_SLICE(3) HX_SLICE(4) HX_SLICE(5) HX_SLICE(6) HX_SLICE(7)
#undef HX_SLICE

  double ya[8], yb[8];
  eo8w(ta, ya);
  eo8w(tb, yb);
  double* ye = a.y + e * N3;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double wk = cW<N1>(k);
    *reinterpret_cast<double2*>(ye + k * 64 + g * 8 + 2 * q) =
        make_double2(fma(wk, xa[k], ya[k]), fma(wk, xb[k], yb[k]));
  }
}

template <int WPB, int MINB, int V = 2>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  const int64_t blocks = (a.n_elements + WPB - 1) / WPB;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  if (V == 1)
    ax8m_v1<WPB, MINB><<<(unsigned)blocks, 32 * WPB, 0, s>>>(a);
  else
    ax8m<WPB, MINB><<<(unsigned)blocks, 32 * WPB, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace mma
}  // namespace hx

// Trilinear Poisson, n_col = 1, element-local x (no fused gather); 16-byte
// aligned x / y.  Returns cudaErrorNotSupported for anything else.
extern "C" cudaError_t hx_mma_launch(const hx_axlocal_args* a, cudaStream_t s) {
  using namespace hx::mma;
  if (a->order != 7 || a->n_col != 1 || a->gather || a->equation != HX_POISSON ||
      a->factor_source != HX_TRILINEAR)
    return cudaErrorNotSupported;
  if (((reinterpret_cast<uintptr_t>(a->x) | reinterpret_cast<uintptr_t>(a->y)) & 15u) != 0)
    return cudaErrorNotSupported;
  switch (a->reserved) {
    case 41: return launch<1, 12>(*a, s);
    case 42: return launch<2, 8>(*a, s);
    case 43: return launch<4, 3>(*a, s);
    case 44: return launch<4, 4>(*a, s);
    case 45: return launch<1, 12, 1>(*a, s);
    case 46: return launch<2, 6>(*a, s);
    default: return launch<1, 12>(*a, s);
  }
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
  if (err == cudaSuccess) err = cudaMemcpyToSymbol(hx::mma::c_IW, iw, sizeof(iw));
  if (err != cudaSuccess) return err;
  return cudaMemcpyToSymbol(g_D8, d, 64 * sizeof(double));
}
