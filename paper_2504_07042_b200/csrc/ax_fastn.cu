// Order-generic fast AxLocal kernel (compiled once per n1 with -DHX_N1=n1).
//
// The design of the N=7 kernel (ax_fast.cu) for every order: thread t of an
// element owns a k-fibre, an i-row and a j-column; even-odd contractions
// (odd n1 has a middle node whose D column / row enter separately); the
// trilinear factors as polynomials in t along each k-fibre with K00(j,k) and
// K11(i,k) in shared tables; factors once per node.  Small elements (n1^2
// threads) are packed several to a CTA so that warps are (nearly) full.
// Shared cubes use padded strides (PJ, PK) chosen per order by an offline
// search over the three access patterns (tools/cube_layout_search.py); where
// tools/role_search.py finds one, a layout whose i-row / j-column tasks are
// dealt to threads by a table so that every 64-bit shared access is
// conflict-free (fastn_roles.cuh; any thread may run any element's row or
// column, they only touch shared memory between barriers).  n_col = 3 runs each
// column in its own CTA with the factors recomputed (identical per-column
// arithmetic, so n_col=3 == 3 x n_col=1 bitwise).
#include "hx_common.cuh"

#ifndef HX_N1
#error "compile with -DHX_N1=<points per direction>"
#endif
#include "fastn_roles.cuh"

namespace hx {
namespace fastn {
namespace {  // internal linkage: every order is its own TU with the same template names

constexpr int N1 = HX_N1;
constexpr int N3 = N1 * N1 * N1;
constexpr int H = N1 / 2;
constexpr bool ODD = N1 & 1;
constexpr int T = N1 * N1;                    // threads per element
// elements per CTA: fill whole warps (lanes of a partial warp idle through every phase)
constexpr int epb_of(int n) {
  return n == 2 ? 16 : n == 3 ? 7 : n == 4 ? 4 : n == 5 ? 5 : n == 6 ? 3 : n == 7 ? 5 : 1;
}
#ifdef HX_FASTN_EPB
constexpr int EPB = HX_FASTN_EPB;
#else
constexpr int EPB = epb_of(N1);
#endif

constexpr int pj_of(int n) {
  return n == 6 ? 9 : n == 8 ? 9 : n == 10 ? 17 : n == 12 ? 13 : n == 14 ? 17 : n == 16 ? 17 : n;
}
constexpr int pk_of(int n) {
  return n == 2 ? 5 : n == 3 ? 18 : n == 4 ? 19 : n == 6 ? 54 : n == 7 ? 52 : n == 8 ? 72 : n == 10 ? 170
       : n == 12 ? 156 : n == 14 ? 238 : n == 16 ? 272 : n * n;
}
template <bool R>  // R: the role-table layout (fastn_roles.cuh)
struct Strides {
  static constexpr int PJ = R ? kRolePJ : pj_of(N1);
  static constexpr int PK = R ? kRolePK : pk_of(N1);
  static constexpr int CUBE = (N1 - 1) * PK + (N1 - 1) * PJ + N1;
};
// stride between the cubes of the elements packed in one CTA (tools/cube_layout_search.py:
// PJ, PK and this stride minimise the weighted shared wavefronts of the three fibre
// patterns over every warp of the CTA; warps straddle elements when n1^2 is not a
// multiple of 32)
constexpr int cs_of(int n) { return n == 2 ? 12 : n == 3 ? 57 : n == 5 ? 137 : n == 6 ? 324 : n == 7 ? 369 : 0; }
template <bool R>
constexpr int cs_for() {
  return cs_of(N1) > Strides<false>::CUBE ? cs_of(N1) : Strides<false>::CUBE;
}

constexpr int EO = 2 * H * H + 2 * H + 1;  // A[H][H], B[H][H], C[H], R[H], M[mid][mid]

}  // namespace
}  // namespace fastn
}  // namespace hx

// even-odd blocks of D (T=0) and D^T (T=1) for this order, in three identical
// copies (one per contraction direction): with a single copy NVVM CSEs the
// constant loads of the three back-to-back contractions into registers, which
// costs 2 x 2H^2 registers and spills for n1 >= 9.  At n1 = 16 three copies
// (7 KB) no longer fit the per-SM constant cache next to the basis tables and
// one copy measures faster (profiles/r01_order_sweep.txt).
namespace hx {
namespace fastn {
namespace {
constexpr int kCopies = N1 >= 16 ? 1 : 3;
}
}  // namespace fastn
}  // namespace hx
static __constant__ double c_EOn[hx::fastn::kCopies][2][hx::fastn::EO];

namespace hx {
namespace fastn {
namespace {  // internal linkage: every order is its own TU with the same template names

// out = M v, M = D (TR=0) or D^T (TR=1), centro-antisymmetric on GLL points.
template <int TR, int COPY>
__device__ __forceinline__ void eon(const double v[N1], double out[N1]) {
  const double* A = c_EOn[COPY % kCopies][TR];
  const double* B = c_EOn[COPY % kCopies][TR] + H * H;
  const double* C = c_EOn[COPY % kCopies][TR] + 2 * H * H;
  const double* R = c_EOn[COPY % kCopies][TR] + 2 * H * H + H;
  double ue[H > 0 ? H : 1], uo[H > 0 ? H : 1];
#pragma unroll
  for (int m = 0; m < H; ++m) {
    ue[m] = v[m] + v[N1 - 1 - m];
    uo[m] = v[m] - v[N1 - 1 - m];
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double p = A[i * H] * ue[0];
    double q = B[i * H] * uo[0];
#pragma unroll
    for (int m = 1; m < H; ++m) {
      p = fma(A[i * H + m], ue[m], p);
      q = fma(B[i * H + m], uo[m], q);
    }
    if (ODD) p = fma(C[i], v[H], p);
    out[i] = p + q;
    out[N1 - 1 - i] = q - p;
  }
  if (ODD) {
    double s = c_EOn[COPY % kCopies][TR][2 * H * H + 2 * H] * v[H];
#pragma unroll
    for (int m = 0; m < H; ++m) s = fma(R[m], uo[m], s);
    out[H] = s;
  }
}

__device__ __forceinline__ double dot3(const double* u, const double* v) {
  return u[0] * v[0] + u[1] * v[1] + u[2] * v[2];
}

__device__ __forceinline__ double div_fast(double w, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  const double wr = w * r;
  return fma(fma(e, e, e), wr, wr);
}

struct TriShared {
  double j[N1][6];
  double i[N1][6];
  double d[12];
  double t00[N1][N1 + 1];
  double t11[N1][N1 + 1];
  double xs[N1];
  double ws[N1];
};

// common_terms (geometry.py:135-184) as independent tasks over the element's threads
__device__ __forceinline__ void stage_a(int t, const double* __restrict__ v, TriShared& s) {
  constexpr int TASKS = 6 * N1 + 12 + N1;
  for (int task = t; task < TASKS; task += T) {
    if (task < 6 * N1) {
      const bool jside = task < 3 * N1;
      const int q = jside ? task : task - 3 * N1;
      const int idx = q / 3, c = q % 3;
      const double xi = c_X[off_p(N1) + idx];
      const double a0 = 1.0 - xi, a1 = 1.0 + xi;
      const int p0 = jside ? 1 : 2, q1 = jside ? 2 : 1, p2 = jside ? 5 : 6, q3 = jside ? 6 : 5;
      const double lo = a0 * (v[p0 * 3 + c] - v[c]) + a1 * (v[9 + c] - v[q1 * 3 + c]);
      const double hi = a0 * (v[p2 * 3 + c] - v[12 + c]) + a1 * (v[21 + c] - v[q3 * 3 + c]);
      double* out = jside ? s.j[idx] : s.i[idx];
      out[c] = lo + hi;
      out[3 + c] = hi - lo;
    } else if (task < 6 * N1 + 12) {
      const int q = task - 6 * N1, pair = q / 3, c = q % 3;
      const int pa = pair == 0 ? 4 : pair == 1 ? 5 : pair == 2 ? 7 : 6;
      const int pb = pair == 0 ? 0 : pair == 1 ? 1 : pair == 2 ? 3 : 2;
      s.d[q] = v[pa * 3 + c] - v[pb * 3 + c];
    } else {
      const int q = task - 6 * N1 - 12;
      s.xs[q] = c_X[off_p(N1) + q];
      s.ws[q] = c_W[off_p(N1) + q];
    }
  }
}

template <bool HELM, bool MERGED, bool PARTIAL>
struct TriPoly {
  // K00(j,k) / K11(i,k) from shared tables (one entry per thread) or as quadratics in
  // t per fibre: the tables cost shared bandwidth, the quadratics FP64.  Measured per
  // order (HX_FASTN_NOTAB builds): quadratics win at n1 = 4, 11, 14 (+3 / +4 / +11 %),
  // tables elsewhere or within noise.
#ifdef HX_FASTN_NOTAB
  static constexpr bool kTab = false;
#else
  static constexpr bool kTab = !(N1 == 4 || N1 == 11 || N1 == 14);
#endif
  static constexpr bool kTri = true;
  static constexpr bool kPpd = false;
  static constexpr bool kHelm = HELM;
  static constexpr bool kMerged = MERGED;
  static constexpr bool kPartial = PARTIAL;
  double k01[3], k02[2], k12[2], k22, det[3];
  double k00[3], k11[3];  // K00 / K11 along the fibre when not tabulated (kTab false)
  double wji8;
  const double* tab00;
  const double* tab11;
  const double* lam_a;
  const double* lam_b;
  double l0v, l1v;

  // per-fibre coefficients; also this thread's K00(j=fj,k=fi) and K11(i=fi,k=fj) table entries
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, int64_t e, TriShared& s, int fi, int fj) {
    double br[3], sr[3], bs[3], ss[3], c[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      br[q] = s.j[fj][q];
      sr[q] = s.j[fj][3 + q];
      bs[q] = s.i[fi][q];
      ss[q] = s.i[fi][3 + q];
    }
    tab00 = s.t00[fj];
    tab11 = s.t11[fi];
    if (kTab) {
      const double tk = s.xs[fi], tj = s.xs[fj];
      double cr[3], cs[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        cr[q] = br[q] + tk * sr[q];
        cs[q] = bs[q] + tj * ss[q];
      }
      s.t00[fj][fi] = dot3(cr, cr);
      s.t11[fi][fj] = dot3(cs, cs);
    } else {
      k00[0] = dot3(br, br);
      k00[1] = 2.0 * dot3(br, sr);
      k00[2] = dot3(sr, sr);
      k11[0] = dot3(bs, bs);
      k11[1] = 2.0 * dot3(bs, ss);
      k11[2] = dot3(ss, ss);
    }
    const double xj = s.xs[fj], xi = s.xs[fi];
    const double a0j = 1.0 - xj, a1j = 1.0 + xj, a0i = 1.0 - xi, a1i = 1.0 + xi;
    const double w00 = a0j * a0i, w01 = a0j * a1i, w10 = a1j * a0i, w11 = a1j * a1i;
#pragma unroll
    for (int q = 0; q < 3; ++q) c[q] = w00 * s.d[q] + w01 * s.d[3 + q] + w11 * s.d[6 + q] + w10 * s.d[9 + q];
    k01[0] = dot3(br, bs);
    k01[1] = dot3(br, ss) + dot3(sr, bs);
    k01[2] = dot3(sr, ss);
    k02[0] = dot3(br, c);
    k02[1] = dot3(sr, c);
    k12[0] = dot3(bs, c);
    k12[1] = dot3(ss, c);
    k22 = dot3(c, c);
    const double P[3] = {bs[1] * c[2] - bs[2] * c[1], bs[2] * c[0] - bs[0] * c[2], bs[0] * c[1] - bs[1] * c[0]};
    const double Q[3] = {ss[1] * c[2] - ss[2] * c[1], ss[2] * c[0] - ss[0] * c[2], ss[0] * c[1] - ss[1] * c[0]};
    det[0] = dot3(br, P);
    det[1] = dot3(br, Q) + dot3(sr, P);
    det[2] = dot3(sr, Q);
    wji8 = 0.125 * (s.ws[fj] * s.ws[fi]);
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
  __device__ __forceinline__ void node(int n, double x0, double x1, double x2, double& rr, double& ss, double& tt,
                                       double& mass) const {
    const double t = cX<N1>(K);
    const double a00 = kTab ? tab00[K] : fma(fma(k00[2], t, k00[1]), t, k00[0]);
    const double a11 = kTab ? tab11[K] : fma(fma(k11[2], t, k11[1]), t, k11[0]);
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
      scale = __ldg(lam_a + n);
      mass = __ldg(lam_b + n);
    } else if (PARTIAL) {
      scale = __ldg(lam_a + n);
    } else {
      const double dt = fma(fma(det[2], t, det[1]), t, det[0]);
      const double lam_geo = div_fast(cW<N1>(K) * wji8, dt);
      if (HELM) {
        const double l0 = lam_a ? __ldg(lam_a + n) : l0v;
        const double l1 = lam_b ? __ldg(lam_b + n) : l1v;
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

template <bool HELM>
struct StoredN {
  static constexpr bool kTri = false;
  static constexpr bool kPpd = false;
  static constexpr bool kHelm = HELM;
  const double* g;
  const double* gwj;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, int64_t e, TriShared&, int, int) {
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

template <bool HELM>
struct PpdN {
  static constexpr bool kTri = false;
  static constexpr bool kPpd = true;
  static constexpr bool kHelm = HELM;
  double h[7];
  double wj, wi;
  const double* lam0;
  const double* lam1;
  double l0v, l1v;
  __device__ __forceinline__ void prepare(const hx_axlocal_args& a, int64_t e, TriShared&, int fi, int fj) {
#pragma unroll
    for (int q = 0; q < 7; ++q) h[q] = __ldg(a.h + e * 7 + q);
    wj = c_W[off_p(N1) + fj];
    wi = c_W[off_p(N1) + fi];
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

// compile-time loop over nodes K = 0..N1-1
template <int K, int END, int PK>
struct NodeLoop {
  template <typename F>
  __device__ __forceinline__ static void run(const F& fac, double* sA, double* sB, int kp, int lin,
                                             const double* x2, const double* xk, double* tt, double* yk) {
    const int adr = K * PK + kp;
    double rr, ss, mass;
    fac.template node<K>(K * N1 * N1 + lin, sA[adr], sB[adr], x2[K], rr, ss, tt[K], mass);
    sA[adr] = rr;
    sB[adr] = ss;
    yk[K] = mass * xk[K];
    NodeLoop<K + 1, END, PK>::run(fac, sA, sB, kp, lin, x2, xk, tt, yk);
  }
};
template <int END, int PK>
struct NodeLoop<END, END, PK> {
  template <typename F>
  __device__ __forceinline__ static void run(const F&, double*, double*, int, int, const double*, const double*,
                                             double*, double*) {}
};

// Packing of elements into a CTA.  The default (EPB, searched cube stride) is per
// order; a source may pack fewer elements (Pack<1 or 2 ...>, unpadded stride).
template <int EPB_, bool R = false>
struct Pack {
  static constexpr int kEpb = EPB_;
  // role table (fastn_roles.cuh) for this packing: whole warps, the lanes past the
  // k-fibre threads take row / column tasks
  static constexpr bool kRoles = HX_ROLES && R && EPB_ == kRoleEPB;
  using S = Strides<kRoles>;
  static constexpr int kFibres = T * EPB_;  // k-fibre threads
  static constexpr int kThreads = kRoles ? (kFibres + 31) / 32 * 32 : kFibres;
  static constexpr int kWarps = (kThreads + 31) / 32;
  static constexpr int kStride = kRoles ? kRoleCS : EPB_ == EPB ? cs_for<false>() : S::CUBE;
  // dynamic shared memory: [X | A | B] cubes per element, then TriShared, then vertices
  static constexpr size_t kSmem =
      sizeof(double) * 3 * EPB_ * kStride + sizeof(TriShared) * EPB_ + sizeof(double) * 24 * EPB_;
};

// natural layout: thread (fi, fj) of element le runs its own k-fibre, i-row
// (j = fi, k = fj) and j-column (i = fi, k = fj)
template <typename F, int NCOL, bool HELM, int MINB, int EPB_>
__global__ void __launch_bounds__(Pack<EPB_, false>::kThreads, MINB) axn(const __grid_constant__ hx_axlocal_args a) {
  constexpr int EPB = EPB_;
  constexpr int CS = Pack<EPB_, false>::kStride;
  constexpr int PJ = Strides<false>::PJ, PK = Strides<false>::PK;
  extern __shared__ __align__(16) double smem[];
  double(*sX)[CS] = reinterpret_cast<double(*)[CS]>(smem);
  double(*sA)[CS] = reinterpret_cast<double(*)[CS]>(smem + EPB * CS);
  double(*sB)[CS] = reinterpret_cast<double(*)[CS]>(smem + 2 * EPB * CS);
  TriShared* sT = reinterpret_cast<TriShared*>(smem + 3 * EPB * CS);
  double(*sV)[24] = reinterpret_cast<double(*)[24]>(reinterpret_cast<char*>(sT) + sizeof(TriShared) * EPB);
  const int le = threadIdx.x / T, t = threadIdx.x - le * T;
  // n_col = 3: the three columns of an element group are three adjacent CTAs (same
  // arithmetic per column, x / y rows shared through L2); no column loop, whose
  // loop-invariant constant loads NVVM would hoist into registers
  const int c = NCOL > 1 ? (int)(blockIdx.x % NCOL) : 0;
  const int64_t e_raw = (int64_t)(blockIdx.x / NCOL) * EPB + le;
  const bool valid = e_raw < a.n_elements;
  const int64_t e = valid ? e_raw : a.n_elements - 1;
  const int fi = t % N1, fj = t / N1;   // k-fibre (i, j); i-row (j = fi, k = fj); j-column (i = fi, k = fj)
  const int kp = fj * PJ + fi;
  const int rb = fj * PK + fi * PJ;
  const int cb = fj * PK + fi;
  const int lin = fj * N1 + fi;
  double* X = sX[le];
  double* A = sA[le];
  double* B = sB[le];
  {
    double xk[N1];
    if constexpr (F::kTri && N1 <= 11) {
      // the fibre's x loads go out before the vertex staging barrier (above n1 = 11
      // the n1 registers held across it cost more than they save: merged -2..-5 %)
#pragma unroll
      for (int k = 0; k < N1; ++k) xk[k] = __ldg(a.x + (e * N3 + k * N1 * N1 + lin) * NCOL + c);
      for (int q = t; q < 24; q += T) sV[le][q] = __ldg(a.verts + e * 24 + q);
      __syncthreads();
    } else {
      if (F::kTri) {
        for (int q = t; q < 24; q += T) sV[le][q] = __ldg(a.verts + e * 24 + q);
        __syncthreads();
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) xk[k] = __ldg(a.x + (e * N3 + k * N1 * N1 + lin) * NCOL + c);
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) X[k * PK + kp] = xk[k];
    if (F::kTri) stage_a(t, sV[le], sT[F::kTri ? le : 0]);
    __syncthreads();

    F fac;
    fac.prepare(a, e, sT[F::kTri ? le : 0], fi, fj);
    double x2[N1];
    eon<0, 0>(xk, x2);
    {
      double v[N1], o[N1];
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = X[rb + n];
      eon<0, 1>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) A[rb + n] = o[n];
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = X[cb + n * PJ];
      eon<0, 2>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) B[cb + n * PJ] = o[n];
    }
    __syncthreads();  // also publishes this element's K00/K11 tables

    double tt[N1], yk[N1];
    NodeLoop<0, N1, PK>::run(fac, A, B, kp, lin, x2, xk, tt, yk);
    double yt[N1];
    eon<1, 0>(tt, yt);
    __syncthreads();
    {
      double v[N1], o[N1];
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = A[rb + n];
      eon<1, 1>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) A[rb + n] = o[n];
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = B[cb + n * PJ];
      eon<1, 2>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) B[cb + n * PJ] = o[n];
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const int adr = k * PK + kp;
        double y = (A[adr] + B[adr]) + yt[k];
        if (HELM) y += yk[k];
        a.y[(e * N3 + k * N1 * N1 + lin) * NCOL + c] = y;
      }
    }
  }
}

// role-table layout (fastn_roles.cuh): whole warps; row / column tasks from the table
template <typename F, int NCOL, bool HELM, int MINB, int EPB_>
__global__ void __launch_bounds__(Pack<EPB_, true>::kThreads, MINB) axn_r(const __grid_constant__ hx_axlocal_args a) {
  using P = Pack<EPB_, true>;
  static_assert(P::kRoles, "role-table kernel without a table");
  constexpr int PJ = P::S::PJ, PK = P::S::PK;
  constexpr int EPB = EPB_;
  constexpr int CS = P::kStride;
  extern __shared__ __align__(16) double smem[];
  double(*sX)[CS] = reinterpret_cast<double(*)[CS]>(smem);
  double(*sA)[CS] = reinterpret_cast<double(*)[CS]>(smem + EPB * CS);
  double(*sB)[CS] = reinterpret_cast<double(*)[CS]>(smem + 2 * EPB * CS);
  TriShared* sT = reinterpret_cast<TriShared*>(smem + 3 * EPB * CS);
  double(*sV)[24] = reinterpret_cast<double(*)[24]>(reinterpret_cast<char*>(sT) + sizeof(TriShared) * EPB);
  // k-fibre threads own (element le, fibre t); padding lanes (role tables only) skip
  // every k-fibre phase and run only their row / column tasks
  const bool kact = P::kThreads == P::kFibres || (int)threadIdx.x < P::kFibres;
  const int le = kact ? (int)threadIdx.x / T : EPB - 1, t = kact ? (int)threadIdx.x - le * T : 0;
  // n_col = 3: the three columns of an element group are three adjacent CTAs (same
  // arithmetic per column, x / y rows shared through L2); no column loop, whose
  // loop-invariant constant loads NVVM would hoist into registers
  const int c = NCOL > 1 ? (int)(blockIdx.x % NCOL) : 0;
  const int64_t e_raw = (int64_t)(blockIdx.x / NCOL) * EPB + le;
  const bool valid = kact && e_raw < a.n_elements;
  const int64_t e = e_raw < a.n_elements ? e_raw : a.n_elements - 1;
  const int fi = t % N1, fj = t / N1;   // k-fibre (i, j); i-row (j = fi, k = fj); j-column (i = fi, k = fj)
  const int kp = fj * PJ + fi;
  const int lin = fj * N1 + fi;
  double* A = sA[le];
  double* B = sB[le];
  double* X = sX[le];
  // i-row / j-column tasks: with a role table any thread may run the row / column of
  // any element of the CTA, placed so that every half-warp's 16 bases are distinct
  // modulo 16 bank pairs (0xffff: no task); else the thread's own (j = fi, k = fj)
  // row and (i = fi, k = fj) column
  double* const X0 = sX[0];
  double* const A0 = sA[0];
  double* const B0 = sB[0];
  int rbA = le * CS + fj * PK + fi * PJ, cbA = le * CS + fj * PK + fi;
#if HX_ROLES
  if constexpr (P::kRoles) {
    const unsigned r = __ldg(c_roles + threadIdx.x);
    rbA = (r & 0xffffu) == 0xffffu ? -1 : (int)(r & 0xffffu);
    cbA = (r >> 16) == 0xffffu ? -1 : (int)(r >> 16);
  }
#endif
  const bool row_task = !P::kRoles || rbA >= 0;
  const bool col_task = !P::kRoles || cbA >= 0;
  // the fibre's x loads go out before the vertex staging barrier (one global latency
  // per CTA instead of two back to back)
  double xk[N1];
  if (kact) {
#pragma unroll
    for (int k = 0; k < N1; ++k) xk[k] = __ldg(a.x + (e * N3 + k * N1 * N1 + lin) * NCOL + c);
  }
  if (F::kTri) {
    if (kact)
      for (int q = t; q < 24; q += T) sV[le][q] = __ldg(a.verts + e * 24 + q);
    __syncthreads();
  }

  if (kact) {
#pragma unroll
    for (int k = 0; k < N1; ++k) X[k * PK + kp] = xk[k];
    if (F::kTri) stage_a(t, sV[le], sT[F::kTri ? le : 0]);
  }
  __syncthreads();

  F fac;
  double x2[N1];
  if (kact) {
    fac.prepare(a, e, sT[F::kTri ? le : 0], fi, fj);
    eon<0, 0>(xk, x2);
  }
  {
    double v[N1], o[N1];
    if (row_task) {
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = X0[rbA + n];
      eon<0, 1>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) A0[rbA + n] = o[n];
    }
    if (col_task) {
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = X0[cbA + n * PJ];
      eon<0, 2>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) B0[cbA + n * PJ] = o[n];
    }
  }
  __syncthreads();  // also publishes this element's K00/K11 tables

  double tt[N1], yk[N1], yt[N1];
  if (kact) {
    NodeLoop<0, N1, PK>::run(fac, A, B, kp, lin, x2, xk, tt, yk);
    eon<1, 0>(tt, yt);
  }
  __syncthreads();
  {
    double v[N1], o[N1];
    if (row_task) {
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = A0[rbA + n];
      eon<1, 1>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) A0[rbA + n] = o[n];
    }
    if (col_task) {
#pragma unroll
      for (int n = 0; n < N1; ++n) v[n] = B0[cbA + n * PJ];
      eon<1, 2>(v, o);
#pragma unroll
      for (int n = 0; n < N1; ++n) B0[cbA + n * PJ] = o[n];
    }
  }
  __syncthreads();
  if (valid) {
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int adr = k * PK + kp;
      double y = (A[adr] + B[adr]) + yt[k];
      if (HELM) y += yk[k];
      a.y[(e * N3 + k * N1 * N1 + lin) * NCOL + c] = y;
    }
  }
}

// register budget per thread -> CTAs per SM the compiler must fit (launch bounds);
// the per-thread fibre state grows with n1 (~4 n1 doubles live plus the factors)
// (two CTAs per SM up to n1 = 15; 16 keeps one copy of the D blocks and needs 255)
#ifdef HX_FASTN_REGS
constexpr int kRegs = HX_FASTN_REGS;
#else
constexpr int regs_of(int n) { return n <= 12 ? 128 : n <= 13 ? 168 : n <= 15 ? 128 : 255; }
constexpr int kRegs = regs_of(N1);
#endif
// trilinear sources at n1 <= 7 run best with 80 registers (96 for Helmholtz, which
// would spill; more CTAs hide the per-element setup: +5-15 % at N = 3-6), and so
// does the Poisson parallelepiped kernel at n1 = 10-13; stored keeps the budget
template <typename F>
constexpr int regs_for() {
#ifdef HX_FASTN_REGS
  return kRegs;
#else
  // measured per order with tools/build_variant.sh libraries at 80 / 96 / 128 / 168
  // registers (profiles/r01_register_budgets.txt); Poisson trilinear and parallelepiped:
  if (F::kTri && N1 <= 7) return F::kHelm ? 96 : 80;
  if (F::kTri && !F::kHelm && (N1 == 12 || N1 == 13)) return 96;  // +9 % at N = 11, 12
  if (F::kPpd && !F::kHelm && (N1 == 7 || (N1 >= 10 && N1 <= 12))) return 80;
  if (F::kPpd && !F::kHelm && N1 == 13) return 96;
  if (F::kPpd && !F::kHelm && N1 == 14) return 168;
  return kRegs;
#endif
}
// role-table layout per (source, n_col), measured against the natural layout with
// A/B libraries (profiles/r01_roles_ab.txt): Poisson parallelepiped +3-32 % at every
// order, Poisson trilinear up to +10 % (not n1 = 13, 15: -1 / -9 %; partial there
// +6 / +11 %), Poisson stored
// (HBM-bound) from n1 = 10; Helmholtz per source at the orders where it gained
// (+2-39 %; elsewhere it lost up to 11 %); merged only at n1 = 16; at n1 = 6
// trilinear n_col = 3 loses 2-8 %
template <typename F, int NCOL>
constexpr bool roles_for() {
  bool r = F::kPpd || N1 >= 10 || N1 == 4;  // Poisson
  if constexpr (F::kTri) r = F::kPartial || !(N1 == 15 || (N1 == 13 && NCOL == 1));
  if (F::kHelm) {
    if (F::kPpd)
      r = N1 == 4 || N1 == 5 || N1 == 9 || N1 == 10 || N1 == 16;
    else if (F::kTri)
      r = N1 == 5 || N1 == 7 || N1 == 9 || N1 == 10 || N1 == 14 || N1 == 16;
    else
      r = N1 == 5 || N1 == 7 || N1 == 9 || N1 == 16;
  }
  if constexpr (F::kTri) r = r && (!F::kMerged || N1 == 16);
  if (N1 == 6) r = r && (F::kPpd || NCOL == 1);
  return HX_ROLES && r;
}

// elements per CTA: the stored source streams six factor fields per node and prefers
// smaller CTAs at n1 = 5 and 7 (+3 / +7 %, A/B libraries with -DHX_FASTN_EPB)
template <typename F, int NCOL>
constexpr int epb_for() {
#ifdef HX_FASTN_EPB
  return EPB;
#else
  if (roles_for<F, NCOL>()) return kRoleEPB;  // the packing the role table was generated for
  return (!F::kTri && !F::kPpd) ? (N1 == 5 ? 3 : N1 == 7 ? 2 : EPB) : EPB;
#endif
}

template <typename F, int NCOL>
using PackFor = Pack<epb_for<F, NCOL>(), roles_for<F, NCOL>()>;

template <typename F, int NCOL>
constexpr int minb_for() {
  constexpr int w = PackFor<F, NCOL>::kWarps;
  return 65536 / (w * 32 * regs_for<F>()) > 0 ? 65536 / (w * 32 * regs_for<F>()) : 1;
}

template <typename F, int NCOL, bool HELM>
cudaError_t launch_ncol(const hx_axlocal_args& a, cudaStream_t s) {
  using P = PackFor<F, NCOL>;
  const int64_t blocks = (a.n_elements + P::kEpb - 1) / P::kEpb * NCOL;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  static_assert(P::kSmem <= 227 * 1024, "shared memory");
  constexpr auto k = [] {
    if constexpr (roles_for<F, NCOL>())
      return axn_r<F, NCOL, HELM, minb_for<F, NCOL>(), P::kEpb>;
    else
      return axn<F, NCOL, HELM, minb_for<F, NCOL>(), P::kEpb>;
  }();
  if (P::kSmem > 48 * 1024) {  // once per device: the attribute lives in each device's module
    static unsigned long long done = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(done & bit)) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::kSmem);
      if (e != cudaSuccess) return e;
      done |= bit;
    }
  }
  k<<<(unsigned)blocks, P::kThreads, P::kSmem, s>>>(a);
  return cudaGetLastError();
}

template <typename F, bool HELM>
cudaError_t launch(const hx_axlocal_args& a, cudaStream_t s) {
  return a.n_col == 3 ? launch_ncol<F, 3, HELM>(a, s) : launch_ncol<F, 1, HELM>(a, s);
}

}  // namespace
}  // namespace fastn
}  // namespace hx

#define HX_CAT2(a, b) a##b
#define HX_CAT(a, b) HX_CAT2(a, b)

extern "C" cudaError_t HX_CAT(hx_fastn_launch_, HX_N1)(const hx_axlocal_args* a, cudaStream_t s) {
  using namespace hx::fastn;
  const bool helm = a->equation == HX_HELMHOLTZ;
  switch (a->factor_source) {
    case HX_TRILINEAR:
      return helm ? launch<TriPoly<true, false, false>, true>(*a, s) : launch<TriPoly<false, false, false>, false>(*a, s);
    case HX_TRILINEAR_PARTIAL:
      return launch<TriPoly<false, false, true>, false>(*a, s);
    case HX_TRILINEAR_MERGED:
      return launch<TriPoly<true, true, false>, true>(*a, s);
    case HX_STORED:
      return helm ? launch<StoredN<true>, true>(*a, s) : launch<StoredN<false>, false>(*a, s);
    case HX_PARALLELEPIPED:
      return helm ? launch<PpdN<true>, true>(*a, s) : launch<PpdN<false>, false>(*a, s);
  }
  return cudaErrorNotSupported;
}

// basis upload: common constants plus this order's even-odd blocks
extern "C" cudaError_t HX_CAT(hx_upload_basis_fastn_, HX_N1)(int n1, const double* pts, const double* w,
                                                             const double* d) {
  using namespace hx::fastn;
  cudaError_t err = hx_upload_basis_local(n1, pts, w, d);
  if (err != cudaSuccess || n1 != N1) return err;
  double eo[kCopies][2][EO];
  for (int tr = 0; tr < 2; ++tr) {
    auto M = [&](int i, int j) { return tr ? d[j * N1 + i] : d[i * N1 + j]; };
    for (int i = 0; i < H; ++i)
      for (int m = 0; m < H; ++m) {
        eo[0][tr][i * H + m] = 0.5 * (M(i, m) + M(i, N1 - 1 - m));
        eo[0][tr][H * H + i * H + m] = 0.5 * (M(i, m) - M(i, N1 - 1 - m));
      }
    for (int i = 0; i < H; ++i) {
      eo[0][tr][2 * H * H + i] = ODD ? M(i, H) : 0.0;
      eo[0][tr][2 * H * H + H + i] = ODD ? M(H, i) : 0.0;
    }
    eo[0][tr][2 * H * H + 2 * H] = ODD ? M(H, H) : 0.0;
  }
  for (int copy = 1; copy < kCopies; ++copy) memcpy(eo[copy], eo[0], sizeof(eo[0]));
  return cudaMemcpyToSymbol(c_EOn, eo, sizeof(eo));
}
