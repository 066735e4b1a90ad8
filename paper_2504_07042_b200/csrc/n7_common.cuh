// Pieces shared by the N = 7 (n1 = 8) kernels: the even-odd D blocks in
// __constant__ memory (one static copy per translation unit, uploaded by that
// unit's basis hook through n7_upload_eo), the 8-point even-odd contraction,
// the fast reciprocal, and stage A of the trilinear geometry
// (common_terms, geometry.py:135-184).
#pragma once

#include "hx_common.cuh"

// Even-odd blocks: [0] forward D, [1] transposed D^T; [.][0] = A (even), [.][1] = B (odd);
// A[i][m] = (M[i][m] + M[i][7-m]) / 2, B[i][m] = (M[i][m] - M[i][7-m]) / 2 for M = D or D^T.
// [copy]: two identical copies so that code for the two fibre roles of the
// warp-per-element kernel does not share (and keep live) the same constants.
static __constant__ double c_EO[2][2][2][4][4];

namespace hx {
namespace fast {

constexpr int N1 = 8;
constexpr int N3 = 512;

// Basis value at a thread-dependent index: eight uniform constant loads and a
// select chain instead of a divergent indexed LDC (which serialises per lane).
__device__ __forceinline__ double pick8(const double* c, int idx) {
  double v = c[0];
#pragma unroll
  for (int q = 1; q < 8; ++q) v = idx == q ? c[q] : v;
  return v;
}
__device__ __forceinline__ double xr(int idx) { return pick8(c_X + off_p(N1), idx); }
__device__ __forceinline__ double wr(int idx) { return pick8(c_W + off_p(N1), idx); }

// out = M v for an 8-point fibre, M = D (T=0) or D^T (T=1).
template <int T, int COPY = 0>
__device__ __forceinline__ void eo8(const double v[8], double out[8]) {
  double ue[4], uo[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    ue[m] = v[m] + v[7 - m];
    uo[m] = v[m] - v[7 - m];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double p = c_EO[COPY][T][0][i][0] * ue[0];
    double q = c_EO[COPY][T][1][i][0] * uo[0];
#pragma unroll
    for (int m = 1; m < 4; ++m) {
      p = fma(c_EO[COPY][T][0][i][m], ue[m], p);
      q = fma(c_EO[COPY][T][1][i][m], uo[m], q);
    }
    out[i] = p + q;
    out[7 - i] = q - p;
  }
}

// w / d: MUFU reciprocal seed r, e = 1 - d r, w r (1 + e + e^2)  (error ~ e^3).
__device__ __forceinline__ double div_fast(double w, double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  const double wr = w * r;
  return fma(fma(e, e, e), wr, wr);
}

// Per-element trilinear pieces shared by the 64 fibres (written by 28 threads).
struct TriShared {
  double j[8][6];  // dr_base[3], dr_slope[3] per j
  double i[8][6];  // ds_base[3], ds_slope[3] per i
  double d[12];     // v4-v0, v5-v1, v7-v3, v6-v2
  double t00[8][9];  // K00(j, k): depends on j and k only (padded rows)
  double t11[8][9];  // K11(i, k): depends on i and k only
  double xs[8];      // GLL points and weights, for thread-dependent indices
  double ws[8];
};

__device__ __forceinline__ double dot3(const double* u, const double* v) {
  return u[0] * v[0] + u[1] * v[1] + u[2] * v[2];
}

// Stage A: common_terms (geometry.py:135-184) split into 60 short independent
// tasks (one coordinate of one j-side or i-side base/slope pair, or one vertex
// difference), so no thread runs a long dependent chain while the others wait.
__device__ __forceinline__ void tri_stage_a(int t, const double* __restrict__ v, TriShared& s) {
  if (t < 48) {
    const bool jside = t < 24;
    const int task = jside ? t : t - 24;
    const int idx = task / 3, c = task % 3;
    const double xi = xr(idx);
    const double a0 = 1.0 - xi, a1 = 1.0 + xi;
    // j side: tmp1 = a0 (v1-v0) + a1 (v3-v2), tmp2 = a0 (v5-v4) + a1 (v7-v6)
    // i side: tmp3 = a0 (v2-v0) + a1 (v3-v1), tmp4 = a0 (v6-v4) + a1 (v7-v5)
    const int p0 = jside ? 1 : 2, p1 = 3, q1 = jside ? 2 : 1;
    const int p2 = jside ? 5 : 6, p3 = 7, q3 = jside ? 6 : 5;
    const double lo = a0 * (v[p0 * 3 + c] - v[c]) + a1 * (v[p1 * 3 + c] - v[q1 * 3 + c]);
    const double hi = a0 * (v[p2 * 3 + c] - v[12 + c]) + a1 * (v[p3 * 3 + c] - v[q3 * 3 + c]);
    double* out = jside ? s.j[idx] : s.i[idx];
    out[c] = lo + hi;
    out[3 + c] = hi - lo;
  } else if (t < 60) {
    const int q = t - 48, pair = q / 3, c = q % 3;
    const int pa = pair == 0 ? 4 : pair == 1 ? 5 : pair == 2 ? 7 : 6;
    const int pb = pair == 0 ? 0 : pair == 1 ? 1 : pair == 2 ? 3 : 2;
    s.d[q] = v[pa * 3 + c] - v[pb * 3 + c];
  }
  if (t < 8) {
    s.xs[t] = xr(t);
    s.ws[t] = wr(t);
  }
}


// Even-odd blocks of D (row-major [i][m], n1 = 8) into this unit's c_EO (static:
// internal linkage, so every unit that includes this uploads its own copy).
static inline cudaError_t n7_upload_eo(const double* d) {
  double eo[2][2][2][4][4];
  for (int cp = 0; cp < 2; ++cp)
    for (int T = 0; T < 2; ++T)
      for (int i = 0; i < 4; ++i)
        for (int m = 0; m < 4; ++m) {
          const double x = T ? d[m * 8 + i] : d[i * 8 + m];            // M[i][m]
          const double y = T ? d[(7 - m) * 8 + i] : d[i * 8 + 7 - m];  // M[i][7-m]
          eo[cp][T][0][i][m] = 0.5 * (x + y);
          eo[cp][T][1][i][m] = 0.5 * (x - y);
        }
  return cudaMemcpyToSymbol(c_EO, eo, sizeof(eo));
}

}  // namespace fast
}  // namespace hx
