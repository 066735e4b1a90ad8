// Setup-stage kernels: geometry validation and the per-variant factor data
// the apply kernels stream (LocalOperator.__init__, axlocal.py:136-169).
//
// These run once per operator, so they are written for clarity (one thread
// per node or element, runtime order) rather than speed; at the 1.5 M-element
// configuration they still take well under a second, where the reference's
// numpy setup cannot allocate its temporaries.
#include "hx_common.cuh"
#include <cstdlib>

namespace hx {
namespace {

__device__ __forceinline__ void atomic_min_i64(int64_t* addr, int64_t v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(v));
}

__global__ void init_i64(int64_t* p, int64_t v) { *p = v; }

// Trilinear-route det(8J), lam_geo and gwj at every node; one thread per node.
// mode 0: validate only; 1: lam_geo; 2: merged lam2/lam3.
__global__ void trilinear_setup_kernel(int n1, int64_t E, const double* __restrict__ verts, int mode,
                                       int64_t* first_bad, double* out_a, double* out_b,
                                       const double* __restrict__ lam0, double l0v,
                                       const double* __restrict__ lam1, double l1v) {
  const int n3 = n1 * n1 * n1;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= E * n3) return;
  const int64_t e = gid / n3;
  const int node = (int)(gid % n3);
  const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
  const int op = off_p(n1);
  double v[24];
  for (int q = 0; q < 24; ++q) v[q] = verts[e * 24 + q];
  TrilinearPencil p;
  trilinear_pencil(v, c_X[op + i], c_X[op + j], p);
  double g[6], det;
  trilinear_node(p, c_X[op + k], g, det);
  if (det <= 0.0 || det != det) {
    if (first_bad) atomic_min_i64(first_bad, gid);
    return;
  }
  if (mode == 0) return;
  const double w = c_W[op + k] * c_W[op + j] * c_W[op + i];
  const double lam_geo = 0.125 * w / det;
  if (mode == 1) {
    out_a[gid] = lam_geo;
  } else {
    const double gwj_weighted = lam_geo * (0.015625 * det * det);
    out_a[gid] = lam_geo * (lam0 ? lam0[gid] : l0v);
    out_b[gid] = gwj_weighted * (lam1 ? lam1[gid] : l1v);
  }
}

// The same at a compile-time order, one thread per k-fibre (element, i, j): the
// vertices are loaded and the (i, j) pencil built once for the fibre's n1 nodes
// instead of once per node (the per-node kernel reloads 24 vertex doubles and
// divides 64-bit indices at every node). Same per-node arithmetic.
template <int N1T>
__global__ void __launch_bounds__(256) trilinear_setup_fibre_kernel(int64_t E, const double* __restrict__ verts,
                                                                    int mode, int64_t* first_bad, double* out_a,
                                                                    double* out_b, const double* __restrict__ lam0,
                                                                    double l0v, const double* __restrict__ lam1,
                                                                    double l1v) {
  constexpr int n1 = N1T, n2 = n1 * n1, n3 = n2 * n1;
  const int64_t fid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (fid >= E * n2) return;
  const int64_t e = fid / n2;
  const int f = (int)(fid - e * n2), i = f % n1, j = f / n1;
  const int op = off_p(n1);
  double v[24];
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(verts + e * 24) + q);
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
  TrilinearPencil p;
  trilinear_pencil(v, c_X[op + i], c_X[op + j], p);
#pragma unroll 1
  for (int k = 0; k < n1; ++k) {
    const int64_t gid = e * n3 + k * n2 + f;
    double g[6], det;
    trilinear_node(p, c_X[op + k], g, det);
    if (det <= 0.0 || det != det) {
      if (first_bad) atomic_min_i64(first_bad, gid);
      continue;
    }
    if (mode == 0) continue;
    const double w = c_W[op + k] * c_W[op + j] * c_W[op + i];
    const double lam_geo = 0.125 * w / det;
    if (mode == 1) {
      out_a[gid] = lam_geo;
    } else {
      const double gwj_weighted = lam_geo * (0.015625 * det * det);
      out_a[gid] = lam_geo * (lam0 ? lam0[gid] : l0v);
      out_b[gid] = gwj_weighted * (lam1 ? lam1[gid] : l1v);
    }
  }
}

// Physical coordinate c of GLL node (i, j, k) under the trilinear map
// (element_node_coords, mesh.py:130-137).
__device__ __forceinline__ double node_coord(const double v[24], const double* xi, int i, int j, int k, int c) {
  // blend weight 0.125 ((b_k b_j) b_i) (the einsum "kc,jb,ia->kjicba"), then the
  // reference's `blend @ v` product, which its BLAS evaluates as one FMA chain
  // over the 8 vertices in order (bitwise-checked against numpy/OpenBLAS)
  const double bi[2] = {1.0 - xi[i], 1.0 + xi[i]};
  const double bj[2] = {1.0 - xi[j], 1.0 + xi[j]};
  const double bk[2] = {1.0 - xi[k], 1.0 + xi[k]};
  double s = 0.0;
  for (int b = 0; b < 8; ++b) {
    const double wgt = __dmul_rn(0.125, __dmul_rn(__dmul_rn(bk[(b >> 2) & 1], bj[(b >> 1) & 1]), bi[b & 1]));
    s = fma(wgt, v[b * 3 + c], s);
  }
  return s;
}

// The collocation derivatives in the reference's own rounding (contractions.py:35-57
// via discrete_jacobians, geometry.py:237-241: np.einsum optimize=False on a strided
// coordinate column, which numpy evaluates as a sequential sum of separately rounded
// products for all three directions; bitwise-checked).  On axis-aligned elements an
// exact-zero Jacobian entry is c * sum_n D_in up to rounding, and a derivative of
// a coordinate whose range is small against its magnitude cancels ~10 digits: on
// C1's 1/512 x 1 x 1 elements either moves the stored factors by ~1e-12 relative
// unless the summation matches.
// Stored (general-route) factors: collocation Jacobian + dense inverse
// (discrete_jacobians + factors_from_jacobians, geometry.py:225-276).
// One block per element: node coordinates staged in shared memory, then each
// thread contracts them with D for its nodes.
__global__ void stored_setup_kernel(int n1, int64_t E, const double* __restrict__ verts, double* g_out,
                                    double* gwj_out, int64_t* first_bad) {
  extern __shared__ double s_xyz[];  // [3][n3]
  const int n3 = n1 * n1 * n1;
  const int64_t e = blockIdx.x;
  const int od = off_d(n1), op = off_p(n1);
  const double* xi = c_X + op;
  double v[24];
  for (int q = 0; q < 24; ++q) v[q] = verts[e * 24 + q];
  for (int node = threadIdx.x; node < n3; node += blockDim.x) {
    const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
    for (int c = 0; c < 3; ++c) s_xyz[c * n3 + node] = node_coord(v, xi, i, j, k, c);
  }
  __syncthreads();
  for (int node = threadIdx.x; node < n3; node += blockDim.x) {
    const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
    double jac[3][3];  // jac[a][b] = d x_a / d r_b
    for (int c = 0; c < 3; ++c) {
      const double* X = s_xyz + c * n3;
      double dr = 0.0, ds = 0.0, dt = 0.0;
      for (int n = 0; n < n1; ++n) {
        dr = __dadd_rn(dr, __dmul_rn(c_D[od + i * n1 + n], X[(k * n1 + j) * n1 + n]));
        ds = __dadd_rn(ds, __dmul_rn(c_D[od + j * n1 + n], X[(k * n1 + n) * n1 + i]));
        dt = __dadd_rn(dt, __dmul_rn(c_D[od + k * n1 + n], X[(n * n1 + j) * n1 + i]));
      }
      jac[c][0] = dr;
      jac[c][1] = ds;
      jac[c][2] = dt;
    }
    const double c0[3] = {jac[0][0], jac[1][0], jac[2][0]};
    const double c1[3] = {jac[0][1], jac[1][1], jac[2][1]};
    const double c2[3] = {jac[0][2], jac[1][2], jac[2][2]};
    const double det = det3_cols(c0, c1, c2);
    const int64_t gid = e * n3 + node;
    if (det <= 0.0 || det != det) {
      atomic_min_i64(first_bad, gid);
      continue;
    }
    // inverse = adj(jac) / det
    double inv[3][3];
    inv[0][0] = (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) / det;
    inv[0][1] = (jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2]) / det;
    inv[0][2] = (jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1]) / det;
    inv[1][0] = (jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2]) / det;
    inv[1][1] = (jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0]) / det;
    inv[1][2] = (jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2]) / det;
    inv[2][0] = (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]) / det;
    inv[2][1] = (jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1]) / det;
    inv[2][2] = (jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0]) / det;
    double m[3][3];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c)
        m[a][c] = inv[a][0] * inv[c][0] + inv[a][1] * inv[c][1] + inv[a][2] * inv[c][2];
    const double w = c_W[op + k] * c_W[op + j] * c_W[op + i];
    const double scale = w * det;
    double* g = g_out + e * 6 * n3 + node;
    g[0 * n3] = scale * m[0][0];
    g[1 * n3] = scale * m[0][1];
    g[2 * n3] = scale * m[0][2];
    g[3 * n3] = scale * m[1][1];
    g[4 * n3] = scale * m[1][2];
    g[5 * n3] = scale * m[2][2];
    if (gwj_out) gwj_out[gid] = scale;
  }
}

// The same computation at a compile-time order (N1T points), the orders the
// bench and the tests build most: unrolled loops, shift / mask node indices,
// D from shared memory (its lane-dependent rows made the constant-bank loads of
// the generic kernel serialize; 65 ms -> see profiles/r02_setup_ab.txt at C4).
// Same operations in the same order as stored_setup_kernel.
template <int N1T>
__global__ void __launch_bounds__(256) stored_setup_kernel_ct(int64_t E, const double* __restrict__ verts,
                                                             double* g_out, double* gwj_out, int64_t* first_bad) {
  constexpr int n1 = N1T, n3 = n1 * n1 * n1;
  __shared__ double s_xyz[3 * n3];
  __shared__ double sD[n1 * n1];
  const int64_t e = blockIdx.x;
  const int od = off_d(n1), op = off_p(n1);
  const double* xi = c_X + op;
  for (int q = threadIdx.x; q < n1 * n1; q += blockDim.x) sD[q] = c_D[od + q];
  double v[24];
#pragma unroll
  for (int q = 0; q < 24; ++q) v[q] = __ldg(verts + e * 24 + q);
  for (int node = threadIdx.x; node < n3; node += blockDim.x) {
    const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
#pragma unroll
    for (int c = 0; c < 3; ++c) s_xyz[c * n3 + node] = node_coord(v, xi, i, j, k, c);
  }
  __syncthreads();
  for (int node = threadIdx.x; node < n3; node += blockDim.x) {
    const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
    double jac[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double* X = s_xyz + c * n3;
      double dr = 0.0, ds = 0.0, dt = 0.0;
#pragma unroll
      for (int n = 0; n < n1; ++n) {
        dr = __dadd_rn(dr, __dmul_rn(sD[i * n1 + n], X[(k * n1 + j) * n1 + n]));
        ds = __dadd_rn(ds, __dmul_rn(sD[j * n1 + n], X[(k * n1 + n) * n1 + i]));
        dt = __dadd_rn(dt, __dmul_rn(sD[k * n1 + n], X[(n * n1 + j) * n1 + i]));
      }
      jac[c][0] = dr;
      jac[c][1] = ds;
      jac[c][2] = dt;
    }
    const double c0[3] = {jac[0][0], jac[1][0], jac[2][0]};
    const double c1[3] = {jac[0][1], jac[1][1], jac[2][1]};
    const double c2[3] = {jac[0][2], jac[1][2], jac[2][2]};
    const double det = det3_cols(c0, c1, c2);
    const int64_t gid = e * n3 + node;
    if (det <= 0.0 || det != det) {
      atomic_min_i64(first_bad, gid);
      continue;
    }
    double inv[3][3];
    inv[0][0] = (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) / det;
    inv[0][1] = (jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2]) / det;
    inv[0][2] = (jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1]) / det;
    inv[1][0] = (jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2]) / det;
    inv[1][1] = (jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0]) / det;
    inv[1][2] = (jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2]) / det;
    inv[2][0] = (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]) / det;
    inv[2][1] = (jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1]) / det;
    inv[2][2] = (jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0]) / det;
    double m[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        m[a][c] = inv[a][0] * inv[c][0] + inv[a][1] * inv[c][1] + inv[a][2] * inv[c][2];
    const double w = c_W[op + k] * c_W[op + j] * c_W[op + i];
    const double scale = w * det;
    double* g = g_out + e * 6 * n3 + node;
    g[0 * n3] = scale * m[0][0];
    g[1 * n3] = scale * m[0][1];
    g[2 * n3] = scale * m[0][2];
    g[3 * n3] = scale * m[1][1];
    g[4 * n3] = scale * m[1][2];
    g[5 * n3] = scale * m[2][2];
    if (gwj_out) gwj_out[gid] = scale;
  }
}

__device__ __forceinline__ double ppd_defect(const double* v, double& scale) {
  double d = 0.0, mx = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double v0 = v[c], v1 = v[3 + c], v2 = v[6 + c], v4 = v[12 + c];
    d = fmax(d, fabs(v[9 + c] - (v1 + v2 - v0)));
    d = fmax(d, fabs(v[15 + c] - (v1 + v4 - v0)));
    d = fmax(d, fabs(v[18 + c] - (v2 + v4 - v0)));
    d = fmax(d, fabs(v[21 + c] - (v1 + v2 + v4 - 2.0 * v0)));
  }
  for (int q = 0; q < 24; ++q) mx = fmax(mx, fabs(v[q]));
  scale = fmax(1.0, mx);
  return d;
}

__global__ void classify_kernel(int64_t E, const double* __restrict__ verts, int8_t* kind) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double v[24];
  for (int q = 0; q < 24; ++q) v[q] = verts[e * 24 + q];
  double scale;
  const double d = ppd_defect(v, scale);
  kind[e] = d <= 1e-12 * scale ? 1 : 0;
}

// parallelepiped_setup (geometry.py:362-380).
__global__ void ppd_setup_kernel(int64_t E, const double* __restrict__ verts, double* h, int64_t* bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double v[24];
  for (int q = 0; q < 24; ++q) v[q] = verts[e * 24 + q];
  double scale;
  const double defect = ppd_defect(v, scale);
  if (defect > 1e-10 * scale) {
    atomic_min_i64(bad, 2 * e);
    return;
  }
  double jac[3][3];
  for (int a = 0; a < 3; ++a) {
    jac[a][0] = 0.5 * (v[3 + a] - v[a]);
    jac[a][1] = 0.5 * (v[6 + a] - v[a]);
    jac[a][2] = 0.5 * (v[12 + a] - v[a]);
  }
  const double c0[3] = {jac[0][0], jac[1][0], jac[2][0]};
  const double c1[3] = {jac[0][1], jac[1][1], jac[2][1]};
  const double c2[3] = {jac[0][2], jac[1][2], jac[2][2]};
  const double det = det3_cols(c0, c1, c2);
  if (det <= 0.0 || det != det) {
    atomic_min_i64(bad, 2 * e + 1);
    return;
  }
  // det * inv inv^T = adj adj^T / det
  double adj[3][3];
  adj[0][0] = jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1];
  adj[0][1] = jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2];
  adj[0][2] = jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1];
  adj[1][0] = jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2];
  adj[1][1] = jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0];
  adj[1][2] = jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2];
  adj[2][0] = jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0];
  adj[2][1] = jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1];
  adj[2][2] = jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0];
  double m[3][3];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      m[a][c] = (adj[a][0] * adj[c][0] + adj[a][1] * adj[c][1] + adj[a][2] * adj[c][2]) / det;
  double* out = h + e * 7;
  out[0] = m[0][0];
  out[1] = m[0][1];
  out[2] = m[0][2];
  out[3] = m[1][1];
  out[4] = m[1][2];
  out[5] = m[2][2];
  out[6] = det;
}

inline unsigned grid_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }

}  // namespace
}  // namespace hx

extern "C" cudaError_t hx_setup_trilinear_impl(int n1, int64_t E, const double* verts, int mode,
                                               int64_t* first_bad, double* a, double* b, const double* lam0,
                                               double l0v, const double* lam1, double l1v, cudaStream_t s) {
  if (first_bad) hx::init_i64<<<1, 1, 0, s>>>(first_bad, INT64_MAX);
  const int64_t n = E * n1 * n1 * n1;
  // 16-byte aligned vertices (double2 loads) at N = 7: one thread per k-fibre (bitwise
  // the same results; HX_SETUP_GENERIC=1 forces the per-node kernel, A/B and tests only)
  if (n > 0 && n1 == 8 && (reinterpret_cast<uintptr_t>(verts) & 15) == 0 && !std::getenv("HX_SETUP_GENERIC")) {
    hx::trilinear_setup_fibre_kernel<8><<<hx::grid_for(E * 64, 256), 256, 0, s>>>(E, verts, mode, first_bad, a, b,
                                                                                 lam0, l0v, lam1, l1v);
    return cudaGetLastError();
  }
  if (n > 0)
    hx::trilinear_setup_kernel<<<hx::grid_for(n, 256), 256, 0, s>>>(n1, E, verts, mode, first_bad, a, b, lam0,
                                                                     l0v, lam1, l1v);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_setup_stored_impl(int n1, int64_t E, const double* verts, double* g, double* gwj,
                                            int64_t* first_bad, cudaStream_t s) {
  hx::init_i64<<<1, 1, 0, s>>>(first_bad, INT64_MAX);
  const int n3 = n1 * n1 * n1;
  const size_t smem = sizeof(double) * 3 * n3;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(hx::stored_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  // grid.x <= 2^31-1 elements. N = 7 takes the compile-time-order kernel (bitwise the
  // same fields); HX_SETUP_GENERIC=1 forces the generic one (A/B and the GPU test
  // test_order7_setup_kernels_match_the_generic_order only)
  if (E > 0 && n1 == 8 && !std::getenv("HX_SETUP_GENERIC")) {
    hx::stored_setup_kernel_ct<8><<<(unsigned)E, 256, 0, s>>>(E, verts, g, gwj, first_bad);
    return cudaGetLastError();
  }
  if (E > 0) hx::stored_setup_kernel<<<(unsigned)E, n3 < 256 ? n3 : 256, smem, s>>>(n1, E, verts, g, gwj, first_bad);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_setup_ppd_impl(int64_t E, const double* verts, double* h, int64_t* bad, cudaStream_t s) {
  hx::init_i64<<<1, 1, 0, s>>>(bad, INT64_MAX);
  if (E > 0) hx::ppd_setup_kernel<<<hx::grid_for(E, 128), 128, 0, s>>>(E, verts, h, bad);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_classify_impl(int64_t E, const double* verts, int8_t* kind, cudaStream_t s) {
  if (E > 0) hx::classify_kernel<<<hx::grid_for(E, 128), 128, 0, s>>>(E, verts, kind);
  return cudaGetLastError();
}

HX_DEFINE_UPLOAD_HOOK(hx_upload_basis_setup)
