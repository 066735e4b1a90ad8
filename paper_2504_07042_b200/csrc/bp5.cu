// BP5 / Nekbone CG proxy on a structured box (reference solver.py:64-308,
// mesh.py:286-335): gather, scatter-add, Dirichlet mask, deterministic dots and
// the CG vector updates.
//
// Global vectors live on the slab lattice of one rank: nodes (gx, gy, gz) with
// gx < nx = ex*N+1, gy < ny = ey*N+1 and gz in [z0*N, z1*N] (both interface
// planes included), x fastest — the reference's lattice numbering
// (mesh.py:271-274) restricted to the slab.  Element-local vectors are
// (E_slab, n1^3) in the reference's node order.
//
// scatter-add is owner-computes: each lattice node sums its (up to 8) element
// copies in ascending element index, the order np.bincount accumulates in
// (mesh.py:297-313), so on one rank it is bit-identical to the reference's
// scatter given identical element-local values; no atomics.
//
// Dots reduce in a fixed tree (fixed grid, per-block partials, one final
// block), so results are bitwise reproducible run to run.
#include "hx_common.cuh"

namespace hx {
namespace bp5 {

using Box = hx_box;  // include/hx_axlocal.h

__global__ void gather_kernel(Box b, const double* __restrict__ u, double* __restrict__ xl) {
  const int n1 = b.order + 1, n3 = n1 * n1 * n1;
  const int64_t nx = (int64_t)b.ex * b.order + 1, ny = (int64_t)b.ey * b.order + 1;
  const int64_t total = (int64_t)b.ex * b.ey * b.nz_el * n3;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = gid / n3;
    const int node = (int)(gid - e * n3);
    const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
    const int64_t cx = e % b.ex, cy = (e / b.ex) % b.ey, cz = e / ((int64_t)b.ex * b.ey);
    const int64_t gx = cx * b.order + i, gy = cy * b.order + j, gz = cz * b.order + k;  // slab-relative z
    xl[gid * b.n_col + b.col] = u[(gz * ny + gy) * nx + gx];
  }
}

// per-axis contributing (element, local index) pairs of lattice coordinate g
__device__ __forceinline__ int axis_owners(int64_t g, int n, int ne, int64_t c[2], int l[2]) {
  const int64_t q = g / n;
  const int r = (int)(g - q * n);
  int cnt = 0;
  if (r == 0) {
    if (q - 1 >= 0 && q - 1 < ne) { c[cnt] = q - 1; l[cnt] = n; ++cnt; }
    if (q < ne) { c[cnt] = q; l[cnt] = 0; ++cnt; }
  } else {
    c[0] = q;
    l[0] = r;
    cnt = 1;
  }
  return cnt;
}

__global__ void scatter_add_kernel(Box b, const double* __restrict__ yl, double* __restrict__ v) {
  const int n1 = b.order + 1, n3 = n1 * n1 * n1;
  const int64_t nx = (int64_t)b.ex * b.order + 1, ny = (int64_t)b.ey * b.order + 1;
  const int64_t nzl = (int64_t)b.nz_el * b.order + 1;
  const int64_t total = nx * ny * nzl;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gx = gid % nx, gy = (gid / nx) % ny, gz = gid / (nx * ny);
    int64_t cxs[2], cys[2], czs[2];
    int ls_x[2], ls_y[2], ls_z[2];
    const int nxo = axis_owners(gx, b.order, b.ex, cxs, ls_x);
    const int nyo = axis_owners(gy, b.order, b.ey, cys, ls_y);
    const int nzo = axis_owners(gz, b.order, b.nz_el, czs, ls_z);
    double acc = 0.0;
    // ascending element index e = (cz*ey + cy)*ex + cx: cz outer, then cy, then cx
    for (int a = 0; a < nzo; ++a)
      for (int bb = 0; bb < nyo; ++bb)
        for (int c = 0; c < nxo; ++c) {
          const int64_t e = (czs[a] * b.ey + cys[bb]) * b.ex + cxs[c];
          const int node = (ls_z[a] * n1 + ls_y[bb]) * n1 + ls_x[c];
          acc += yl[(e * n3 + node) * b.n_col + b.col];
        }
    v[gid] = acc;
  }
}

// v = mask(Q^T yl) and block partials of p.v over the owned nodes (fused CG step)
__global__ void scatter_dot_kernel(Box b, const double* __restrict__ yl, double* __restrict__ v,
                                   const double* __restrict__ p, int64_t n_owned, double* __restrict__ partial) {
  __shared__ double sred[256];
  const int n1 = b.order + 1, n3 = n1 * n1 * n1;
  const int64_t nx = (int64_t)b.ex * b.order + 1, ny = (int64_t)b.ey * b.order + 1;
  const int64_t nzl = (int64_t)b.nz_el * b.order + 1;
  const int64_t nz_glob = (int64_t)b.ez * b.order + 1;
  const int64_t gz_off = (int64_t)b.z0 * b.order;
  const int64_t total = nx * ny * nzl;
  double dot = 0.0;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gx = gid % nx, gy = (gid / nx) % ny, gz = gid / (nx * ny);
    double acc = 0.0;
    const int64_t gzg = gz + gz_off;
    const bool boundary = gx == 0 || gx == nx - 1 || gy == 0 || gy == ny - 1 || gzg == 0 || gzg == nz_glob - 1;
    if (!boundary) {
      int64_t cxs[2], cys[2], czs[2];
      int ls_x[2], ls_y[2], ls_z[2];
      const int nxo = axis_owners(gx, b.order, b.ex, cxs, ls_x);
      const int nyo = axis_owners(gy, b.order, b.ey, cys, ls_y);
      const int nzo = axis_owners(gz, b.order, b.nz_el, czs, ls_z);
      for (int a = 0; a < nzo; ++a)
        for (int bb = 0; bb < nyo; ++bb)
          for (int c = 0; c < nxo; ++c) {
            const int64_t e = (czs[a] * b.ey + cys[bb]) * b.ex + cxs[c];
            const int node = (ls_z[a] * n1 + ls_y[bb]) * n1 + ls_x[c];
            acc += yl[(e * n3 + node) * b.n_col + b.col];
          }
    }
    v[gid] = acc;
    if (gid < n_owned) dot = fma(p[gid], acc, dot);
  }
  sred[threadIdx.x] = dot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sred[threadIdx.x] += sred[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sred[0];
}

// zero the physical boundary of the global box (solver.py:56-61, mesh.py:316-335)
__global__ void mask_kernel(Box b, double* __restrict__ v) {
  const int64_t nx = (int64_t)b.ex * b.order + 1, ny = (int64_t)b.ey * b.order + 1;
  const int64_t nzl = (int64_t)b.nz_el * b.order + 1;
  const int64_t nz_glob = (int64_t)b.ez * b.order + 1;
  const int64_t gz_off = (int64_t)b.z0 * b.order;
  const int64_t total = nx * ny * nzl;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gx = gid % nx, gy = (gid / nx) % ny, gz = gid / (nx * ny) + gz_off;
    if (gx == 0 || gx == nx - 1 || gy == 0 || gy == ny - 1 || gz == 0 || gz == nz_glob - 1) v[gid] = 0.0;
  }
}

constexpr int kDotBlocks = 1184;  // fixed grid: the reduction tree never changes
constexpr int kDotThreads = 256;

// Block partial sums of a*b over [lo, hi) (fixed strided order, fixed tree).
__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t lo,
                                   int64_t hi, double* __restrict__ partial) {
  __shared__ double s[kDotThreads];
  double acc = 0.0;
  for (int64_t i = lo + (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < hi;
       i += (int64_t)kDotBlocks * kDotThreads)
    acc = fma(a[i], b[i], acc);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void dot_final_kernel(const double* __restrict__ partial, double* __restrict__ out) {
  __shared__ double s[kDotThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) acc += partial[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// x += alpha p; r -= alpha ap   (solver.py:159-160); alpha = rr / pap read on device
__global__ void cg_xr_kernel(const double* __restrict__ scal, double* __restrict__ x, const double* __restrict__ p,
                             double* __restrict__ r, const double* __restrict__ ap, int64_t n) {
  const double alpha = scal[0] / scal[1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // two roundings like numpy's x += alpha * p (no FMA contraction)
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
  }
}

// x += alpha p; r -= alpha ap; block partials of r.r over the owned nodes
__global__ void cg_xr_dot_kernel(const double* __restrict__ scal, double* __restrict__ x,
                                 const double* __restrict__ p, double* __restrict__ r,
                                 const double* __restrict__ ap, int64_t n, int64_t n_owned,
                                 double* __restrict__ partial) {
  __shared__ double sred[256];
  const double alpha = scal[0] / scal[1];
  double dot = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
    r[i] = ri;
    if (i < n_owned) dot = fma(ri, ri, dot);
  }
  sred[threadIdx.x] = dot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sred[threadIdx.x] += sred[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sred[0];
}

// p = r + (rr_new / rr) p   (solver.py:170)
__global__ void cg_p_kernel(const double* __restrict__ scal, double* __restrict__ p, const double* __restrict__ r,
                            int64_t n) {
  const double beta = scal[2] / scal[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

inline unsigned grid_for(int64_t n, int tpb) {
  const int64_t g = (n + tpb - 1) / tpb;
  return (unsigned)(g < 148 * 64 ? (g > 0 ? g : 1) : 148 * 64);
}

}  // namespace bp5
}  // namespace hx

using hx::bp5::Box;

extern "C" cudaError_t hx_bp5_gather_impl(Box b, const double* u, double* xl, cudaStream_t s) {
  const int64_t n = (int64_t)b.ex * b.ey * b.nz_el * (b.order + 1) * (b.order + 1) * (b.order + 1);
  hx::bp5::gather_kernel<<<hx::bp5::grid_for(n, 256), 256, 0, s>>>(b, u, xl);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_bp5_scatter_impl(Box b, const double* yl, double* v, cudaStream_t s) {
  const int64_t n = ((int64_t)b.ex * b.order + 1) * ((int64_t)b.ey * b.order + 1) * ((int64_t)b.nz_el * b.order + 1);
  hx::bp5::scatter_add_kernel<<<hx::bp5::grid_for(n, 256), 256, 0, s>>>(b, yl, v);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_bp5_mask_impl(Box b, double* v, cudaStream_t s) {
  const int64_t n = ((int64_t)b.ex * b.order + 1) * ((int64_t)b.ey * b.order + 1) * ((int64_t)b.nz_el * b.order + 1);
  hx::bp5::mask_kernel<<<hx::bp5::grid_for(n, 256), 256, 0, s>>>(b, v);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_dot_impl(const double* a, const double* b, int64_t lo, int64_t hi, double* work,
                                   double* out, cudaStream_t s) {
  hx::bp5::dot_partial_kernel<<<hx::bp5::kDotBlocks, hx::bp5::kDotThreads, 0, s>>>(a, b, lo, hi, work);
  hx::bp5::dot_final_kernel<<<1, hx::bp5::kDotThreads, 0, s>>>(work, out);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_cg_xr_impl(const double* scal, double* x, const double* p, double* r, const double* ap,
                                     int64_t n, cudaStream_t s) {
  hx::bp5::cg_xr_kernel<<<hx::bp5::grid_for(n, 256), 256, 0, s>>>(scal, x, p, r, ap, n);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_cg_p_impl(const double* scal, double* p, const double* r, int64_t n, cudaStream_t s) {
  hx::bp5::cg_p_kernel<<<hx::bp5::grid_for(n, 256), 256, 0, s>>>(scal, p, r, n);
  return cudaGetLastError();
}


extern "C" cudaError_t hx_bp5_scatter_dot_impl(Box b, const double* yl, double* v, const double* p, int64_t n_owned,
                                               double* work, double* out, cudaStream_t s) {
  hx::bp5::scatter_dot_kernel<<<hx::bp5::kDotBlocks, 256, 0, s>>>(b, yl, v, p, n_owned, work);
  hx::bp5::dot_final_kernel<<<1, hx::bp5::kDotThreads, 0, s>>>(work, out);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_cg_xr_dot_impl(const double* scal, double* x, const double* p, double* r,
                                         const double* ap, int64_t n, int64_t n_owned, double* work, double* out,
                                         cudaStream_t s) {
  hx::bp5::cg_xr_dot_kernel<<<hx::bp5::kDotBlocks, 256, 0, s>>>(scal, x, p, r, ap, n, n_owned, work);
  hx::bp5::dot_final_kernel<<<1, hx::bp5::kDotThreads, 0, s>>>(work, out);
  return cudaGetLastError();
}
