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

#ifndef HX_BAND_MINB
#define HX_BAND_MINB 4
#endif

namespace hx {
namespace bp5 {

using Box = hx_box;  // include/hx_axlocal.h


// The (up to two) element copies of lattice coordinate g along one axis, lower
// element first: element q-1 at local index n and element q at local index 0 when
// g = q n (a shared plane), else element q at local g - q n.  off = that copy's
// contribution to the element-local address (element index x stride + local x
// node stride), so a node's copy address is a sum of three per-axis offsets.
struct AxisCopies {
  int64_t off[2];
  bool ok[2];
};

__device__ __forceinline__ AxisCopies axis_copies(int g, int n, int ne, int64_t elem_stride, int node_stride) {
  const int q = (int)((unsigned)g / (unsigned)n);  // lattice coordinates fit in 32 bits
  const int r = g - q * n;
  AxisCopies a;
  if (r == 0) {
    a.ok[0] = q >= 1 && q - 1 < ne;
    a.off[0] = (int64_t)(q - 1) * elem_stride + (int64_t)n * node_stride;
    a.ok[1] = q < ne;
    a.off[1] = (int64_t)q * elem_stride;
  } else {
    a.ok[0] = false;
    a.off[0] = 0;
    a.ok[1] = true;
    a.off[1] = (int64_t)q * elem_stride + (int64_t)r * node_stride;
  }
  return a;
}

constexpr int kRowsPerBlock = 16;  // a block owns a band of lattice rows (fixed gz)
constexpr int kDotBlocks = 1184;   // fixed grids: the reduction trees never change
constexpr int kDotThreads = 256;

// Blocks start in launch order with ~4 x 148 resident: warm L2 with the element
// k-planes (512 B each, one bulk prefetch per thread) that the block two waves
// ahead will read -- the band kernel is otherwise DRAM-latency bound.
constexpr int64_t kBandAhead = 148 * 4 * 2;

template <int NT>
__device__ __forceinline__ void prefetch_band_ahead(const Box& b, const double* yl, int nx, int ny) {
  constexpr int n = NT, n1 = n + 1, n2 = n1 * n1, n3 = n2 * n1;
  const int64_t nblk = (int64_t)gridDim.x * gridDim.y;
  const int64_t ahead = (int64_t)blockIdx.y * gridDim.x + blockIdx.x + kBandAhead;
  if (ahead >= nblk) return;
  const int band = (int)(ahead % gridDim.x), gz = (int)(ahead / gridDim.x);
  const int q = gz / n, r = gz - q * n;
  int cz0, k0, nzc;  // z copies: element layer and k-plane of each
  if (r == 0) {
    nzc = (q >= 1 && q - 1 < b.nz_el ? 1 : 0) + (q < b.nz_el ? 1 : 0);
    cz0 = q >= 1 ? q - 1 : q;
    k0 = q >= 1 ? n : 0;
  } else {
    nzc = 1;
    cz0 = q;
    k0 = r;
  }
  const int gy0 = band * kRowsPerBlock, gy1 = min(gy0 + kRowsPerBlock, ny);
  const int cy0 = max(0, gy0 / n - 1), cy1 = min(b.ey - 1, (gy1 - 1) / n);
  const int ncy = cy1 - cy0 + 1;
  const int total = nzc * ncy * b.ex;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int zc = t / (ncy * b.ex), rem = t - zc * ncy * b.ex;
    const int cy = cy0 + rem / b.ex, cx = rem % b.ex;
    const int cz = cz0 + zc, kz = zc ? 0 : k0;
    const int64_t e = ((int64_t)cz * b.ey + cy) * b.ex + cx;
    bulk_prefetch_l2(yl + e * n3 + (int64_t)kz * n2, n2 * 8);
  }
  (void)nx;
}

// NT = compile-time order (7) or 0 (runtime b.order).  Each thread walks one
// lattice column x = gx through the band's rows; copies are summed z-lower,
// y-lower, x-lower first (ascending element index, np.bincount's order).  All
// per-axis state lives in registers (no local-memory arrays), and the rows'
// loads are independent so several rows are in flight per thread.
template <int NT>
__global__ void __launch_bounds__(256, HX_BAND_MINB) scatter_band_kernel(Box b, const double* __restrict__ yl,
                                                           double* __restrict__ v, const double* __restrict__ p,
                                                           int64_t n_owned, double* __restrict__ partial,
                                                           int do_mask) {
  __shared__ double sred[256];
  const int n = NT ? NT : b.order;
  const int n1 = n + 1, n3 = n1 * n1 * n1;
  const int nx = b.ex * n + 1, ny = b.ey * n + 1;
  const int gz = blockIdx.y;
  const int gzg = gz + b.z0 * n, nzg = b.ez * n + 1;
  const int64_t ncol = b.n_col;
  const int64_t ex_n3 = (int64_t)b.ex * n3;
  const AxisCopies az = axis_copies(gz, n, b.nz_el, (int64_t)b.ey * ex_n3, n1 * n1);
  const bool plane_boundary = gzg == 0 || gzg == nzg - 1;
  const int gy0 = blockIdx.x * kRowsPerBlock;
  const int gy1 = min(gy0 + kRowsPerBlock, ny);
  if constexpr (NT == 7) {
    if (ncol == 1) prefetch_band_ahead<NT>(b, yl, nx, ny);
  }
  double dot = 0.0;
  for (int gx = threadIdx.x; gx < nx; gx += blockDim.x) {
    const AxisCopies ax = axis_copies(gx, n, b.ex, n3, 1);
    const bool col_boundary = plane_boundary || gx == 0 || gx == nx - 1;
#pragma unroll 4
    for (int gy = gy0; gy < gy1; ++gy) {
      const AxisCopies ay = axis_copies(gy, n, b.ey, ex_n3, n1);
      double acc = 0.0;
      if (!(do_mask && (col_boundary || gy == 0 || gy == ny - 1))) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // ascending element index: z, y, x lower copy first
          const int iz = q >> 2, iy = (q >> 1) & 1, ix = q & 1;
          if (az.ok[iz] && ay.ok[iy] && ax.ok[ix])
            acc += __ldg(yl + (az.off[iz] + ay.off[iy] + ax.off[ix]) * ncol + b.col);
        }
      }
      const int64_t gid = ((int64_t)gz * ny + gy) * nx + gx;
      v[gid] = acc;
      if (p && gid < n_owned) dot = fma(p[gid], acc, dot);
    }
  }
  if (!partial) return;
  sred[threadIdx.x] = dot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sred[threadIdx.x] += sred[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = sred[0];
}

// The same band scatter with 32-bit indices (slab element-local vector and
// lattice below 2^31 entries, one column): fewer registers -> 8 blocks of 256
// threads per SM instead of 4, and the kernel is latency bound, so occupancy is
// what pays (76^3 elements: 2.0 -> 1.7 ms).
struct AxisCopies32 {
  int off[2];
  bool ok[2];
};

__device__ __forceinline__ AxisCopies32 axis_copies32(int g, int n, int ne, int elem_stride, int node_stride) {
  const int q = (int)((unsigned)g / (unsigned)n);
  const int r = g - q * n;
  AxisCopies32 a;
  if (r == 0) {
    a.ok[0] = q >= 1 && q - 1 < ne;
    a.off[0] = (q - 1) * elem_stride + n * node_stride;
    a.ok[1] = q < ne;
    a.off[1] = q * elem_stride;
  } else {
    a.ok[0] = false;
    a.off[0] = 0;
    a.ok[1] = true;
    a.off[1] = q * elem_stride + r * node_stride;
  }
  return a;
}

// rows in flight per thread / blocks per SM: deeper unrolling (8, 16 rows at 4 or 2
// blocks per SM) made the C5 solve 15 % slower (profiles/r02_scatter_ab.txt)
#ifndef HX_SCATTER_UNROLL
#define HX_SCATTER_UNROLL 4
#endif
#ifndef HX_SCATTER_MINB
#define HX_SCATTER_MINB 8
#endif
constexpr int kScatterUnroll = HX_SCATTER_UNROLL;
__global__ void __launch_bounds__(256, HX_SCATTER_MINB) scatter_band32_kernel(Box b, const double* __restrict__ yl,
                                                                double* __restrict__ v, const double* __restrict__ p,
                                                                int64_t n_owned, double* __restrict__ partial,
                                                                int do_mask) {
  __shared__ double sred[256];
  constexpr int n = 7, n1 = 8, n3 = 512;
  const int nx = b.ex * n + 1, ny = b.ey * n + 1;
  const int gz = blockIdx.y;
  const int gzg = gz + b.z0 * n, nzg = b.ez * n + 1;
  const int ex_n3 = b.ex * n3;
  const AxisCopies32 az = axis_copies32(gz, n, b.nz_el, b.ey * ex_n3, n1 * n1);
  const bool plane_boundary = gzg == 0 || gzg == nzg - 1;
  const int gy0 = blockIdx.x * kRowsPerBlock;
  const int gy1 = min(gy0 + kRowsPerBlock, ny);
  prefetch_band_ahead<7>(b, yl, nx, ny);
  const int owned = n_owned < 0x7fffffffLL ? (int)n_owned : 0x7fffffff;
  double dot = 0.0;
  for (int gx = threadIdx.x; gx < nx; gx += blockDim.x) {
    const AxisCopies32 ax = axis_copies32(gx, n, b.ex, n3, 1);
    const bool col_boundary = plane_boundary || gx == 0 || gx == nx - 1;
#pragma unroll kScatterUnroll
    for (int gy = gy0; gy < gy1; ++gy) {
      const AxisCopies32 ay = axis_copies32(gy, n, b.ey, ex_n3, n1);
      double acc = 0.0;
      if (!(do_mask && (col_boundary || gy == 0 || gy == ny - 1))) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // ascending element index: z, y, x lower copy first
          const int iz = q >> 2, iy = (q >> 1) & 1, ix = q & 1;
          if (az.ok[iz] && ay.ok[iy] && ax.ok[ix]) acc += __ldg(yl + (az.off[iz] + ay.off[iy] + ax.off[ix]));
        }
      }
      const int gid = (gz * ny + gy) * nx + gx;
      v[gid] = acc;
      if (p && gid < owned) dot = fma(p[gid], acc, dot);
    }
  }
  if (!partial) return;
  sred[threadIdx.x] = dot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sred[threadIdx.x] += sred[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = sred[0];
}

// sums the per-row partials in a fixed order (one block)
__global__ void rows_final_kernel(const double* __restrict__ partial, int64_t count, double* __restrict__ out) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += 256) acc += partial[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// zero the physical boundary of the global box (solver.py:56-61, mesh.py:316-335)
__global__ void mask_rows_kernel(Box b, double* __restrict__ v) {
  const int nx = b.ex * b.order + 1, ny = b.ey * b.order + 1;
  const int gy = blockIdx.y, gz = blockIdx.z;
  const int gzg = gz + b.z0 * b.order, nzg = b.ez * b.order + 1;
  const bool row_boundary = gy == 0 || gy == ny - 1 || gzg == 0 || gzg == nzg - 1;
  const int64_t row = ((int64_t)gz * ny + gy) * nx;
  for (int gx = blockIdx.x * blockDim.x + threadIdx.x; gx < nx; gx += gridDim.x * blockDim.x)
    if (row_boundary || gx == 0 || gx == nx - 1) v[row + gx] = 0.0;
}

// gather with a 3D grid: one element-row (e, j, k) per thread group, no 64-bit division
__global__ void gather_rows_kernel(Box b, const double* __restrict__ u, double* __restrict__ xl) {
  const int n1 = b.order + 1, n3 = n1 * n1 * n1;
  const int nx = b.ex * b.order + 1, ny = b.ey * b.order + 1;
  // element rows (cy, cz) grid-strided over grid.y (<= 65535 rows per launch)
  for (int rowe = blockIdx.y; rowe < b.ey * b.nz_el; rowe += gridDim.y) {
    const int cy = rowe % b.ey, cz = rowe / b.ey;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < b.ex * n3; t += gridDim.x * blockDim.x) {
      const int cx = t / n3, node = t - cx * n3;
      const int i = node % n1, j = (node / n1) % n1, k = node / (n1 * n1);
      const int64_t e = ((int64_t)cz * b.ey + cy) * b.ex + cx;
      const int64_t g = ((int64_t)(cz * b.order + k) * ny + cy * b.order + j) * nx + cx * b.order + i;
      xl[(e * n3 + node) * b.n_col + b.col] = u[g];
    }
  }
}

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

namespace {
dim3 rows_grid(const Box& b, int tpb) {
  const int nx = b.ex * b.order + 1, ny = b.ey * b.order + 1, nzl = b.nz_el * b.order + 1;
  return dim3((nx + tpb - 1) / tpb, ny, nzl);
}
dim3 band_grid(const Box& b) {
  const int ny = b.ey * b.order + 1, nzl = b.nz_el * b.order + 1;
  return dim3((ny + hx::bp5::kRowsPerBlock - 1) / hx::bp5::kRowsPerBlock, nzl);
}
}  // namespace

extern "C" cudaError_t hx_bp5_gather_impl(Box b, const double* u, double* xl, cudaStream_t s) {
  const int n3 = (b.order + 1) * (b.order + 1) * (b.order + 1);
  const int per_row = b.ex * n3;
  const int rows = b.ey * b.nz_el;
  dim3 grid((per_row + 255) / 256, rows < 65535 ? rows : 65535);
  hx::bp5::gather_rows_kernel<<<grid, 256, 0, s>>>(b, u, xl);
  return cudaGetLastError();
}

namespace {
// the 32-bit band kernel covers N = 7, one column, both index spaces below 2^31
bool band32_ok(const Box& b) {
  if (b.order != 7 || b.n_col != 1) return false;
  const int64_t local = (int64_t)b.ex * b.ey * b.nz_el * 512;
  const int64_t lattice = ((int64_t)b.ex * 7 + 1) * ((int64_t)b.ey * 7 + 1) * ((int64_t)b.nz_el * 7 + 1);
  return local < 0x7fffffffLL && lattice < 0x7fffffffLL;
}
}  // namespace

extern "C" cudaError_t hx_bp5_scatter_impl(Box b, const double* yl, double* v, cudaStream_t s) {
  if (band32_ok(b))
    hx::bp5::scatter_band32_kernel<<<band_grid(b), 256, 0, s>>>(b, yl, v, nullptr, 0, nullptr, 0);
  else if (b.order == 7)
    hx::bp5::scatter_band_kernel<7><<<band_grid(b), 256, 0, s>>>(b, yl, v, nullptr, 0, nullptr, 0);
  else
    hx::bp5::scatter_band_kernel<0><<<band_grid(b), 256, 0, s>>>(b, yl, v, nullptr, 0, nullptr, 0);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_bp5_mask_impl(Box b, double* v, cudaStream_t s) {
  hx::bp5::mask_rows_kernel<<<rows_grid(b, 128), 128, 0, s>>>(b, v);
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


// work must hold one partial per band of rows: ceil(ny/16) * nzl doubles
extern "C" cudaError_t hx_bp5_scatter_dot_impl(Box b, const double* yl, double* v, const double* p, int64_t n_owned,
                                               double* work, double* out, cudaStream_t s) {
  const dim3 grid = band_grid(b);
  if (band32_ok(b))
    hx::bp5::scatter_band32_kernel<<<grid, 256, 0, s>>>(b, yl, v, p, n_owned, work, 1);
  else if (b.order == 7)
    hx::bp5::scatter_band_kernel<7><<<grid, 256, 0, s>>>(b, yl, v, p, n_owned, work, 1);
  else
    hx::bp5::scatter_band_kernel<0><<<grid, 256, 0, s>>>(b, yl, v, p, n_owned, work, 1);
  hx::bp5::rows_final_kernel<<<1, 256, 0, s>>>(work, (int64_t)grid.x * grid.y, out);
  return cudaGetLastError();
}

extern "C" cudaError_t hx_cg_xr_dot_impl(const double* scal, double* x, const double* p, double* r,
                                         const double* ap, int64_t n, int64_t n_owned, double* work, double* out,
                                         cudaStream_t s) {
  hx::bp5::cg_xr_dot_kernel<<<hx::bp5::kDotBlocks, 256, 0, s>>>(scal, x, p, r, ap, n, n_owned, work);
  hx::bp5::dot_final_kernel<<<1, hx::bp5::kDotThreads, 0, s>>>(work, out);
  return cudaGetLastError();
}
