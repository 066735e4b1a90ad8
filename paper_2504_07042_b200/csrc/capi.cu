// extern "C" entry points of libhx_axlocal.so (declared in include/hx_axlocal.h).
//
// Validation mirrors the reference's ValueError cases for the apply path
// (axlocal.py:67-81, 123-127, 238-243); geometry failures are reported through
// device-side "first bad index" words that the Python layer turns into
// GeometryError with the reference's messages.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "hx_common.cuh"

#define HX_VERSION_STRING "hx_axlocal 0.1.0 (sm_100a)"

extern "C" {
// per-order generic kernels (ax_generic.cu compiled with -DHX_N1=2..16)
#define HX_DECL_GENERIC(n)                                                                    \
  cudaError_t hx_generic_launch_##n(const hx_axlocal_args*, cudaStream_t);                   \
  cudaError_t hx_upload_basis_generic_##n(int, const double*, const double*, const double*);
HX_DECL_GENERIC(2)
HX_DECL_GENERIC(3)
HX_DECL_GENERIC(4)
HX_DECL_GENERIC(5)
HX_DECL_GENERIC(6)
HX_DECL_GENERIC(7)
HX_DECL_GENERIC(8)
HX_DECL_GENERIC(9)
HX_DECL_GENERIC(10)
HX_DECL_GENERIC(11)
HX_DECL_GENERIC(12)
HX_DECL_GENERIC(13)
HX_DECL_GENERIC(14)
HX_DECL_GENERIC(15)
HX_DECL_GENERIC(16)
#define HX_DECL_FASTN(n)                                                                      \
  cudaError_t hx_fastn_launch_##n(const hx_axlocal_args*, cudaStream_t);                     \
  cudaError_t hx_upload_basis_fastn_##n(int, const double*, const double*, const double*);
HX_DECL_FASTN(2)
HX_DECL_FASTN(3)
HX_DECL_FASTN(4)
HX_DECL_FASTN(5)
HX_DECL_FASTN(6)
HX_DECL_FASTN(7)
HX_DECL_FASTN(9)
HX_DECL_FASTN(10)
HX_DECL_FASTN(11)
HX_DECL_FASTN(12)
HX_DECL_FASTN(13)
HX_DECL_FASTN(14)
HX_DECL_FASTN(15)
HX_DECL_FASTN(16)
cudaError_t hx_low_launch_2(const hx_axlocal_args*, cudaStream_t);
cudaError_t hx_low_launch_3(const hx_axlocal_args*, cudaStream_t);
cudaError_t hx_upload_basis_low_2(int, const double*, const double*, const double*);
// j-plane kernels (ax_plane.cu) for orders 2, 3
cudaError_t hx_plane_launch_3(const hx_axlocal_args*, cudaStream_t);
cudaError_t hx_plane_launch_4(const hx_axlocal_args*, cudaStream_t);
cudaError_t hx_upload_basis_plane_3(int, const double*, const double*, const double*);
cudaError_t hx_upload_basis_plane_4(int, const double*, const double*, const double*);
cudaError_t hx_upload_basis_low_3(int, const double*, const double*, const double*);
cudaError_t hx_upload_basis_setup(int, const double*, const double*, const double*);
cudaError_t hx_upload_basis_fast(int, const double*, const double*, const double*);
// specialised kernels (ax_fast.cu): returns cudaErrorNotSupported when no
// specialised kernel covers the request.
cudaError_t hx_fast_launch(const hx_axlocal_args*, cudaStream_t);
// DMMA (mma.sync m8n8k4 f64) N = 7 kernel (ax_mma.cu); NotSupported outside its scope.
cudaError_t hx_mma_launch(const hx_axlocal_args*, cudaStream_t);
cudaError_t hx_upload_basis_mma(int, const double*, const double*, const double*);

cudaError_t hx_setup_trilinear_impl(int, int64_t, const double*, int, int64_t*, double*, double*, const double*,
                                    double, const double*, double, cudaStream_t);
cudaError_t hx_setup_stored_impl(int, int64_t, const double*, double*, double*, int64_t*, cudaStream_t);
cudaError_t hx_setup_ppd_impl(int64_t, const double*, double*, int64_t*, cudaStream_t);
cudaError_t hx_classify_impl(int64_t, const double*, int8_t*, cudaStream_t);
cudaError_t hx_bp5_gather_impl(hx_box, const double*, double*, cudaStream_t);
cudaError_t hx_bp5_scatter_impl(hx_box, const double*, double*, cudaStream_t);
cudaError_t hx_bp5_mask_impl(hx_box, double*, cudaStream_t);
cudaError_t hx_dot_impl(const double*, const double*, int64_t, int64_t, double*, double*, cudaStream_t);
cudaError_t hx_cg_xr_impl(const double*, double*, const double*, double*, const double*, int64_t, cudaStream_t);
cudaError_t hx_cg_p_impl(const double*, double*, const double*, int64_t, cudaStream_t);
cudaError_t hx_bp5_scatter_dot_impl(hx_box, const double*, double*, const double*, int64_t, double*, double*,
                                    cudaStream_t);
cudaError_t hx_cg_xr_dot_impl(const double*, double*, const double*, double*, const double*, int64_t, int64_t,
                              double*, double*, cudaStream_t);
}

namespace {

thread_local std::string g_last_error;

typedef cudaError_t (*generic_fn)(const hx_axlocal_args*, cudaStream_t);
typedef cudaError_t (*upload_fn)(int, const double*, const double*, const double*);

const generic_fn kGeneric[hx::kMaxN1 + 1] = {
    nullptr,
    nullptr,
    hx_generic_launch_2,
    hx_generic_launch_3,
    hx_generic_launch_4,
    hx_generic_launch_5,
    hx_generic_launch_6,
    hx_generic_launch_7,
    hx_generic_launch_8,
    hx_generic_launch_9,
    hx_generic_launch_10,
    hx_generic_launch_11,
    hx_generic_launch_12,
    hx_generic_launch_13,
    hx_generic_launch_14,
    hx_generic_launch_15,
    hx_generic_launch_16,
};

// order-generic fast kernels (ax_fastn.cu); n1 = 8 is served by ax_fast.cu
const generic_fn kFastN[hx::kMaxN1 + 1] = {
    nullptr,           nullptr,           hx_fastn_launch_2,  hx_fastn_launch_3,  hx_fastn_launch_4,
    hx_fastn_launch_5, hx_fastn_launch_6, hx_fastn_launch_7,  nullptr,            hx_fastn_launch_9,
    hx_fastn_launch_10, hx_fastn_launch_11, hx_fastn_launch_12, hx_fastn_launch_13, hx_fastn_launch_14,
    hx_fastn_launch_15, hx_fastn_launch_16,
};

const upload_fn kUploads[] = {
    hx_upload_basis_low_2,    hx_upload_basis_low_3,
    hx_upload_basis_fastn_2,  hx_upload_basis_fastn_3,  hx_upload_basis_fastn_4,  hx_upload_basis_fastn_5,
    hx_upload_basis_fastn_6,  hx_upload_basis_fastn_7,  hx_upload_basis_fastn_9,  hx_upload_basis_fastn_10,
    hx_upload_basis_fastn_11, hx_upload_basis_fastn_12, hx_upload_basis_fastn_13, hx_upload_basis_fastn_14,
    hx_upload_basis_fastn_15, hx_upload_basis_fastn_16,
    hx_upload_basis_generic_2,  hx_upload_basis_generic_3,  hx_upload_basis_generic_4,  hx_upload_basis_generic_5,
    hx_upload_basis_generic_6,  hx_upload_basis_generic_7,  hx_upload_basis_generic_8,  hx_upload_basis_generic_9,
    hx_upload_basis_generic_10, hx_upload_basis_generic_11, hx_upload_basis_generic_12, hx_upload_basis_generic_13,
    hx_upload_basis_generic_14, hx_upload_basis_generic_15, hx_upload_basis_generic_16, hx_upload_basis_setup,
    hx_upload_basis_fast,     hx_upload_basis_mma,     hx_upload_basis_plane_3,   hx_upload_basis_plane_4,
};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HX_OK;
  return fail(HX_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool order_ok(int order) { return order >= 1 && order + 1 <= hx::kMaxN1; }

// The library links the CUDA runtime statically, so its per-thread "current
// device" is not the host framework's (torch keeps its own runtime's).  Every
// entry point that takes device memory binds the device owning its first device
// pointer before launching, so a rank whose framework device is k launches on k.
int bind_device(const void* p) {
  if (!p) return HX_OK;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return HX_OK;
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return HX_OK;
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur == at.device) return HX_OK;
  return cuda_status(cudaSetDevice(at.device), "binding the device of the arguments");
}

}  // namespace

extern "C" int hx_set_device(int32_t device) {
  g_last_error.clear();
  return cuda_status(cudaSetDevice(device), "hx_set_device");
}

extern "C" const char* hx_version(void) { return HX_VERSION_STRING; }

extern "C" const char* hx_last_error(void) { return g_last_error.c_str(); }

extern "C" int hx_set_basis(int32_t order, const double* points, const double* weights, const double* dmat) {
  g_last_error.clear();
  if (!order_ok(order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (!points || !weights || !dmat) return fail(HX_ERR_INVALID, "hx_set_basis: null basis array");
  const int n1 = order + 1;
  for (upload_fn f : kUploads) {
    int st = cuda_status(f(n1, points, weights, dmat), "hx_set_basis");
    if (st) return st;
  }
  return cuda_status(cudaDeviceSynchronize(), "hx_set_basis");
}

// Nonzero hx_axlocal_args.reserved selects experimental kernel variants for the
// development A/B tools; it is honoured only with HX_TUNING=1 in the environment.
static bool tuning_enabled() {
  static const bool on = [] {
    const char* v = getenv("HX_TUNING");
    return v && v[0] && strcmp(v, "0") != 0;
  }();
  return on;
}

extern "C" int hx_axlocal(const hx_axlocal_args* a, void* stream) {
  g_last_error.clear();
  if (!a) return fail(HX_ERR_INVALID, "null args");
  if (a->reserved != 0 && !tuning_enabled())
    return fail(HX_ERR_INVALID, "hx_axlocal_args.reserved must be 0 (tuning hooks need HX_TUNING=1)");
  if (int st = bind_device(a->x)) return st;
  if (!order_ok(a->order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (a->n_col != 1 && a->n_col != 3) return fail(HX_ERR_INVALID, "n_col must be 1 or 3");
  if (a->equation != HX_POISSON && a->equation != HX_HELMHOLTZ) return fail(HX_ERR_INVALID, "bad equation");
  if (a->factor_source < HX_STORED || a->factor_source > HX_PARALLELEPIPED)
    return fail(HX_ERR_INVALID, "bad factor source");
  const bool helm = a->equation == HX_HELMHOLTZ;
  if (a->factor_source == HX_TRILINEAR_MERGED && !helm)
    return fail(HX_ERR_INVALID, "the merged-scalar variant exists for Helmholtz only");
  if (a->factor_source == HX_TRILINEAR_PARTIAL && helm)
    return fail(HX_ERR_INVALID, "the partial-recompute variant exists for Poisson only");
  if (a->n_elements < 0) return fail(HX_ERR_INVALID, "negative element count");
  if (a->n_elements == 0) return HX_OK;
  if (!a->x || !a->y) return fail(HX_ERR_INVALID, "null x or y");
  switch (a->factor_source) {
    case HX_STORED:
      if (!a->g || (helm && !a->gwj)) return fail(HX_ERR_INVALID, "stored factors missing");
      break;
    case HX_PARALLELEPIPED:
      if (!a->h) return fail(HX_ERR_INVALID, "parallelepiped constants missing");
      break;
    case HX_TRILINEAR:
      if (!a->verts) return fail(HX_ERR_INVALID, "vertices missing");
      break;
    case HX_TRILINEAR_MERGED:
      if (!a->verts || !a->lam2 || !a->lam3) return fail(HX_ERR_INVALID, "merged scalars missing");
      break;
    case HX_TRILINEAR_PARTIAL:
      if (!a->verts || !a->lam_geo) return fail(HX_ERR_INVALID, "partial lam_geo missing");
      break;
  }
  if (!helm && (a->lam0 || a->lam1))
    return fail(HX_ERR_INVALID, "coefficient fields apply to the Helmholtz operator only");
  if (a->gather) {
    const hx_box& b = a->gather_box;
    if (a->order != 7 || a->n_col != 1 || b.order != 7)
      return fail(HX_ERR_UNSUPPORTED, "fused lattice gather needs order 7 and n_col 1");
    if ((int64_t)b.ex * b.ey * b.nz_el != a->n_elements) return fail(HX_ERR_INVALID, "gather box / element mismatch");
    if (a->kernel == 1) return fail(HX_ERR_UNSUPPORTED, "fused lattice gather is not in the generic kernel");
  }
  if (a->cg_r) {
    if (!a->gather) return fail(HX_ERR_INVALID, "the fused CG update needs the fused lattice gather");
    if (!a->cg_scal || !a->cg_p_out) return fail(HX_ERR_INVALID, "fused CG update: null scalar / output");
    if (a->cg_p_out == a->x || a->cg_p_out == a->cg_r)
      return fail(HX_ERR_INVALID, "fused CG update: p_out must not alias p or r");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n1 = a->order + 1;
  // kernel 0 at orders 2 and 3: the j-plane kernel (ax_plane.cu) wherever it measures
  // faster -- every source but parallelepiped at order 2 (element per thread) and
  // stored at order 3 (order-generic); n_col 1 and 3 alike (profiles/r02_plane_ab.txt)
  const bool plane_default = a->kernel == 0 && !a->gather &&
                             ((n1 == 3 && a->factor_source != HX_PARALLELEPIPED) ||
                              (n1 == 4 && a->factor_source != HX_STORED));
  if (a->kernel == 5 || plane_default) {  // j-plane kernel (orders 2, 3)
    if (a->gather) return fail(HX_ERR_UNSUPPORTED, "fused lattice gather is not in the j-plane kernel");
    if (n1 == 3) return cuda_status(hx_plane_launch_3(a, s), "hx_axlocal(plane)");
    if (n1 == 4) return cuda_status(hx_plane_launch_4(a, s), "hx_axlocal(plane)");
    return fail(HX_ERR_UNSUPPORTED, "kernel 5 (j-plane) covers orders 2 and 3");
  }
  // kernel 0 at orders 1-2: the element-per-thread kernel wherever it measures fastest
  // (every source but stored; stored streams 6 factor fields per node and the
  // block-per-element kernels coalesce those better; profiles/r01_order_sweep.txt)
  const bool low_default = a->kernel == 0 && n1 <= 3 && !a->gather && a->factor_source != HX_STORED;
  if (a->kernel == 3 || low_default) {  // element-per-thread low-order kernel
    if (n1 > 3) return fail(HX_ERR_UNSUPPORTED, "kernel 3 (element per thread) covers orders 1 and 2");
    if (a->gather) return fail(HX_ERR_UNSUPPORTED, "fused lattice gather is not in the low-order kernel");
    return cuda_status(n1 == 2 ? hx_low_launch_2(a, s) : hx_low_launch_3(a, s), "hx_axlocal(low)");
  }
  // kernel 0 at order 7: the DMMA kernel (ax_mma.cu) for every factor source of
  // both equations but Helmholtz stored (nine per-node streams: ax8s / ax8c3
  // measure 12 % / 7 % faster), at n_col 1 and 3 alike, so that n_col = 3 stays
  // bitwise three n_col = 1 applies, and with the fused BP5 lattice gather, so
  // fused and unfused stay bitwise equal
  // (profiles/r02_n7_variants_c4.txt, r02_mma_stage_ab.txt, r02_mma_xstage_ab.txt)
  const bool helm_eq = a->equation == HX_HELMHOLTZ;
  const bool mma_default = a->kernel == 0 && a->order == 7 && !(helm_eq && a->factor_source == HX_STORED);
  if (a->kernel == 4 || mma_default) {  // DMMA kernel (order 7, element-local x)
    cudaError_t e = hx_mma_launch(a, s);
    if (e != cudaErrorNotSupported) return cuda_status(e, "hx_axlocal(mma)");
    (void)cudaGetLastError();
    if (a->kernel == 4)
      return fail(HX_ERR_UNSUPPORTED, "kernel 4 (DMMA) covers order 7 with element-local, 16-byte aligned x / y");
  }
  if (a->kernel != 1) {
    cudaError_t e = hx_fast_launch(a, s);  // specialised N = 7
    if (e != cudaErrorNotSupported) return cuda_status(e, "hx_axlocal(fast)");
    (void)cudaGetLastError();
    // only the N = 7 kernels read the lattice; never fall through to an
    // element-local kernel with a lattice x (out-of-bounds reads)
    if (a->gather)
      return fail(HX_ERR_UNSUPPORTED,
                  "fused lattice gather: no kernel for this request (the ax8s gather path needs 16-byte "
                  "aligned x and vertices)");
    // kernel 0 keeps the slice kernel where it measures faster (stored at order 1;
    // the fused-gather path at orders 1-2; profiles/r01_order_sweep.txt)
    const bool tri = a->factor_source == HX_TRILINEAR || a->factor_source == HX_TRILINEAR_PARTIAL ||
                     a->factor_source == HX_TRILINEAR_MERGED;
    const bool slice_wins = a->order == 1 || (a->order == 2 && tri);
    if (kFastN[n1] && !a->gather && (a->kernel == 2 || !slice_wins))
      return cuda_status(kFastN[n1](a, s), "hx_axlocal(fastn)");
  }
  if (n1 < 2) {
    // order must be >= 1 so n1 >= 2 always; kept for clarity
    return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  }
  return cuda_status(kGeneric[n1](a, s), "hx_axlocal(generic)");
}

extern "C" int hx_trilinear_validate(int32_t order, int64_t E, const double* verts, int64_t* first_bad,
                                     void* stream) {
  g_last_error.clear();
  if (int st = bind_device(verts)) return st;
  if (!order_ok(order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (!verts || !first_bad) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_setup_trilinear_impl(order + 1, E, verts, 0, first_bad, nullptr, nullptr, nullptr, 1.0,
                                             nullptr, 1.0, static_cast<cudaStream_t>(stream)),
                     "hx_trilinear_validate");
}

extern "C" int hx_setup_partial(int32_t order, int64_t E, const double* verts, double* lam_geo, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(verts)) return st;
  if (!order_ok(order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (!verts || !lam_geo) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_setup_trilinear_impl(order + 1, E, verts, 1, nullptr, lam_geo, nullptr, nullptr, 1.0,
                                             nullptr, 1.0, static_cast<cudaStream_t>(stream)),
                     "hx_setup_partial");
}

extern "C" int hx_setup_merged(int32_t order, int64_t E, const double* verts, const double* lam0, double l0v,
                               const double* lam1, double l1v, double* lam2, double* lam3, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(verts)) return st;
  if (!order_ok(order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (!verts || !lam2 || !lam3) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_setup_trilinear_impl(order + 1, E, verts, 2, nullptr, lam2, lam3, lam0, l0v, lam1, l1v,
                                             static_cast<cudaStream_t>(stream)),
                     "hx_setup_merged");
}

extern "C" int hx_setup_stored(int32_t order, int64_t E, const double* verts, double* g, double* gwj,
                               int64_t* first_bad, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(verts)) return st;
  if (!order_ok(order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (!verts || !g || !first_bad) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(
      hx_setup_stored_impl(order + 1, E, verts, g, gwj, first_bad, static_cast<cudaStream_t>(stream)),
      "hx_setup_stored");
}

extern "C" int hx_setup_parallelepiped(int64_t E, const double* verts, double* h, int64_t* bad, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(verts)) return st;
  if (!verts || !h || !bad) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_setup_ppd_impl(E, verts, h, bad, static_cast<cudaStream_t>(stream)),
                     "hx_setup_parallelepiped");
}

extern "C" int hx_classify_elements(int64_t E, const double* verts, int8_t* kind, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(verts)) return st;
  if (!verts || !kind) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_classify_impl(E, verts, kind, static_cast<cudaStream_t>(stream)), "hx_classify_elements");
}

namespace {
int box_ok(const hx_box* b) {
  if (!b) return fail(HX_ERR_INVALID, "null box");
  if (!order_ok(b->order)) return fail(HX_ERR_UNSUPPORTED, "order must be in 1..15");
  if (b->ex < 1 || b->ey < 1 || b->nz_el < 1 || b->ez < 1 || b->z0 < 0 || b->z0 + b->nz_el > b->ez)
    return fail(HX_ERR_INVALID, "bad box / slab extents");
  // lattice coordinates and slab element indices are 32-bit in the BP5 kernels
  if ((int64_t)b->ex * b->ey * b->nz_el > 0x7fffffffLL || (int64_t)b->ex * b->order + 1 > 0x7fffffffLL ||
      (int64_t)b->ey * b->order + 1 > 0x7fffffffLL || (int64_t)b->ez * b->order + 1 > 0x7fffffffLL)
    return fail(HX_ERR_UNSUPPORTED, "box too large for 32-bit element / lattice indices");
  if ((b->n_col != 1 && b->n_col != 3) || b->col < 0 || b->col >= b->n_col)
    return fail(HX_ERR_INVALID, "bad column selection");
  // lattice rows / planes of the slab index grid.y / grid.z of the row and band kernels
  if ((int64_t)b->ey * b->order + 1 > 65535 || (int64_t)b->nz_el * b->order + 1 > 65535)
    return fail(HX_ERR_UNSUPPORTED, "slab too large: at most 65535 lattice rows along y and planes along z");
  return HX_OK;
}
}  // namespace

extern "C" int hx_bp5_gather(const hx_box* box, const double* u, double* xl, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(u)) return st;
  if (int st = box_ok(box)) return st;
  if (!u || !xl) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_bp5_gather_impl(*box, u, xl, static_cast<cudaStream_t>(stream)), "hx_bp5_gather");
}

extern "C" int hx_bp5_scatter_add(const hx_box* box, const double* yl, double* v, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(yl)) return st;
  if (int st = box_ok(box)) return st;
  if (!yl || !v) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_bp5_scatter_impl(*box, yl, v, static_cast<cudaStream_t>(stream)), "hx_bp5_scatter_add");
}

extern "C" int hx_bp5_mask(const hx_box* box, double* v, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(v)) return st;
  if (int st = box_ok(box)) return st;
  if (!v) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_bp5_mask_impl(*box, v, static_cast<cudaStream_t>(stream)), "hx_bp5_mask");
}

extern "C" int hx_dot(const double* a, const double* b, int64_t lo, int64_t hi, double* work, double* out,
                      void* stream) {
  g_last_error.clear();
  if (int st = bind_device(a)) return st;
  if (!a || !b || !work || !out) return fail(HX_ERR_INVALID, "null pointer");
  if (lo < 0 || hi < lo) return fail(HX_ERR_INVALID, "bad range");
  return cuda_status(hx_dot_impl(a, b, lo, hi, work, out, static_cast<cudaStream_t>(stream)), "hx_dot");
}

extern "C" int hx_cg_update_xr(const double* scal, double* x, const double* p, double* r, const double* ap,
                               int64_t n, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(x)) return st;
  if (!scal || !x || !p || !r || !ap || n < 0) return fail(HX_ERR_INVALID, "bad arguments");
  return cuda_status(hx_cg_xr_impl(scal, x, p, r, ap, n, static_cast<cudaStream_t>(stream)), "hx_cg_update_xr");
}

extern "C" int hx_cg_update_p(const double* scal, double* p, const double* r, int64_t n, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(p)) return st;
  if (!scal || !p || !r || n < 0) return fail(HX_ERR_INVALID, "bad arguments");
  return cuda_status(hx_cg_p_impl(scal, p, r, n, static_cast<cudaStream_t>(stream)), "hx_cg_update_p");
}

extern "C" int hx_bp5_scatter_dot(const hx_box* box, const double* yl, double* v, const double* p, int64_t n_owned,
                                  double* work, double* out, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(yl)) return st;
  if (int st = box_ok(box)) return st;
  if (!yl || !v || !p || !work || !out) return fail(HX_ERR_INVALID, "null pointer");
  return cuda_status(hx_bp5_scatter_dot_impl(*box, yl, v, p, n_owned, work, out, static_cast<cudaStream_t>(stream)),
                     "hx_bp5_scatter_dot");
}

extern "C" int hx_cg_update_xr_dot(const double* scal, double* x, const double* p, double* r, const double* ap,
                                   int64_t n, int64_t n_owned, double* work, double* out, void* stream) {
  g_last_error.clear();
  if (int st = bind_device(x)) return st;
  if (!scal || !x || !p || !r || !ap || !work || !out || n < 0 || n_owned > n) return fail(HX_ERR_INVALID, "bad arguments");
  return cuda_status(hx_cg_xr_dot_impl(scal, x, p, r, ap, n, n_owned, work, out, static_cast<cudaStream_t>(stream)),
                     "hx_cg_update_xr_dot");
}
