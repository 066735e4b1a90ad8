// Specialised AxLocal kernels (filled in by the optimisation rounds).
#include "hx_common.cuh"

extern "C" cudaError_t hx_fast_launch(const hx_axlocal_args* a, cudaStream_t s) {
  (void)a;
  (void)s;
  return cudaErrorNotSupported;
}

HX_DEFINE_UPLOAD_HOOK(hx_upload_basis_fast)
