/*
 * hx_axlocal.h — C ABI of the B200-native AxLocal (CEED BK5) library.
 *
 * Drop-in boundary for the reference's element-local operator
 * (hosfem, pkg/src/hosfem/axlocal.py).  The reference is a Python class API,
 * not an FFI; each entry point below replaces one piece of it and is bound
 * from Python with ctypes (see INTEGRATION.md for the stub).
 *
 * Conventions (all match the reference):
 *   - fp64 everywhere; node (i,j,k) of an element is flat i + j*n1 + k*n1*n1;
 *   - fields x, y are (E, n1^3, n_col) row-major, n_col innermost
 *     (LocalField, mesh.py:140-155);
 *   - vertices are (E, 8, 3), vertex b at reference corner bits (r,s,t);
 *   - stored factors are SoA (E, 6, n1^3) in the order g00 g01 g02 g11 g12 g22
 *     (the reference keeps AoS (E, n1^3, 6), geometry.py:264-275);
 *   - every pointer in an hx_* call is a DEVICE pointer owned by the caller
 *     (torch), except hx_set_basis's host arrays; nothing here allocates;
 *   - calls are stream-ordered on the given cudaStream_t (passed as void*),
 *     and never synchronise except where documented;
 *   - no C++ exception crosses this boundary; every call returns an hx_status
 *     and hx_last_error() describes the last failure on the calling thread.
 */
#ifndef HX_AXLOCAL_H
#define HX_AXLOCAL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HX_OK = 0,
  HX_ERR_INVALID = 1,     /* maps to ValueError (axlocal.py:68-81, 123-127, 238-243) */
  HX_ERR_GEOMETRY = 2,    /* maps to GeometryError (geometry.py:64-65, 243-247, 344-346) */
  HX_ERR_CUDA = 3,        /* launch / runtime failure */
  HX_ERR_UNSUPPORTED = 4  /* order outside 1..15 etc. */
} hx_status;

/* Equation (axlocal.py:45-47). */
typedef enum { HX_POISSON = 0, HX_HELMHOLTZ = 1 } hx_equation;

/* FactorSource (axlocal.py:50-55). */
typedef enum {
  HX_STORED = 0,
  HX_TRILINEAR = 1,
  HX_TRILINEAR_MERGED = 2,
  HX_TRILINEAR_PARTIAL = 3,
  HX_PARALLELEPIPED = 4
} hx_factor_source;

/* ------------------------------------------------------------------------
 * BP5 / Nekbone CG proxy on a structured box (reference solver.py:64-308).
 * A rank owns element z-layers [z0, z0+nz_el) of an ex x ey x ez box of
 * order N; its global vectors are the slab lattice
 * (ex*N+1) x (ey*N+1) x (nz_el*N+1), x fastest (mesh.py:271-274 numbering
 * restricted to the slab, both interface planes included).
 */
typedef struct {
  int32_t order;  /* N */
  int32_t ex, ey; /* elements along x and y */
  int32_t nz_el;  /* element layers in this slab */
  int32_t z0;     /* first global element layer of the slab */
  int32_t ez;     /* global element layers (physical boundary at 0 and ez*N) */
  int32_t n_col;  /* columns of the element-local array (1 or 3) */
  int32_t col;    /* which column gather writes / scatter-add reads */
} hx_box;

/*
 * Arguments of one apply.  Replaces LocalOperator.apply/_apply_range/_factor_stage
 * (axlocal.py:171-258): y = A x for all E elements of the operator.
 * Which factor pointers must be non-NULL depends on (equation, source):
 *   STORED              g (E,6,n1^3) SoA;  Helmholtz: gwj (E,n1^3)
 *   TRILINEAR           verts (E,8,3)
 *   TRILINEAR_PARTIAL   verts, lam_geo (E,n1^3)       [Poisson only]
 *   TRILINEAR_MERGED    verts, lam2, lam3 (E,n1^3)    [Helmholtz only]
 *   PARALLELEPIPED      h (E,7)
 * Helmholtz coefficients (all but MERGED): lam0 / lam1 (E,n1^3) device fields,
 * or NULL to use the scalar lam0_value / lam1_value for every node
 * (_coeff_field, axlocal.py:88-101; None means 1).
 */
typedef struct {
  int32_t order;          /* N, 1..15 */
  int32_t n_col;          /* 1 or 3 */
  int32_t equation;       /* hx_equation */
  int32_t factor_source;  /* hx_factor_source */
  int64_t n_elements;     /* E >= 0 (0 is a no-op) */
  const double* x;
  double* y;
  const double* verts;
  const double* h;
  const double* g;
  const double* gwj;
  const double* lam_geo;
  const double* lam2;
  const double* lam3;
  const double* lam0;
  const double* lam1;
  double lam0_value;
  double lam1_value;
  int32_t kernel;         /* 0 = best measured kernel for (order, factor source);
                             1 = slice kernel (paper Algorithm 4, every order);
                             2 = fast kernel (specialised N=7 ax8s / ax8c3, else order-generic);
                             3 = element-per-thread kernel (orders 1, 2 only);
                             4 = DMMA kernel (order 7 only: r/s contractions on
                                 mma.sync m8n8k4 f64, ax_mma.cu; the kernel-0
                                 choice at order 7 for every source and equation
                                 but Helmholtz stored);
                             5 = j-plane kernel (orders 2, 3: one thread per
                                 j-plane, s direction by warp shuffles, ax_plane.cu) */
  int32_t reserved;       /* must be 0: nonzero values select experimental kernel
                             variants for the A/B tools and are rejected
                             (HX_ERR_INVALID) unless HX_TUNING=1 is set */
  /* Optional fused gather (BP5): when gather != 0, x is NOT element-local but
   * the slab lattice vector of gather_box and each element reads its nodes
   * straight from it (Q u, mesh.py:286-294).  Order 7, n_col 1, and the
   * elements must be the box's slab in its element order. */
  int32_t gather;
  int32_t reserved2;
  hx_box gather_box;
  /* Optional fused CG direction update (BP5, requires gather): when cg_r != NULL the
   * apply first forms p = r + (cg_scal[2] / cg_scal[0]) * x on the lattice, with
   * the rounding of the standalone update (solver.py:170), writes it to cg_p_out
   * (a different lattice vector than x) and applies A to it. */
  const double* cg_r;
  const double* cg_scal;
  double* cg_p_out;
} hx_axlocal_args;

/* Library version string. */
const char* hx_version(void);

/* Human-readable description of the last error on this thread ("" if none). */
const char* hx_last_error(void);

/*
 * Make `device` the current device of the library's (statically linked) CUDA
 * runtime for this thread.  Needed before hx_set_basis, whose arguments are host
 * arrays; every other entry point binds the device owning its first device
 * pointer itself.
 */
int hx_set_device(int32_t device);

/*
 * Upload the GLL basis of one order to the current device's __constant__ bank.
 * points (n1), weights (n1), dmat (n1*n1 row-major, [i][j] = l_j'(x_i)) are HOST
 * arrays from SpectralBasis.build (basis.py:110-136).  Synchronous.  Must be
 * called once per (device, order) before any other call with that order.
 */
int hx_set_basis(int32_t order, const double* points, const double* weights, const double* dmat);

/* y = A x.  Replaces LocalOperator.apply (axlocal.py:235-258). */
int hx_axlocal(const hx_axlocal_args* args, void* stream);

/*
 * Degenerate-geometry check of the trilinear route over all GLL nodes
 * (trilinear_factors(validate=True), geometry.py:342-346, run once in
 * LocalOperator.__init__, axlocal.py:156).  Writes into *first_bad_out (device,
 * int64) the smallest flat index e*n1^3 + node with det(8J) <= 0, or INT64_MAX
 * when every node is valid.  The call initialises *first_bad_out itself
 * (stream-ordered); the caller reads it back after the stream reaches it.
 */
int hx_trilinear_validate(int32_t order, int64_t n_elements, const double* verts,
                          int64_t* first_bad_out, void* stream);

/* lam_geo = 0.125 w / det(8J) per node (partial_recompute_setup, geometry.py:414-424). */
int hx_setup_partial(int32_t order, int64_t n_elements, const double* verts, double* lam_geo_out,
                     void* stream);

/*
 * lam2 = lam_geo * lam0, lam3 = (lam_geo * det(8J)^2/64) * lam1
 * (merged_scalar_setup, geometry.py:401-411, as called at axlocal.py:159-165).
 * lam0/lam1 may be NULL to use the scalar values.
 */
int hx_setup_merged(int32_t order, int64_t n_elements, const double* verts, const double* lam0,
                    double lam0_value, const double* lam1, double lam1_value, double* lam2_out,
                    double* lam3_out, void* stream);

/*
 * Stored (Nek-style) factors through the general route: nodal coordinates of
 * the trilinear map, collocation Jacobian by D contractions, w|J| J^-1 J^-T
 * (element_node_coords + discrete_jacobians + factors_from_jacobians,
 * mesh.py:130-137, geometry.py:225-276).  g_out SoA (E,6,n1^3); gwj_out
 * (E,n1^3) may be NULL.  *first_bad_out as in hx_trilinear_validate.
 */
int hx_setup_stored(int32_t order, int64_t n_elements, const double* verts, double* g_out,
                    double* gwj_out, int64_t* first_bad_out, void* stream);

/*
 * Parallelepiped constants h (E,7) = (det J^-1 J^-T sym6, det) with
 * J = (v1-v0 | v2-v0 | v4-v0)/2 (parallelepiped_setup, geometry.py:362-380).
 * *bad_out (device int64) receives 2*e + 0 for the smallest element e whose
 * vertices fail the parallelepiped identities (defect > 1e-10 * scale), or
 * 2*e + 1 when its det <= 0 (whichever e is smaller), else INT64_MAX.
 */
int hx_setup_parallelepiped(int64_t n_elements, const double* verts, double* h_out, int64_t* bad_out,
                            void* stream);

/*
 * Element classification (make_element, mesh.py:97-107): kind_out[e] = 1 when
 * the defect is <= 1e-12 * max(1, max|v|) (parallelepiped), else 0 (trilinear).
 */
int hx_classify_elements(int64_t n_elements, const double* verts, int8_t* kind_out, void* stream);



/* xl[:, :, col] (E_slab, n1^3, n_col) = Q u: copy lattice values to element-local
 * storage (gather, mesh.py:286-294); the lattice index is computed, not loaded. */
int hx_bp5_gather(const hx_box* box, const double* u, double* xl, void* stream);

/* v = Q^T yl[:, :, col] on the slab lattice (scatter_add, mesh.py:297-313): owner-computes,
 * each node sums its element copies in ascending element index, the
 * np.bincount order; interface planes hold this slab's partial sums. */
int hx_bp5_scatter_add(const hx_box* box, const double* yl, double* v, void* stream);

/* v = 0 on the physical boundary of the box (boundary_node_mask, mesh.py:316-335). */
int hx_bp5_mask(const hx_box* box, double* v, void* stream);

/* Fused CG step pieces:
 *  hx_bp5_scatter_dot: v = mask(Q^T yl) and *out = sum_{i < n_owned} p[i] v[i]
 *    (the pap of solver.py:152-153; v = ap);
 *  hx_cg_update_xr_dot: x += (rr/pap) p, r -= (rr/pap) ap and *out = sum_{i < n_owned} r[i]^2.
 * Both reduce in a fixed tree; work holds >= 1184 doubles for hx_cg_update_xr_dot and
 * ceil((ey*N+1)/16) * (nz_el*N+1) doubles (one per band of 16 lattice rows)
 * for hx_bp5_scatter_dot. */
int hx_bp5_scatter_dot(const hx_box* box, const double* yl, double* v, const double* p, int64_t n_owned,
                       double* work, double* out, void* stream);
int hx_cg_update_xr_dot(const double* scal, double* x, const double* p, double* r, const double* ap, int64_t n,
                        int64_t n_owned, double* work, double* out, void* stream);

/* *out = sum_{lo <= i < hi} a[i] b[i] on the device, fixed reduction tree
 * (bitwise reproducible); work holds >= 1184 doubles. */
int hx_dot(const double* a, const double* b, int64_t lo, int64_t hi, double* work, double* out, void* stream);

/* CG updates (solver.py:158-170) with device scalars scal = {rr, pap, rr_new}:
 * x += (rr/pap) p, r -= (rr/pap) ap  — and —  p = r + (rr_new/rr) p. */
int hx_cg_update_xr(const double* scal, double* x, const double* p, double* r, const double* ap, int64_t n,
                    void* stream);
int hx_cg_update_p(const double* scal, double* p, const double* r, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HX_AXLOCAL_H */
