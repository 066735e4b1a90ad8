"""ctypes binding of the in-tree C-ABI library ``_lib/libhx_axlocal.so``.

The library is the product: there is no CPU fallback.  Loading fails loudly
when the shared object is missing (run ``make`` or ``__graft_entry__.build()``),
and every call that returns a non-zero ``hx_status`` raises: HX_ERR_INVALID and
HX_ERR_UNSUPPORTED as ``ValueError`` (like the reference's validation,
axlocal.py:67-81), HX_ERR_CUDA as ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

__all__ = ["lib", "AxArgs", "Box", "check", "LIB_PATH", "SYMBOLS"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libhx_axlocal.so")

#: Every entry point declared in include/hx_axlocal.h.
SYMBOLS = (
    "hx_version",
    "hx_last_error",
    "hx_set_device",
    "hx_set_basis",
    "hx_axlocal",
    "hx_trilinear_validate",
    "hx_setup_partial",
    "hx_setup_merged",
    "hx_setup_stored",
    "hx_setup_parallelepiped",
    "hx_classify_elements",
    "hx_bp5_gather",
    "hx_bp5_scatter_add",
    "hx_bp5_mask",
    "hx_dot",
    "hx_cg_update_xr",
    "hx_cg_update_p",
    "hx_bp5_scatter_dot",
    "hx_cg_update_xr_dot",
)

HX_OK, HX_ERR_INVALID, HX_ERR_GEOMETRY, HX_ERR_CUDA, HX_ERR_UNSUPPORTED = range(5)

_c_p = ctypes.c_void_p
_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class Box(ctypes.Structure):
    """Mirror of ``hx_box`` (include/hx_axlocal.h)."""

    _fields_ = [("order", _i32), ("ex", _i32), ("ey", _i32), ("nz_el", _i32), ("z0", _i32), ("ez", _i32),
                ("n_col", _i32), ("col", _i32)]


class AxArgs(ctypes.Structure):
    """Mirror of ``hx_axlocal_args`` (include/hx_axlocal.h)."""

    _fields_ = [
        ("order", _i32),
        ("n_col", _i32),
        ("equation", _i32),
        ("factor_source", _i32),
        ("n_elements", _i64),
        ("x", _c_p),
        ("y", _c_p),
        ("verts", _c_p),
        ("h", _c_p),
        ("g", _c_p),
        ("gwj", _c_p),
        ("lam_geo", _c_p),
        ("lam2", _c_p),
        ("lam3", _c_p),
        ("lam0", _c_p),
        ("lam1", _c_p),
        ("lam0_value", _f64),
        ("lam1_value", _f64),
        ("kernel", _i32),
        ("reserved", _i32),
        ("gather", _i32),
        ("reserved2", _i32),
        ("gather_box", Box),
        ("cg_r", _c_p),
        ("cg_scal", _c_p),
        ("cg_p_out", _c_p),
    ]


_lock = threading.Lock()
_lib = None


def _load():
    # HX_AXLOCAL_LIB: an alternative build of the same library (tuning experiments, tools/tune_fastn.sh)
    path = os.environ.get("HX_AXLOCAL_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"CUDA library {path} is missing; build it with `make -j` (or __graft_entry__.build()). "
            "There is no CPU fallback."
        )
    so = ctypes.CDLL(path)
    so.hx_version.restype = ctypes.c_char_p
    so.hx_version.argtypes = []
    so.hx_last_error.restype = ctypes.c_char_p
    so.hx_last_error.argtypes = []
    so.hx_set_device.restype = ctypes.c_int
    so.hx_set_device.argtypes = [_i32]
    so.hx_set_basis.restype = ctypes.c_int
    so.hx_set_basis.argtypes = [_i32, _c_p, _c_p, _c_p]
    so.hx_axlocal.restype = ctypes.c_int
    so.hx_axlocal.argtypes = [ctypes.POINTER(AxArgs), _c_p]
    so.hx_trilinear_validate.restype = ctypes.c_int
    so.hx_trilinear_validate.argtypes = [_i32, _i64, _c_p, _c_p, _c_p]
    so.hx_setup_partial.restype = ctypes.c_int
    so.hx_setup_partial.argtypes = [_i32, _i64, _c_p, _c_p, _c_p]
    so.hx_setup_merged.restype = ctypes.c_int
    so.hx_setup_merged.argtypes = [_i32, _i64, _c_p, _c_p, _f64, _c_p, _f64, _c_p, _c_p, _c_p]
    so.hx_setup_stored.restype = ctypes.c_int
    so.hx_setup_stored.argtypes = [_i32, _i64, _c_p, _c_p, _c_p, _c_p, _c_p]
    so.hx_setup_parallelepiped.restype = ctypes.c_int
    so.hx_setup_parallelepiped.argtypes = [_i64, _c_p, _c_p, _c_p, _c_p]
    so.hx_classify_elements.restype = ctypes.c_int
    so.hx_classify_elements.argtypes = [_i64, _c_p, _c_p, _c_p]
    bp = ctypes.POINTER(Box)
    for name, args in (
        ("hx_bp5_gather", [bp, _c_p, _c_p, _c_p]),
        ("hx_bp5_scatter_add", [bp, _c_p, _c_p, _c_p]),
        ("hx_bp5_mask", [bp, _c_p, _c_p]),
        ("hx_dot", [_c_p, _c_p, _i64, _i64, _c_p, _c_p, _c_p]),
        ("hx_cg_update_xr", [_c_p, _c_p, _c_p, _c_p, _c_p, _i64, _c_p]),
        ("hx_cg_update_p", [_c_p, _c_p, _c_p, _i64, _c_p]),
        ("hx_bp5_scatter_dot", [bp, _c_p, _c_p, _c_p, _i64, _c_p, _c_p, _c_p]),
        ("hx_cg_update_xr_dot", [_c_p, _c_p, _c_p, _c_p, _c_p, _i64, _i64, _c_p, _c_p, _c_p]),
    ):
        fn = getattr(so, name)
        fn.restype = ctypes.c_int
        fn.argtypes = args
    return so


def lib():
    """The loaded library (loaded once per process)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = _load()
    return _lib


def check(status: int) -> None:
    if status == HX_OK:
        return
    msg = lib().hx_last_error().decode(errors="replace")
    if status in (HX_ERR_INVALID, HX_ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(f"hx_axlocal library error {status}: {msg}")
