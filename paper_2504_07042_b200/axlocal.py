"""B200 AxLocal operator: drop-in for ``hosfem.axlocal`` (reference pkg/src/hosfem/axlocal.py).

Same public surface — ``Equation``, ``FactorSource``, ``KernelSpec``,
``LocalOperator(spec, elements, basis, lam0=None, lam1=None)`` with
``.apply(x, threads=1)``, and ``ax_local_apply`` — with the same validation
and error types (axlocal.py:67-81, 123-169, 238-243).  Setup and apply run as
hand-written sm_100a kernels in ``_lib/libhx_axlocal.so`` (C ABI in
``include/hx_axlocal.h``); there is no CPU fallback.

Inputs beyond the reference's:
* ``elements`` may also be a ``BoxMesh``, a ``Mesh`` (e.g. from ``load_mesh``),
  or an (E, 8, 3) fp64 array / torch tensor of vertices (kinds then classified
  on the GPU with make_element's rule);
* ``apply`` also takes an (E, n1^3, n_col) or (E, n1^3) fp64 CUDA tensor and then
  returns a CUDA tensor (no host round trip); ``apply_(x, y)`` writes into a
  preallocated output.  A host ``LocalField`` in gives a host ``LocalField`` out
  (copied through pinned memory).
``threads`` is accepted for signature compatibility and ignored: the element
split is the CUDA grid, and results are bitwise independent of it.
"""

from __future__ import annotations

import ctypes
import os
import enum
from dataclasses import dataclass

import numpy as np

from . import _native
from .mesh import BoxMesh, Element, ElementKind, LocalField, Mesh

__all__ = [
    "Equation",
    "FactorSource",
    "KernelSpec",
    "LocalOperator",
    "ax_local_apply",
    "dense_local_matrix",
    "GeometryError",
]


class GeometryError(ValueError):
    """Degenerate or inconsistent element geometry (geometry.py:64-65)."""


class Equation(enum.Enum):
    POISSON = "poisson"
    HELMHOLTZ = "helmholtz"


class FactorSource(enum.Enum):
    STORED = "stored"
    TRILINEAR_RECOMPUTE = "trilinear"
    TRILINEAR_MERGED = "trilinear-merged"
    TRILINEAR_PARTIAL = "trilinear-partial"
    PARALLELEPIPED_RECOMPUTE = "parallelepiped"


_HX_SOURCE = {
    FactorSource.STORED: 0,
    FactorSource.TRILINEAR_RECOMPUTE: 1,
    FactorSource.TRILINEAR_MERGED: 2,
    FactorSource.TRILINEAR_PARTIAL: 3,
    FactorSource.PARALLELEPIPED_RECOMPUTE: 4,
}


def _coerce_enum(cls, value):
    if isinstance(value, cls):
        return value
    # accept the reference's own enum members (same values) and plain strings
    return cls(getattr(value, "value", value))


def _as_spec(spec):
    """This package's KernelSpec from ours, the reference's (same fields, its own
    enums) or a (equation, n_col, factor_source, order) tuple."""
    if isinstance(spec, KernelSpec):
        return spec
    if isinstance(spec, tuple):
        return KernelSpec(*spec)
    return KernelSpec(spec.equation, spec.n_col, spec.factor_source, spec.order)


@dataclass(frozen=True)
class KernelSpec:
    """What to apply: equation, columns, factor variant, order (axlocal.py:58-85)."""

    equation: Equation
    n_col: int
    factor_source: FactorSource
    order: int

    def __post_init__(self):
        object.__setattr__(self, "equation", _coerce_enum(Equation, self.equation))
        object.__setattr__(self, "factor_source", _coerce_enum(FactorSource, self.factor_source))
        if self.n_col not in (1, 3):
            raise ValueError("n_col must be 1 or 3")
        if self.order < 1:
            raise ValueError("order must be at least 1")
        if self.factor_source is FactorSource.TRILINEAR_MERGED and self.equation is not Equation.HELMHOLTZ:
            raise ValueError("the merged-scalar variant exists for Helmholtz only")
        if self.factor_source is FactorSource.TRILINEAR_PARTIAL and self.equation is not Equation.POISSON:
            raise ValueError("the partial-recompute variant exists for Poisson only")

    @property
    def n1(self) -> int:
        return self.order + 1


def _torch():
    import torch

    return torch


_BASIS_UPLOADED: set = set()


def _ensure_basis(device_index: int, basis) -> None:
    key = (device_index, int(basis.order))
    if key in _BASIS_UPLOADED:
        return
    torch = _torch()
    pts = np.ascontiguousarray(basis.points, dtype=np.float64)
    wts = np.ascontiguousarray(basis.weights, dtype=np.float64)
    dm = np.ascontiguousarray(basis.diff_matrix, dtype=np.float64)
    with torch.cuda.device(device_index):
        _native.check(_native.lib().hx_set_device(int(device_index)))
        _native.check(
            _native.lib().hx_set_basis(
                int(basis.order), pts.ctypes.data, wts.ctypes.data, dm.ctypes.data
            )
        )
    _BASIS_UPLOADED.add(key)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device):
    return ctypes.c_void_p(_torch().cuda.current_stream(device).cuda_stream)


def _read_i64(t) -> int:
    return int(t.item())


class LocalOperator:
    """Batched Y = A X over a fixed element set on one GPU (axlocal.py:107-258)."""

    def __init__(self, spec: KernelSpec, elements, basis, lam0=None, lam1=None, device=None):
        torch = _torch()
        spec = _as_spec(spec)
        if not torch.cuda.is_available():
            raise RuntimeError("LocalOperator needs a CUDA device (B200); there is no CPU fallback")
        if basis.order != spec.order:
            raise ValueError("basis order does not match the kernel spec")
        self.spec = spec
        self.basis = basis
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        dev = self.device
        n1 = basis.n1
        n3 = n1**3
        helm = spec.equation is Equation.HELMHOLTZ
        if not helm and (lam0 is not None or lam1 is not None):
            raise ValueError("coefficient fields apply to the Helmholtz operator only")

        verts, kinds = self._vertices(elements, dev)
        self.n_elements = int(verts.shape[0])
        if self.n_elements == 0:
            raise ValueError("need at least one element")
        self._verts = verts
        _ensure_basis(dev.index, basis)
        source = spec.factor_source
        E = self.n_elements
        stream = _stream(dev)
        L = _native.lib()
        self._h = self._g = self._gwj = self._lam_geo = self._lam2 = self._lam3 = None

        kinds = kinds if kinds is not None else self._classify(verts, stream)
        if source is FactorSource.PARALLELEPIPED_RECOMPUTE:
            if kinds - {ElementKind.PARALLELEPIPED}:
                raise ValueError("parallelepiped recompute needs an all-parallelepiped element set")
            self._h = torch.empty((E, 7), dtype=torch.float64, device=dev)
            bad = torch.empty((1,), dtype=torch.int64, device=dev)
            _native.check(L.hx_setup_parallelepiped(E, _ptr(verts), _ptr(self._h), _ptr(bad), stream))
            b = _read_i64(bad)
            if b != np.iinfo(np.int64).max:
                if b % 2 == 0:
                    raise GeometryError("vertices do not form a parallelepiped")
                raise GeometryError("degenerate parallelepiped (det <= 0)")
        elif source is FactorSource.STORED:
            self._g = torch.empty((E, 6, n3), dtype=torch.float64, device=dev)
            self._gwj = torch.empty((E, n3), dtype=torch.float64, device=dev) if helm else None
            bad = torch.empty((1,), dtype=torch.int64, device=dev)
            _native.check(
                L.hx_setup_stored(spec.order, E, _ptr(verts), _ptr(self._g), _ptr(self._gwj), _ptr(bad), stream)
            )
            b = _read_i64(bad)
            if b != np.iinfo(np.int64).max:
                raise GeometryError(f"non-positive Jacobian determinant at element {b // n3}, node {b % n3}")
        else:
            if kinds - {ElementKind.TRILINEAR, ElementKind.PARALLELEPIPED}:
                raise ValueError("trilinear recompute variants need trilinear elements")
            bad = torch.empty((1,), dtype=torch.int64, device=dev)
            _native.check(L.hx_trilinear_validate(spec.order, E, _ptr(verts), _ptr(bad), stream))
            b = _read_i64(bad)
            if b != np.iinfo(np.int64).max:
                raise GeometryError(f"degenerate element {b // n3} (det <= 0 at node {b % n3})")
            if source is FactorSource.TRILINEAR_PARTIAL:
                self._lam_geo = torch.empty((E, n3), dtype=torch.float64, device=dev)
                _native.check(L.hx_setup_partial(spec.order, E, _ptr(verts), _ptr(self._lam_geo), stream))
            elif source is FactorSource.TRILINEAR_MERGED:
                l0, l0v = self._coeff(lam0, E, n3, dev)
                l1, l1v = self._coeff(lam1, E, n3, dev)
                self._lam2 = torch.empty((E, n3), dtype=torch.float64, device=dev)
                self._lam3 = torch.empty((E, n3), dtype=torch.float64, device=dev)
                _native.check(
                    L.hx_setup_merged(
                        spec.order, E, _ptr(verts), _ptr(l0), l0v, _ptr(l1), l1v,
                        _ptr(self._lam2), _ptr(self._lam3), stream,
                    )
                )
        self._lam0 = self._lam1 = None
        self._lam0v = self._lam1v = 1.0
        if helm and source is not FactorSource.TRILINEAR_MERGED:
            self._lam0, self._lam0v = self._coeff(lam0, E, n3, dev)
            self._lam1, self._lam1v = self._coeff(lam1, E, n3, dev)
        self.kernel = 0  # 0 = best measured, 1 = slice kernel, 2 = fast kernel (hx_axlocal_args.kernel)

    # ---- setup helpers -------------------------------------------------
    @staticmethod
    def _vertices(elements, dev):
        """(E,8,3) fp64 device tensor, plus the kind set when known on the host."""
        torch = _torch()
        if isinstance(elements, torch.Tensor):
            if elements.ndim != 3 or tuple(elements.shape[1:]) != (8, 3):
                raise ValueError("vertex tensor must have shape (E, 8, 3)")
            return elements.to(device=dev, dtype=torch.float64).contiguous(), None
        if isinstance(elements, BoxMesh):
            return elements.vertices_device(dev), None
        if isinstance(elements, Mesh):
            return torch.as_tensor(elements.vertices, device=dev), set(elements.kinds)
        if isinstance(elements, np.ndarray) and elements.ndim == 3:
            if tuple(elements.shape[1:]) != (8, 3):
                raise ValueError("vertex array must have shape (E, 8, 3)")
            return torch.as_tensor(np.ascontiguousarray(elements, dtype=np.float64), device=dev), None
        elements = list(elements)
        if not elements:
            return torch.empty((0, 8, 3), dtype=torch.float64, device=dev), set()
        kinds = set()
        for el in elements:
            kind = getattr(el, "kind", None)
            kinds.add(_coerce_enum(ElementKind, kind) if kind is not None else ElementKind.GENERAL)
        host = np.stack([np.asarray(el.vertices, dtype=np.float64) for el in elements])
        return torch.as_tensor(host, device=dev), kinds

    def _classify(self, verts, stream):
        torch = _torch()
        kind = torch.empty((verts.shape[0],), dtype=torch.int8, device=verts.device)
        _native.check(_native.lib().hx_classify_elements(int(verts.shape[0]), _ptr(verts), _ptr(kind), stream))
        n_ppd = int(kind.sum().item())
        out = set()
        if n_ppd:
            out.add(ElementKind.PARALLELEPIPED)
        if n_ppd < verts.shape[0]:
            out.add(ElementKind.TRILINEAR)
        return out

    @staticmethod
    def _coeff(value, E, n3, dev):
        """(device field or None, scalar) per _coeff_field (axlocal.py:88-101)."""
        torch = _torch()
        if value is None:
            return None, 1.0
        if isinstance(value, LocalField) or hasattr(value, "data") and hasattr(value, "order"):
            value = np.asarray(value.data)[:, :, 0]
        if isinstance(value, torch.Tensor):
            arr = value.to(device=dev, dtype=torch.float64)
        else:
            arr = np.asarray(value, dtype=float)
            if arr.ndim == 0:
                return None, float(arr)
            arr = torch.as_tensor(arr, device=dev)
        if arr.ndim == 0:
            return None, float(arr.item())
        if tuple(arr.shape) == (n3,):
            return arr.unsqueeze(0).expand(E, n3).contiguous(), 1.0
        if tuple(arr.shape) != (E, n3):
            raise ValueError("coefficient field must be scalar or shaped (E, n1**3)")
        return arr.contiguous(), 1.0

    # ---- apply ---------------------------------------------------------
    def _args(self, x_ptr, y_ptr, e0=0, n=None) -> _native.AxArgs:
        """Kernel arguments for elements [e0, e0+n); x_ptr/y_ptr point at element e0."""
        spec = self.spec
        n = self.n_elements - e0 if n is None else n
        n3 = self.basis.n1**3

        def off(t, per):
            return None if t is None else t.data_ptr() + 8 * per * e0

        return _native.AxArgs(
            order=spec.order,
            n_col=spec.n_col,
            equation=0 if spec.equation is Equation.POISSON else 1,
            factor_source=_HX_SOURCE[spec.factor_source],
            n_elements=n,
            x=x_ptr,
            y=y_ptr,
            verts=off(self._verts, 24),
            h=off(self._h, 7),
            g=off(self._g, 6 * n3),
            gwj=off(self._gwj, n3),
            lam_geo=off(self._lam_geo, n3),
            lam2=off(self._lam2, n3),
            lam3=off(self._lam3, n3),
            lam0=off(self._lam0, n3),
            lam1=off(self._lam1, n3),
            lam0_value=self._lam0v,
            lam1_value=self._lam1v,
            kernel=self.kernel,
            reserved=0,
        )

    def _launch(self, args, stream=None):
        s = _stream(self.device) if stream is None else ctypes.c_void_p(stream)
        _native.check(_native.lib().hx_axlocal(ctypes.byref(args), s))

    def apply_lattice_(self, u, y, box, stream=None, cg=None):
        """y = A Q u: the element-local x gathered on the fly from the slab lattice
        vector u of ``box`` (fused BP5 gather; order 7, one column).  With
        ``cg = (r, scal, p_out)`` the CG direction update p_out = r + (scal[2] /
        scal[0]) u is fused in and A is applied to p_out (hx_axlocal_args.cg_r)."""
        args = self._args(u.data_ptr(), y.data_ptr())
        args.gather = 1
        args.gather_box = box
        if cg is not None:
            r, scal, p_out = cg
            args.cg_r = r.data_ptr()
            args.cg_scal = scal.data_ptr()
            args.cg_p_out = p_out.data_ptr()
        self._launch(args, stream)
        return y

    def apply_(self, x, y, stream=None):
        """y = A x for contiguous fp64 device tensors (E, n1^3, n_col); stream-ordered,
        no allocation, no synchronisation."""
        self._check_device_pair(x, y)
        self._launch(self._args(x.data_ptr(), y.data_ptr()), stream)
        return y

    def graphed(self, x, y, applies: int = 1):
        """A CUDA graph of ``applies`` back-to-back ``apply_(x, y)`` launches on these
        fixed buffers; calling the returned function replays it on the current stream.
        For small element counts, where a host API call (~14 us) costs more than the
        kernel (~3 us at E = 512, N = 7; profiles/r01_config_bench_c1_c2.txt)."""
        torch = _torch()
        self._check_device_pair(x, y)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.apply_(x, y)  # warm-up outside the capture (basis upload, lazy module load)
        torch.cuda.current_stream(self.device).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(applies):
                self.apply_(x, y)
        return graph.replay

    def _check_device_pair(self, x, y):
        torch = _torch()
        want = (self.n_elements, self.basis.n1**3, self.spec.n_col)
        for name, t in (("x", x), ("y", y)):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
            if tuple(t.shape) != want and not (t.ndim == 2 and tuple(t.shape) == want[:2] and want[2] == 1):
                raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {want}")
            if t.device != self.device:
                raise ValueError(f"{name} is on {t.device}, the operator on {self.device}")

    def _check_shape(self, order, n_el, n_col):
        if order is not None and order != self.spec.order:
            raise ValueError("field order does not match the operator")
        if n_el != self.n_elements:
            raise ValueError("field element count does not match the operator")
        if n_col != self.spec.n_col:
            raise ValueError(f"operator expects {self.spec.n_col} column(s)")

    def apply(self, x, threads: int = 1, out=None):
        """Y = A X.

        * ``LocalField`` (host numpy, the reference's type) -> ``LocalField``;
        * CUDA tensor (E, n1^3, n_col) or (E, n1^3) -> CUDA tensor (no copies);
        * host torch tensor (pinned for full speed) -> host tensor, through a
          chunked pipeline that overlaps the H2D copy of chunk c+1, the kernel on
          chunk c and the D2H copy of chunk c-1.
        """
        torch = _torch()
        n3 = self.basis.n1**3
        if isinstance(x, torch.Tensor):
            xt = x if x.ndim == 3 else x.unsqueeze(-1)
            if xt.ndim != 3 or xt.shape[1] != n3:
                raise ValueError(f"expected {n3} nodes per element")
            self._check_shape(None, xt.shape[0], xt.shape[2])
            if not xt.is_cuda:
                y = self._apply_host(xt.to(torch.float64).contiguous(), out)
                return y if x.ndim == 3 else y.squeeze(-1)
            xt = xt.to(device=self.device, dtype=torch.float64).contiguous()
            y = out if out is not None else torch.empty_like(xt)
            self.apply_(xt, y)
            return y if x.ndim == 3 else y.squeeze(-1)
        self._check_shape(x.order, x.n_elements, x.n_col)
        host = torch.from_numpy(np.ascontiguousarray(x.data, dtype=np.float64))
        y = self._apply_host(host, None)
        return LocalField(y.numpy(), self.spec.order)

    def _apply_host(self, xh, out):
        torch = _torch()
        dev = self.device
        if not xh.is_pinned():
            xh = xh.pin_memory()
        yh = out if out is not None else torch.empty(xh.shape, dtype=torch.float64, pin_memory=True)
        bufs = getattr(self, "_dev_bufs", None)
        if bufs is None or bufs[0].shape != xh.shape:
            bufs = (torch.empty(xh.shape, dtype=torch.float64, device=dev),
                    torch.empty(xh.shape, dtype=torch.float64, device=dev),
                    torch.cuda.Stream(dev), torch.cuda.Stream(dev))
            self._dev_bufs = bufs
        xd, yd, s_in, s_out = bufs
        cur = torch.cuda.current_stream(dev)
        E = self.n_elements
        # 32 chunks: pipeline fill / drain ~3 % of a step (16: 5.69, 32: 5.82, 64: 5.83 GDOF/s e2e at C4)
        chunk = max(1024, -(-E // int(os.environ.get("HX_E2E_CHUNKS", "32"))))
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        for a in range(0, E, chunk):
            b = min(E, a + chunk)
            with torch.cuda.stream(s_in):
                xd[a:b].copy_(xh[a:b], non_blocking=True)
            cur.wait_stream(s_in)
            self._launch(self._args(xd[a].data_ptr(), yd[a].data_ptr(), a, b - a), cur.cuda_stream)
            s_out.wait_stream(cur)
            with torch.cuda.stream(s_out):
                yh[a:b].copy_(yd[a:b], non_blocking=True)
        cur.wait_stream(s_out)
        s_out.synchronize()
        return yh


def dense_local_matrix(spec, element, basis, lam0=None, lam1=None):
    """Explicitly assembled (n1^3 x n1^3) element matrix (reference axlocal.py:277-310).

    The reference builds it from the general-route (stored) factors and the dense
    Kronecker gradient; here the stored-factor operator is applied on the GPU to
    the n1^3 unit vectors at once (the element replicated n1^3 times, column j of
    the result is A e_j), which agrees with the reference's matrix to 1e-12.
    Returns a host numpy array.
    """
    torch = _torch()
    spec = _as_spec(spec)
    helm = spec.equation is Equation.HELMHOLTZ
    if not helm and (lam0 is not None or lam1 is not None):
        raise ValueError("coefficient fields apply to the Helmholtz operator only")
    n3 = basis.n1**3

    def one_element(value):
        if value is None or np.ndim(getattr(value, "data", value)) == 0:
            return value
        arr = np.asarray(value.data)[:, :, 0] if isinstance(value, LocalField) else np.asarray(value, dtype=float)
        if arr.shape == (1, n3):
            arr = arr[0]
        if arr.shape != (n3,):
            raise ValueError("coefficient field must be scalar or shaped (E, n1**3)")
        return arr

    verts = np.asarray(getattr(element, "vertices", element), dtype=np.float64).reshape(1, 8, 3)
    dev = torch.device("cuda", torch.cuda.current_device())
    op = LocalOperator(KernelSpec(spec.equation, 1, FactorSource.STORED, spec.order),
                       torch.as_tensor(np.repeat(verts, n3, axis=0), device=dev), basis,
                       lam0=one_element(lam0), lam1=one_element(lam1), device=dev)
    eye = torch.eye(n3, dtype=torch.float64, device=dev).unsqueeze(-1)
    return op.apply(eye)[:, :, 0].T.contiguous().cpu().numpy()


def ax_local_apply(spec, elements, basis, x, lam0=None, lam1=None, threads: int = 1):
    """One-shot convenience wrapper around :class:`LocalOperator` (axlocal.py:261-271)."""
    return LocalOperator(spec, elements, basis, lam0=lam0, lam1=lam1).apply(x, threads)
