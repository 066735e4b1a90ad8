"""BP5 / Nekbone conjugate-gradient proxy on the GPU (reference pkg/src/hosfem/solver.py).

Same public surface as the reference module — ``GlobalOperator`` (64-99),
``cg_solve`` (124-178), ``global_node_coords`` (181-194),
``sine_product_field`` (197-199), ``NekboneConfig`` / ``NekboneResult``
(202-225), ``compatible_variants`` (228-237), ``nekbone_benchmark``
(240-308) — for structured box meshes, with every vector resident on the
device:

* Q (gather) and Q^T (scatter-add) are C-ABI kernels on the structured lattice
  (``hx_bp5_gather`` / ``hx_bp5_scatter_add``): the lattice index is computed,
  not loaded, and scatter-add is owner-computes in ascending element order
  (the order of the reference's np.bincount), so no atomics;
* the local operator is the B200 AxLocal (``LocalOperator.apply_``);
* dots are fixed-tree device reductions (``hx_dot``), the CG updates fused
  kernels (``hx_cg_update_xr`` / ``hx_cg_update_p``) that read alpha and beta
  from device scalars; the host reads two scalars per iteration (the
  reference's breakdown and convergence tests).

Multi-GPU (one process per GPU): ranks own z-slabs of elements
(``sharding.slab_layers``). After the local scatter-add each interface plane
holds two partial sums; neighbours swap them (NCCL send/recv) and both form
``lower + upper`` in that order, so the two copies stay bit-identical. Dot
products sum each rank's owned planes (a shared plane belongs to the lower
rank) and the per-rank partials are combined in rank order (all_gather), so
the solve is bitwise reproducible for a given rank count.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .axlocal import Equation, FactorSource, KernelSpec, LocalOperator
from .basis import SpectralBasis
from .mesh import BoxMesh, _kinds_from_defects, box_mesh
from .sharding import World, slab_layers
from .workload import ax_flops

__all__ = [
    "SlabLayout",
    "GlobalOperator",
    "CgReport",
    "cg_solve",
    "global_node_coords",
    "sine_product_field",
    "NekboneConfig",
    "NekboneResult",
    "compatible_variants",
    "nekbone_benchmark",
]


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
@dataclass
class SlabLayout:
    """The slab of one rank: element layers [z0, z1) of an ex x ey x ez box."""

    counts: tuple
    order: int
    rank: int = 0
    size: int = 1

    def __post_init__(self):
        ex, ey, ez = self.counts
        self.z0, self.z1 = slab_layers(ez, self.size, self.rank)
        n = self.order
        self.nx, self.ny = ex * n + 1, ey * n + 1
        self.nz_el = self.z1 - self.z0
        self.planes = self.nz_el * n + 1
        self.plane = self.nx * self.ny
        self.n_local = self.plane * self.planes
        # nodes this rank owns for reductions: the top plane belongs to the next rank
        self.n_owned = self.n_local if self.rank == self.size - 1 else self.n_local - self.plane
        self.n_elements = ex * ey * self.nz_el

    @property
    def global_node_count(self) -> int:
        ex, ey, ez = self.counts
        return self.nx * self.ny * (ez * self.order + 1)

    def box(self, n_col: int = 1, col: int = 0):
        ex, ey, ez = self.counts
        return _native.Box(order=self.order, ex=ex, ey=ey, nz_el=self.nz_el, z0=self.z0, ez=ez, n_col=n_col,
                           col=col)

    def global_slice(self):
        """The slab's range in the reference's flat lattice numbering."""
        start = self.z0 * self.order * self.plane
        return slice(start, start + self.n_local)


# ---------------------------------------------------------------------------
class CudaBackend:
    """The C-ABI kernels (the product path)."""

    def __init__(self, device):
        torch = _torch()
        self.device = device
        self.work = torch.empty(1184, dtype=torch.float64, device=device)

    def _s(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def local_operator(self, spec, verts, basis, lam0, lam1):
        return LocalOperator(spec, verts, basis, lam0=lam0, lam1=lam1, device=self.device)

    def gather(self, layout, u, xl, n_col=1, col=0):
        b = layout.box(n_col, col)
        _native.check(_native.lib().hx_bp5_gather(ctypes.byref(b), u.data_ptr(), xl.data_ptr(), self._s()))

    def scatter(self, layout, yl, v, n_col=1, col=0):
        b = layout.box(n_col, col)
        _native.check(_native.lib().hx_bp5_scatter_add(ctypes.byref(b), yl.data_ptr(), v.data_ptr(), self._s()))

    def mask(self, layout, v):
        b = layout.box()
        _native.check(_native.lib().hx_bp5_mask(ctypes.byref(b), v.data_ptr(), self._s()))

    def dot(self, a, b, n, out):
        """out (1-element device view) = sum_{i<n} a[i] b[i]."""
        _native.check(_native.lib().hx_dot(a.data_ptr(), b.data_ptr(), 0, n, self.work.data_ptr(),
                                           out.data_ptr(), self._s()))

    def update_xr(self, scal, x, p, r, ap):
        _native.check(_native.lib().hx_cg_update_xr(scal.data_ptr(), x.data_ptr(), p.data_ptr(), r.data_ptr(),
                                                    ap.data_ptr(), x.numel(), self._s()))

    def update_p(self, scal, p, r):
        _native.check(_native.lib().hx_cg_update_p(scal.data_ptr(), p.data_ptr(), r.data_ptr(), p.numel(),
                                                   self._s()))

    # fused CG pieces (single kernels; optional in a backend)
    def scatter_dot(self, layout, yl, v, p, n_owned, out):
        torch = _torch()
        need = -(-layout.ny // 16) * layout.planes  # one partial per band of 16 lattice rows (hx_axlocal.h)
        if getattr(self, "_row_work", None) is None or self._row_work.numel() < need:
            self._row_work = torch.empty(need, dtype=torch.float64, device=self.device)
        b = layout.box()
        _native.check(_native.lib().hx_bp5_scatter_dot(ctypes.byref(b), yl.data_ptr(), v.data_ptr(), p.data_ptr(),
                                                       n_owned, self._row_work.data_ptr(), out.data_ptr(),
                                                       self._s()))

    def update_xr_dot(self, scal, x, p, r, ap, n_owned, out):
        _native.check(_native.lib().hx_cg_update_xr_dot(scal.data_ptr(), x.data_ptr(), p.data_ptr(), r.data_ptr(),
                                                        ap.data_ptr(), x.numel(), n_owned, self.work.data_ptr(),
                                                        out.data_ptr(), self._s()))

    fused_gather = os.environ.get("HX_BP5_FUSED_GATHER", "1") != "0"

    def local_apply_lattice(self, local_op, layout, u, yl, cg=None):
        """y = A Q u with the gather fused into the AxLocal loads, when supported
        (and, with ``cg = (r, scal, p_out)``, the CG direction update too)."""
        if not self.supports_lattice_apply(local_op):
            return False
        local_op.apply_lattice_(u, yl, layout.box(), cg=cg)
        return True

    def supports_lattice_apply(self, local_op) -> bool:
        return self.fused_gather and local_op.spec.order == 7 and local_op.spec.n_col == 1


# ---------------------------------------------------------------------------
class GlobalOperator:
    """Q^T A Q on the rank's slab (reference solver.py:64-99), device vectors.

    ``apply(u)`` takes and returns flat slab-lattice tensors (``layout.n_local``);
    ``apply_global(u)`` is the reference's host-array form (single process).
    """

    def __init__(self, mesh: BoxMesh, spec: KernelSpec, basis, lam0=None, lam1=None, world: World | None = None,
                 device=None, backend=None):
        torch = _torch()
        if spec.order != mesh.order:
            raise ValueError("kernel spec order does not match the mesh")
        self.mesh, self.spec, self.basis = mesh, spec, basis
        self.world = world or World({})
        self.layout = SlabLayout(tuple(mesh.counts), mesh.order, self.world.rank, self.world.size)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.backend = backend or CudaBackend(self.device)
        L = self.layout
        if self.device.type == "cuda":
            verts = mesh.vertices_device(self.device, L.z0, L.z1)
        else:
            verts = torch.as_tensor(mesh.vertices_slab(L.z0, L.z1))
        l0, l1 = self._distribute(lam0), self._distribute(lam1)
        self.local_op = self.backend.local_operator(spec, verts, basis, l0, l1)
        n3 = basis.n1**3
        shape = (L.n_elements, n3, spec.n_col)
        self._xl = torch.empty(shape, dtype=torch.float64, device=self.device)
        self._yl = torch.empty(shape, dtype=torch.float64, device=self.device)
        self._events = []  # (start, after-gather, after-local, end) per apply, read lazily
        self._t_local = self._t_apply = 0.0
        self.applies = 0

    def _flush_events(self):
        if self._events:
            self._events[-1][3].synchronize()
            for ev in self._events:
                self._t_local += ev[1].elapsed_time(ev[2]) * 1e-3
                self._t_apply += ev[0].elapsed_time(ev[3]) * 1e-3
            self._events = []

    @property
    def seconds_local(self) -> float:
        """Cumulative element-local (AxLocal) device time, as the reference keeps it (solver.py:79-99)."""
        self._flush_events()
        return self._t_local

    @property
    def seconds_apply(self) -> float:
        self._flush_events()
        return self._t_apply

    def _distribute(self, value):
        """Scalars pass through; global nodal arrays are gathered to the slab's elements (solver.py:102-109)."""
        if value is None or np.ndim(value) == 0:
            return value
        torch = _torch()
        arr = np.asarray(value, dtype=float)
        if arr.shape != (self.layout.global_node_count,):
            return value
        u = torch.as_tensor(arr[self.layout.global_slice()], device=self.device)
        n3 = self.basis.n1**3
        xl = torch.empty((self.layout.n_elements, n3, 1), dtype=torch.float64, device=self.device)
        self.backend.gather(self.layout, u, xl)
        return xl[:, :, 0]

    def reset_counters(self) -> None:
        self._flush_events()
        self._t_local = self._t_apply = 0.0
        self.applies = 0

    def new_vector(self):
        """Zero slab vector: (n_local,) for one column, (n_col, n_local) otherwise."""
        torch = _torch()
        nc = self.spec.n_col
        shape = (self.layout.n_local,) if nc == 1 else (nc, self.layout.n_local)
        return torch.zeros(shape, dtype=torch.float64, device=self.device)

    def columns(self, v):
        return [v] if self.spec.n_col == 1 else [v[c] for c in range(self.spec.n_col)]

    def apply(self, u, out=None, dot_with=None, dot_out=None, cg_update=None):
        """v = Q^T A Q u on the slab (interfaces completed).  With ``dot_with``
        (single rank, one column) the boundary mask and the dot
        dot_out = dot_with . v over owned nodes are fused into the scatter.  With
        ``cg_update = (r, scal, p_new)`` (see :meth:`can_fuse_cg_update`) the CG
        direction update p_new = r + (scal[2] / scal[0]) u runs inside the AxLocal
        gather and v = Q^T A Q p_new."""
        torch = _torch()
        L, B = self.layout, self.backend
        nc = self.spec.n_col
        v = out if out is not None else self.new_vector()
        timing = self.device.type == "cuda"
        if timing:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
        fused_gather = nc == 1 and hasattr(B, "local_apply_lattice")
        if fused_gather and timing:
            ev[1].record()
        if cg_update is not None:
            if not (fused_gather and B.local_apply_lattice(self.local_op, L, u, self._yl, cg=cg_update)):
                raise ValueError("the fused CG update needs the fused lattice gather (order 7, one column)")
        elif not (fused_gather and B.local_apply_lattice(self.local_op, L, u, self._yl)):
            for c, uc in enumerate(self.columns(u)):
                B.gather(L, uc, self._xl, nc, c)
            if timing:
                ev[1].record()
            self.local_op.apply_(self._xl, self._yl)
        if timing:
            ev[2].record()
        fused = dot_with is not None
        if fused:
            B.scatter_dot(L, self._yl, v, dot_with, L.n_owned, dot_out)
        else:
            for c, vc in enumerate(self.columns(v)):
                B.scatter(L, self._yl, vc, nc, c)
                self._exchange_interfaces(vc)
        if timing:
            ev[3].record()
            self._events.append(ev)
        self.applies += 1
        return v

    def can_fuse_cg(self) -> bool:
        return self.world.size == 1 and self.spec.n_col == 1 and hasattr(self.backend, "scatter_dot")

    #: fold p = r + beta p into the next apply's lattice gather (HX_BP5_FUSED_P=1).  Off by
    #: default: at 76^3 it saves 2 % of the trilinear solve, costs 4 % on stored, and the
    #: AxLocal share of the solve (the reference's reported rate) stops being separable.
    fuse_p_update = os.environ.get("HX_BP5_FUSED_P", "0") == "1"

    def can_fuse_cg_update(self) -> bool:
        """p = r + beta p fused into the next apply's lattice gather (N = 7, one rank)."""
        B = self.backend
        return (self.fuse_p_update and self.can_fuse_cg() and hasattr(B, "supports_lattice_apply")
                and B.supports_lattice_apply(self.local_op))

    def _exchange_interfaces(self, v):
        """Complete the shared z-planes: both neighbours end with lower + upper."""
        w = self.world
        if w.size == 1:
            return
        torch = _torch()
        dist = w.pg
        L = self.layout
        P = L.plane
        # NCCL moves device planes directly; gloo has no device P2P, so its planes
        # are staged through host memory (the CPU-only test / debugging path)
        stage = w.host_staged(v)
        ops, recv_lo, recv_hi = [], None, None
        if w.rank > 0:
            send_lo = v[:P].contiguous()
            send_lo = send_lo.cpu() if stage else send_lo
            recv_lo = torch.empty_like(send_lo)
            ops += [dist.P2POp(dist.isend, send_lo, w.rank - 1), dist.P2POp(dist.irecv, recv_lo, w.rank - 1)]
        if w.rank < w.size - 1:
            send_hi = v[-P:].contiguous()
            send_hi = send_hi.cpu() if stage else send_hi
            recv_hi = torch.empty_like(send_hi)
            ops += [dist.P2POp(dist.isend, send_hi, w.rank + 1), dist.P2POp(dist.irecv, recv_hi, w.rank + 1)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if recv_lo is not None:
            v[:P] = recv_lo.to(v.device) + v[:P]  # lower rank's partial first
        if recv_hi is not None:
            v[-P:] = v[-P:] + recv_hi.to(v.device)

    def apply_global(self, global_values):
        """Reference form (single process): host (n_global,) or (n_global, n_col) in and out."""
        torch = _torch()
        if self.world.size != 1:
            raise ValueError("apply_global is the single-process form; use apply() per rank")
        g = np.asarray(global_values, dtype=float)
        if g.shape[0] != self.layout.global_node_count:
            raise ValueError("global vector length does not match the mesh")
        dev = torch.as_tensor(np.ascontiguousarray(g.T if g.ndim == 2 else g), device=self.device)
        v = self.apply(dev).cpu().numpy()
        return v.T if g.ndim == 2 else v

    def mask(self, v):
        """Zero the box boundary of every column (in place)."""
        for vc in self.columns(v):
            self.backend.mask(self.layout, vc)
        return v


# ---------------------------------------------------------------------------
@dataclass
class CgReport:
    iterations: int
    final_relative_residual: float
    residual_history: list
    converged: bool
    solution: object
    solution_error: float | None = None


class _Reducer:
    """Fixed-order scalar reductions across ranks (device scalars -> host floats)."""

    def __init__(self, op: GlobalOperator):
        torch = _torch()
        self.op = op
        self.scal = torch.zeros(3, dtype=torch.float64, device=op.device)  # rr, pap, rr_new

    def dot(self, a, b, slot):
        """scal[slot] = global sum a.b over owned nodes (columns in order); returns the host value."""
        torch = _torch()
        op, w = self.op, self.op.world
        n = op.layout.n_owned
        cols_a, cols_b = op.columns(a), op.columns(b)
        op.backend.dot(cols_a[0], cols_b[0], n, self.scal[slot:slot + 1])
        for ca, cb in zip(cols_a[1:], cols_b[1:]):
            part = torch.zeros(1, dtype=torch.float64, device=op.device)
            op.backend.dot(ca, cb, n, part)
            self.scal[slot:slot + 1] += part
        return self.reduce_slot(slot)

    def reduce_slot(self, slot):
        """Combine a per-rank partial already in scal[slot] across ranks (rank order)."""
        torch = _torch()
        w = self.op.world
        if w.size > 1:
            mine = self.scal[slot:slot + 1].clone()
            dev = "cpu" if w.host_staged(mine) else self.op.device
            parts = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(w.size)]
            w.pg.all_gather(parts, mine.to(dev))
            total = parts[0].clone()
            for t in parts[1:]:
                total = total + t  # rank order: bitwise reproducible for a given rank count
            self.scal[slot:slot + 1] = total.to(self.op.device)
        return float(self.scal[slot].item())


def _node_mask(op: GlobalOperator, mask):
    """The reference's ``mask`` argument as (kind, device tensor): kind "none"
    (None / False: unmasked), "box" (True, or an array equal to the box
    interior: the kernel-computed mask and the fused CG paths), or "array"
    (any other boolean node array, True = kept, applied as given)."""
    torch = _torch()
    if mask is None or mask is False:
        return "none", None
    if mask is True:
        return "box", None
    L = op.layout
    m = mask.to(torch.bool) if isinstance(mask, torch.Tensor) else torch.as_tensor(np.asarray(mask, dtype=bool))
    if m.ndim != 1:
        raise ValueError("mask must be a boolean node array (True = kept)")
    if m.numel() == L.global_node_count and m.numel() != L.n_local:
        if op.world.size != 1:
            raise ValueError("a global mask is the single-process form; pass the slab's (n_local,) mask per rank")
        m = m[L.global_slice()]
    if m.numel() != L.n_local:
        raise ValueError("mask length does not match the mesh")
    m = m.to(op.device)
    box = torch.ones(L.n_local, dtype=torch.float64, device=op.device)
    op.backend.mask(L, box)
    if torch.equal(m, box.to(torch.bool)):
        return "box", None
    return "array", m.to(torch.float64)


def cg_solve(op: GlobalOperator, b, tol: float = 1e-8, max_iter: int = 1000, mask=None, threads: int = 1) -> CgReport:
    """Unpreconditioned CG on M A M (reference solver.py:124-178), all on the device.

    ``b`` is the rank's slab vector (device tensor) or, single process, a host
    (n_global,) array.  ``mask`` follows the reference: None (the default)
    solves unmasked; a boolean node array keeps the nodes where it is True (the
    negated boundary mask gives homogeneous Dirichlet conditions) -- the global
    (n_global,) array single-process, or the slab's (n_local,) array per rank;
    ``True`` is shorthand for the box interior.  The box-interior mask runs the
    fused kernels; any other mask is applied as given.  ``threads`` is accepted
    and ignored (the reference's thread-pool split has no GPU meaning).
    """
    torch = _torch()
    B, L = op.backend, op.layout
    if not isinstance(b, torch.Tensor):
        hb = np.asarray(b, dtype=float)
        b = torch.as_tensor(np.ascontiguousarray(hb.T if hb.ndim == 2 else hb), device=op.device)
    b = b.to(device=op.device, dtype=torch.float64).clone()
    kind, marr = _node_mask(op, mask)
    masked = kind == "box"

    def apply_mask(v):
        if kind == "box":
            op.mask(v)
        elif kind == "array":
            v.mul_(marr)  # columns broadcast over the last (node) axis
        return v

    apply_mask(b)
    red = _Reducer(op)
    x = torch.zeros_like(b)
    bb = red.dot(b, b, 0)
    b_norm = math.sqrt(bb)
    if b_norm == 0.0:
        return CgReport(0, 0.0, [0.0], True, x)
    r = b.clone()
    p = r.clone()
    rr = red.dot(r, r, 0)
    ap = op.new_vector()
    history = [1.0]
    converged = False
    iterations = 0
    fuse = masked and op.can_fuse_cg()
    fuse_update = hasattr(B, "update_xr_dot") and op.spec.n_col == 1
    # p = r + beta p folded into the next apply's lattice gather (same rounding as the
    # standalone update, so the iterates are bit-identical); p is double-buffered
    fuse_p = fuse and op.can_fuse_cg_update()
    p_next = torch.empty_like(p) if fuse_p else None
    pending_p = False
    for iterations in range(1, max_iter + 1):
        if fuse_p and pending_p:
            op.apply(p, out=ap, dot_with=p_next, dot_out=red.scal[1:2], cg_update=(r, red.scal, p_next))
            p, p_next = p_next, p
            red.scal[0:1] = red.scal[2:3]  # rr = rr_new, after the update read beta
            pap = float(red.scal[1].item())
        elif fuse:
            # ap = M Q^T A Q p and pap = p . ap in one scatter pass
            op.apply(p, out=ap, dot_with=p, dot_out=red.scal[1:2])
            pap = float(red.scal[1].item())
        else:
            op.apply(p, out=ap)
            apply_mask(ap)
            pap = red.dot(p, ap, 1)
        if not math.isfinite(pap):
            raise FloatingPointError("CG broke down: non-finite curvature")
        if pap <= 0.0:
            raise FloatingPointError("CG broke down: operator is not positive definite")
        if fuse_update:
            B.update_xr_dot(red.scal, x, p, r, ap, L.n_owned, red.scal[2:3])  # alpha = rr / pap
            rr_new = red.reduce_slot(2)
        else:
            B.update_xr(red.scal, x.reshape(-1), p.reshape(-1), r.reshape(-1), ap.reshape(-1))  # alpha = rr / pap
            rr_new = red.dot(r, r, 2)
        if not math.isfinite(rr_new):
            raise FloatingPointError("CG broke down: non-finite residual")
        rel = math.sqrt(rr_new) / b_norm
        history.append(rel)
        if rel <= tol:
            converged = True
            break
        if fuse_p:
            pending_p = True  # applied by the next iteration's fused gather
        else:
            B.update_p(red.scal, p.reshape(-1), r.reshape(-1))  # beta = rr_new / rr
            red.scal[0:1] = red.scal[2:3]
        rr = rr_new
    return CgReport(iterations, history[-1], history, converged, x)


# ---------------------------------------------------------------------------
def global_node_coords(mesh: BoxMesh, basis, layout: SlabLayout | None = None, device=None):
    """(n_local, 3) physical coordinates of the slab's lattice nodes, taken from
    the lowest-index element containing each node — the reference's
    first-writer rule (solver.py:181-194)."""
    torch = _torch()
    L = layout or SlabLayout(tuple(mesh.counts), mesh.order)
    n, ex, ey = mesh.order, mesh.counts[0], mesh.counts[1]
    dev = device
    g = torch.arange(L.n_local, device=dev)
    gx, gy, gz = g % L.nx, (g // L.nx) % L.ny, g // L.plane + L.z0 * n

    def owner(gc, ne):
        c = torch.div(gc, n, rounding_mode="floor")
        loc = gc - c * n
        back = (loc == 0) & (c > 0)  # lowest element: the previous one, at its last node
        c = torch.where(back, c - 1, c)
        loc = torch.where(back, torch.full_like(loc, n), loc)
        over = c >= ne
        c = torch.where(over, c - 1, c)
        loc = torch.where(over, torch.full_like(loc, n), loc)
        return c, loc

    cx, i = owner(gx, ex)
    cy, j = owner(gy, ey)
    cz, k = owner(gz, mesh.counts[2])
    corners = torch.as_tensor(mesh.corners, dtype=torch.float64, device=dev)
    xi = torch.as_tensor(np.array(basis.points, dtype=np.float64), device=dev)
    lo, hi = 0.5 * (1.0 - xi), 0.5 * (1.0 + xi)
    out = torch.zeros((L.n_local, 3), dtype=torch.float64, device=dev)
    for bit in range(8):
        fr = (hi if bit & 1 else lo)[i]
        fs = (hi if bit & 2 else lo)[j]
        ft = (hi if bit & 4 else lo)[k]
        vtx = corners[cx + (bit & 1), cy + ((bit >> 1) & 1), cz + ((bit >> 2) & 1)]
        out += ((ft * fs) * fr)[:, None] * vtx
    return out


def sine_product_field(coords):
    """sin(pi x) sin(pi y) sin(pi z) (solver.py:197-199)."""
    torch = _torch()
    if isinstance(coords, torch.Tensor):
        return torch.prod(torch.sin(math.pi * coords), dim=1)
    return np.prod(np.sin(np.pi * coords), axis=1)


@dataclass
class NekboneConfig:
    order: int = 7
    elements: tuple = (4, 4, 4)
    equation: Equation = Equation.POISSON
    n_col: int = 1
    variants: tuple | None = None
    tol: float = 1e-8
    max_iter: int = 200
    perturbation: float = 0.0
    seed: int = 0
    threads: int = 1


@dataclass
class NekboneResult:
    variant: str
    iterations: int
    error: float
    wall_time_s: float
    gflops_effective: float
    axlocal_share: float
    history: list = field(default_factory=list, repr=False)


def compatible_variants(equation, all_parallelepiped: bool) -> tuple:
    """solver.py:228-237."""
    eq = Equation(getattr(equation, "value", equation))
    out = [FactorSource.STORED, FactorSource.TRILINEAR_RECOMPUTE]
    out.append(FactorSource.TRILINEAR_MERGED if eq is Equation.HELMHOLTZ else FactorSource.TRILINEAR_PARTIAL)
    if all_parallelepiped:
        out.append(FactorSource.PARALLELEPIPED_RECOMPUTE)
    return tuple(out)


def nekbone_benchmark(config: NekboneConfig, world: World | None = None, device=None, backend=None):
    """The CG proxy once per factor variant on a shared right-hand side
    (solver.py:240-308).  Returns (results, mesh)."""
    torch = _torch()
    world = world or World({})
    eq = Equation(getattr(config.equation, "value", config.equation))
    basis = SpectralBasis.build(config.order)
    ex, ey, ez = config.elements
    mesh = box_mesh(ex, ey, ez, config.order, perturbation=config.perturbation, seed=config.seed)
    # classify the elements with make_element's defect rule, as the reference does
    # (solver.py:260), not from the perturbation value (a tiny jitter may stay
    # within the 1e-12 defect tolerance)
    all_ppd = bool(_kinds_from_defects(mesh.vertices).all())
    variants = config.variants or compatible_variants(eq, all_ppd)
    variants = tuple(FactorSource(getattr(v, "value", v)) for v in variants)
    variants = tuple(v for v in variants if not (v is FactorSource.PARALLELEPIPED_RECOMPUTE and not all_ppd))
    if config.n_col not in (1, 3):
        raise ValueError("n_col must be 1 or 3")

    def build(source):
        spec = KernelSpec(eq, config.n_col, source, config.order)
        kw = {"lam0": 1.0, "lam1": 1.0} if eq is Equation.HELMHOLTZ else {}
        return GlobalOperator(mesh, spec, basis, world=world, device=device, backend=backend, **kw)

    reference = build(FactorSource.STORED)
    L = reference.layout
    coords = global_node_coords(mesh, basis, L, device=reference.device)
    exact = sine_product_field(coords)
    if config.n_col == 3:
        exact = exact[None, :].repeat(3, 1).contiguous()
    # b = M A_stored M u*  (solver.py:275-278)
    b = reference.mask(reference.apply(reference.mask(exact.clone())))
    del reference
    results = []
    flops_per_apply = mesh.n_elements * ax_flops(eq, config.n_col, config.order + 1)
    for source in variants:
        op = build(source)
        op.reset_counters()
        if op.device.type == "cuda":
            torch.cuda.synchronize(op.device)
        t0 = time.perf_counter()
        report = cg_solve(op, b, tol=config.tol, max_iter=config.max_iter, mask=True)
        if op.device.type == "cuda":
            torch.cuda.synchronize(op.device)
        wall = time.perf_counter() - t0
        diff = op.mask(report.solution - exact)
        local_err = float(diff[..., : L.n_owned].abs().max().item()) if diff.numel() else 0.0
        red_dev = op.device if op.device.type == "cuda" else None
        error = world.max(local_err, red_dev)
        seconds_local = world.max(max(op.seconds_local, 1e-12), red_dev)
        results.append(
            NekboneResult(
                variant=source.value,
                iterations=report.iterations,
                error=error,
                wall_time_s=wall,
                gflops_effective=op.applies * flops_per_apply / seconds_local / 1e9,
                axlocal_share=min(seconds_local / max(wall, 1e-12), 1.0),
                history=report.residual_history,
            )
        )
        del op
    return results, mesh
