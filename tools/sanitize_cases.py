"""Small applies of every kernel family: the memory and race checks of this pool.

    python tools/sanitize_cases.py [--dump out.npz] [--compare ref.npz]
    HX_AXLOCAL_LIB=_variants/perturb/libhx_axlocal.so python tools/sanitize_cases.py --compare ref.npz

compute-sanitizer is closed on the GPU pool, so:
* memory (memcheck's job): every array a kernel reads or writes -- x, y,
  vertices, the operator's factor fields, BP5 lattice vectors -- is a view into
  a larger buffer whose guard bands hold NaN (an out-of-bounds read poisons
  the output, which must stay finite and match the oracle to 1e-12) or a
  sentinel bit pattern (an out-of-bounds write changes it; checked after
  every launch);
* races (racecheck's job): the same cases with the timing-perturbation build
  (tools/race_perturb.sh: every barrier jittered by 0..4 us per thread) must
  reproduce the normal build's outputs bit for bit (--dump / --compare).

~64 elements per case.  Covers
the N=7 kernels (DMMA ax8m n_col 1 / 3 (ax8m3, CTA3) with 0 / 1 / 2 staged
coefficient fields / fused lattice gather + CG update, ax8s, ax8c3), the order-generic role-table kernels (axn_r) at
n1 = 4, 7, 11, the slice kernel, the element-per-thread kernel, the j-plane
kernel (orders 2, 3), the setup
kernels and the BP5 gather / scatter (scatter_band32_kernel) / mask / dot /
CG-update kernels, every factor source and both equations.  The plain run
also checks every case against the oracle (1e-12).
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200 import solver as S  # noqa: E402

CHECK = os.environ.get("HX_SANITIZE_CHECK", "1") == "1"
DEV = torch.device("cuda", 0)
SHEAR = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
GUARD = 4096  # doubles on each side (32 KB)
SENTINEL = -1.2345678901234567e300
OUTPUTS = {}
_GUARDED = []  # (buffer, lo, hi, kind) of every guarded array


def guarded(t, kind):
    """A copy of ``t`` inside a buffer with GUARD doubles of NaN ("read") or of
    SENTINEL ("write") on each side; returns the (16-byte aligned) view."""
    n = t.numel()
    fill = float("nan") if kind == "read" else SENTINEL
    buf = torch.full((GUARD + n + GUARD,), fill, dtype=torch.float64, device=DEV)
    view = buf[GUARD:GUARD + n].view(t.shape)
    view.copy_(t)
    _GUARDED.append((buf, GUARD, GUARD + n, kind))
    return view


def check_guards(tag):
    for buf, lo, hi, kind in _GUARDED:
        if kind != "write":
            continue
        bad = int((buf[:lo] != SENTINEL).sum().item() + (buf[hi:] != SENTINEL).sum().item())
        assert bad == 0, f"{tag}: {bad} guard words overwritten (out-of-bounds write)"
    _GUARDED.clear()


def guard_operator(op):
    """Move the operator's vertex and factor arrays into NaN-guarded buffers."""
    for name in ("_verts", "_h", "_g", "_gwj", "_lam_geo", "_lam2", "_lam3", "_lam0", "_lam1"):
        t = getattr(op, name, None)
        if t is not None:
            setattr(op, name, guarded(t.contiguous(), "read"))


def case(order, dims, eq, src, n_col, kernel, fields="lam0"):
    mesh = hx.box_mesh(*dims, order, perturbation=0.0 if src == "parallelepiped" else 0.12, seed=order)
    verts = mesh.vertices @ SHEAR.T if src == "parallelepiped" else mesh.vertices
    E, n3 = len(verts), (order + 1) ** 3
    rng = np.random.default_rng(order + n_col)
    kw = {}
    if eq == "helmholtz":  # fields: which coefficients are (E, n1^3) fields (the DMMA kernel stages them)
        kw = {"lam0": rng.uniform(0.5, 2.0, (E, n3)) if fields in ("lam0", "both") else 1.3,
              "lam1": rng.uniform(0.5, 2.0, (E, n3)) if fields == "both" else 0.7}
    op = hx.LocalOperator(hx.KernelSpec(eq, n_col, src, order), torch.as_tensor(verts, device=DEV),
                          hx.SpectralBasis.build(order), **kw)
    op.kernel = kernel
    guard_operator(op)
    x = rng.standard_normal((E, n3, n_col))
    xd = guarded(torch.as_tensor(x, device=DEV), "read")
    yd = guarded(torch.zeros_like(xd), "write")
    op.apply_(xd, yd)
    torch.cuda.synchronize()
    tag = f"N={order} {eq} {src} n_col={n_col} kernel={kernel}" + ("" if fields == "lam0" else f" fields={fields}")
    check_guards(tag)
    y = yd.cpu().numpy()
    assert np.isfinite(y).all(), f"{tag}: non-finite output (out-of-bounds read of a NaN guard?)"
    if CHECK:
        from oracle import hosfem_oracle as O  # checker only

        err = O.rel_diff(y, O.apply(src, eq, order, verts, x, kw.get("lam0"), kw.get("lam1")))
        assert err <= 1e-12, (tag, err)
    OUTPUTS[tag] = y
    return y


def main():
    n = 0
    # N = 7: DMMA (kernel 4; n_col 3 -> ax8m3 for the trilinear sources), ax8s / ax8c3 (kernel 2)
    for kernel in (4, 2):
        for eq, src in (("poisson", "trilinear"), ("poisson", "trilinear-partial"), ("poisson", "stored"),
                        ("poisson", "parallelepiped"), ("helmholtz", "trilinear"), ("helmholtz", "trilinear-merged"),
                        ("helmholtz", "stored"), ("helmholtz", "parallelepiped")):
            for n_col in (1, 3):
                case(7, (4, 4, 4), eq, src, n_col, kernel)
                n += 1
                if kernel == 4 and eq == "helmholtz":  # staged coefficient fields: both / none
                    for fields in ("both", "none"):
                        case(7, (4, 4, 4), eq, src, n_col, kernel, fields)
                        n += 1
    # order-generic role-table kernels (axn_r) at n1 = 4, 7, 11; slice kernel; element per thread
    for order in (3, 6, 10):
        for src in ("trilinear", "stored", "parallelepiped"):
            case(order, (4, 4, 4) if order < 10 else (3, 3, 2), "poisson", src, 1, 2)
            n += 1
        case(order, (3, 3, 2), "helmholtz", "trilinear-merged", 3, 2)
        n += 1
    for order in (2, 5):
        case(order, (3, 3, 2), "helmholtz", "trilinear", 1, 1)
        n += 1
    for order in (1, 2):
        case(order, (4, 4, 4), "poisson", "trilinear", 3, 3)
        n += 1
    # j-plane kernel (ax_plane.cu, kernel 5) at orders 2 and 3: every source, n_col 1 and 3
    for order in (2, 3):
        for eq, src in (("poisson", "trilinear"), ("poisson", "stored"), ("poisson", "parallelepiped"),
                        ("helmholtz", "trilinear-merged"), ("helmholtz", "trilinear")):
            case(order, (5, 3, 2), eq, src, 3 if src == "trilinear" else 1, 5)
            n += 1
    # setup kernels (stored / partial / merged / ppd / validation / classification) ran above;
    # BP5: gather, scatter (band32 at N = 7), fused scatter + dot, mask, CG updates, fused-gather AxLocal
    for order, dims in ((7, (3, 2, 4)), (3, (4, 3, 2))):
        mesh = hx.box_mesh(*dims, order, perturbation=0.1, seed=1)
        for ws in (1, 2):
            for r in range(ws):
                L = S.SlabLayout(dims, order, r, ws)
                be = S.CudaBackend(DEV)
                gen = torch.Generator(device=DEV).manual_seed(100 * order + 10 * ws + r)
                u = guarded(torch.randn(L.n_local, dtype=torch.float64, device=DEV, generator=gen), "read")
                xl = guarded(torch.zeros((L.n_elements, (order + 1) ** 3, 1), dtype=torch.float64, device=DEV),
                             "write")
                be.gather(L, u, xl)
                v = guarded(torch.zeros_like(u), "write")
                be.scatter(L, xl, v)
                be.mask(L, v)
                out = guarded(torch.zeros(1, dtype=torch.float64, device=DEV), "write")
                be.dot(u, v, L.n_owned, out)
                w = guarded(torch.zeros_like(u), "write")
                out2 = guarded(torch.zeros(1, dtype=torch.float64, device=DEV), "write")
                be.scatter_dot(L, xl, w, u, L.n_owned, out2)
                yl = guarded(torch.zeros_like(xl), "write")
                if order == 7:  # fused lattice gather (DMMA kernel) on the slab
                    lop = hx.LocalOperator(hx.KernelSpec("poisson", 1, "trilinear", order),
                                           mesh.vertices_device(DEV, L.z0, L.z1), hx.SpectralBasis.build(order))
                    guard_operator(lop)
                    lop.apply_lattice_(u, yl, L.box())
                torch.cuda.synchronize()
                tag = f"bp5 N={order} ws={ws} r={r}"
                check_guards(tag)
                for name, t in (("xl", xl), ("v", v), ("w", w), ("dot", out), ("sdot", out2), ("yl", yl)):
                    arr = t.cpu().numpy()
                    assert np.isfinite(arr).all(), (tag, name)
                    OUTPUTS[f"{tag} {name}"] = arr
                n += 1
        op = S.GlobalOperator(mesh, hx.KernelSpec("poisson", 1, "trilinear", order), hx.SpectralBasis.build(order))
        b = torch.randn(op.layout.n_local, dtype=torch.float64, device=DEV,
                        generator=torch.Generator(device=DEV).manual_seed(order))
        OUTPUTS[f"cg N={order}"] = S.cg_solve(op, b, tol=1e-6, max_iter=4, mask=True).solution.cpu().numpy()
        if order == 7:
            op.fuse_p_update = True  # the fused CG update inside the DMMA lattice gather
            OUTPUTS[f"cg fused-p N={order}"] = S.cg_solve(op, b, tol=1e-6, max_iter=4, mask=True).solution.cpu().numpy()
        n += 1
    torch.cuda.synchronize()
    lib = os.environ.get("HX_AXLOCAL_LIB", "in-tree build")
    print(f"sanitize_cases: {n} cases ok with {lib}: guard bands intact, outputs finite, "
          f"parity vs oracle <= 1e-12 (checked: {CHECK})")
    return OUTPUTS


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--dump", default=None, help="write every output to this .npz")
    ap.add_argument("--compare", default=None, help="require bitwise equality with this .npz")
    a = ap.parse_args()
    outs = main()
    if a.dump:
        np.savez(a.dump, **outs)
    if a.compare:
        ref = np.load(a.compare)
        diff = [k for k in outs if k not in ref.files or not np.array_equal(outs[k], ref[k])]
        print(f"bitwise comparison with {a.compare}: {len(outs) - len(diff)}/{len(outs)} outputs identical")
        assert not diff, f"outputs differ (race?): {diff[:10]}"
