"""CUDA AxLocal vs the oracle / reference golden vectors (needs a B200).

Bar: fp64 relative difference (verify.py:37-39 metric) <= 1e-12 against the
reference's own outputs, like-for-like variant; bitwise where the reference
promises bitwise (n_col=3 == 3 x n_col=1, run-to-run determinism).
"""

import numpy as np
import pytest

import paper_2504_07042_b200 as hx
from conftest import golden_case, n_golden_cases
from oracle import hosfem_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

DEV = torch.device("cuda", 0)
# 0 = best measured, 1 = slice kernel (Algorithm 4), 2 = fast kernel (specialised / order-generic),
# 4 = DMMA kernel (order 7 only, ax_mma.cu), 5 = j-plane kernel (orders 2, 3, ax_plane.cu)
KERNELS = (0, 1, 2, 4, 5)


def _need(kernel, order):
    if kernel == 4 and order != 7:
        pytest.skip("kernel 4 (DMMA) covers order 7")
    if kernel == 5 and order not in (2, 3):
        pytest.skip("kernel 5 (j-plane) covers orders 2 and 3")


def _op(c, elements, kernel):
    _need(kernel, c["order"])
    spec = hx.KernelSpec(c["equation"], c["n_col"], c["source"], c["order"])
    op = hx.LocalOperator(spec, elements, hx.SpectralBasis.build(c["order"]), lam0=c["lam0"], lam1=c["lam1"])
    op.kernel = kernel
    return op


@pytest.mark.parametrize("kernel", KERNELS + (3,))
@pytest.mark.parametrize("idx", range(n_golden_cases()))
def test_golden_case(golden, idx, kernel):
    c = golden_case(golden, idx)
    if kernel == 3 and c["order"] > 2:
        pytest.skip("kernel 3 (element per thread) covers orders 1 and 2")
    elements = [hx.make_element(v) for v in c["verts"]]
    op = _op(c, elements, kernel)
    got = op.apply(hx.LocalField(c["x"], c["order"])).data
    err = O.rel_diff(got, c["y"])
    assert err <= TOL, (c["order"], c["equation"], c["source"], c["n_col"], err)


@pytest.mark.parametrize("kernel", KERNELS)
def test_device_tensor_path_matches_host_path(golden, kernel):
    c = golden_case(golden, 30)
    op = _op(c, torch.as_tensor(c["verts"], device=DEV), kernel)
    x = torch.as_tensor(c["x"], device=DEV)
    y = op.apply(x)
    assert y.is_cuda and y.shape == x.shape
    assert O.rel_diff(y.cpu().numpy(), c["y"]) <= TOL


def _random_box(order, ex, ey, ez, pert=0.1, seed=0):
    return hx.box_mesh(ex, ey, ez, order, perturbation=pert, seed=seed)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15])
def test_every_order_trilinear_and_stored(order, kernel):
    """All orders N=1..15 (config C3's sweep) on a perturbed box, vs the oracle."""
    _need(kernel, order)
    mesh = _random_box(order, 3, 2, 2, pert=0.15, seed=order)
    rng = np.random.default_rng(order)
    x = rng.standard_normal((mesh.n_elements, (order + 1) ** 3, 1))
    for src in ("trilinear", "stored", "trilinear-partial"):
        op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), mesh, hx.SpectralBasis.build(order))
        op.kernel = kernel
        got = op.apply(torch.as_tensor(x, device=DEV)).cpu().numpy()
        want = O.apply(src, "poisson", order, mesh.vertices, x)
        assert O.rel_diff(got, want) <= TOL, (order, src)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("order", [3, 7, 11])
def test_every_variant_helmholtz_ncol3(order, kernel):
    _need(kernel, order)
    mesh = _random_box(order, 2, 2, 2, pert=0.2, seed=3)
    E, n3 = mesh.n_elements, (order + 1) ** 3
    rng = np.random.default_rng(5)
    x = rng.standard_normal((E, n3, 3))
    lam0 = rng.uniform(0.5, 2.0, (E, n3))
    lam1 = rng.uniform(0.5, 2.0, (E, n3))
    for src in ("stored", "trilinear", "trilinear-merged"):
        op = hx.LocalOperator(hx.KernelSpec("helmholtz", 3, src, order), mesh, hx.SpectralBasis.build(order),
                              lam0=lam0, lam1=lam1)
        op.kernel = kernel
        got = op.apply(torch.as_tensor(x, device=DEV)).cpu().numpy()
        want = O.apply(src, "helmholtz", order, mesh.vertices, x, lam0, lam1)
        assert O.rel_diff(got, want) <= TOL, (order, src)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("order", [2, 7])
def test_parallelepiped_sheared_box(order, kernel):
    """Axis-aligned boxes would hide off-diagonal factor bugs: shear the box."""
    _need(kernel, order)
    mesh = hx.box_mesh(3, 2, 2, order)
    shear = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
    verts = mesh.vertices @ shear.T
    rng = np.random.default_rng(2)
    x = rng.standard_normal((len(verts), (order + 1) ** 3, 1))
    for eq in ("poisson", "helmholtz"):
        op = hx.LocalOperator(hx.KernelSpec(eq, 1, "parallelepiped", order), torch.as_tensor(verts, device=DEV),
                              hx.SpectralBasis.build(order))
        op.kernel = kernel
        got = op.apply(torch.as_tensor(x, device=DEV)).cpu().numpy()
        want = O.apply("parallelepiped", eq, order, verts, x)
        assert O.rel_diff(got, want) <= TOL
        # and the parallelepiped route agrees with the general (stored) route
        want_st = O.apply("stored", eq, order, verts, x)
        assert O.rel_diff(got, want_st) <= 1e-12


@pytest.mark.parametrize("order", [3, 7])
def test_c1_high_aspect_stored_setup(order):
    """C1 (box_mesh(512,1,1,N), elements 1/512 x 1 x 1).  Exact-zero Jacobian entries
    come out of the collocation derivative as rounding noise that the aspect ratio
    amplifies to ~1e-12 of the output (the reference's own stored and parallelepiped
    routes differ by 7.6e-12 here, and numpy/BLAS builds differ at that level).  The
    setup kernel reproduces the reference's rounding of node coordinates and
    derivatives, so it matches the reference's own run (tests/golden/golden_c1.npz,
    every 8th element) to 1e-12."""
    import os

    fx = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_c1.npz"))
    verts = hx.box_mesh(512, 1, 1, order).vertices
    x = np.random.default_rng(0).standard_normal((512, (order + 1) ** 3, 1))
    for src in ("stored", "parallelepiped"):
        op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), torch.as_tensor(verts, device=DEV),
                              hx.SpectralBasis.build(order))
        got = op.apply(torch.as_tensor(x, device=DEV)).cpu().numpy()
        assert O.rel_diff(got[::8], fx[f"n{order}_{src}"]) <= TOL, src


@pytest.mark.parametrize("order", [1, 2])
def test_low_order_element_per_thread_kernel(order):
    """kernel 3: every source / equation / n_col at N = 1, 2 with a ragged element
    count (130: one full and one partial block), vs the oracle; n_col=3 bitwise =
    three n_col=1 applies."""
    mesh = _random_box(order, 13, 5, 2, pert=0.15, seed=order)
    E, n3 = mesh.n_elements, (order + 1) ** 3
    rng = np.random.default_rng(11)
    lam0 = rng.uniform(0.5, 2.0, (E, n3))
    lam1 = rng.uniform(0.5, 2.0, (E, n3))
    shear = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
    ppd = hx.box_mesh(13, 5, 2, order).vertices @ shear.T
    cases = [("poisson", s, mesh.vertices) for s in ("stored", "trilinear", "trilinear-partial")]
    cases += [("helmholtz", s, mesh.vertices) for s in ("stored", "trilinear", "trilinear-merged")]
    cases += [("poisson", "parallelepiped", ppd), ("helmholtz", "parallelepiped", ppd)]
    for eq, src, verts in cases:
        kw = {"lam0": lam0, "lam1": lam1} if eq == "helmholtz" else {}
        x = rng.standard_normal((E, n3, 3))
        op3 = hx.LocalOperator(hx.KernelSpec(eq, 3, src, order), torch.as_tensor(verts, device=DEV),
                               hx.SpectralBasis.build(order), **kw)
        op1 = hx.LocalOperator(hx.KernelSpec(eq, 1, src, order), torch.as_tensor(verts, device=DEV),
                               hx.SpectralBasis.build(order), **kw)
        op3.kernel = op1.kernel = 3
        y3 = op3.apply(torch.as_tensor(x, device=DEV))
        want = O.apply(src, eq, order, verts, x, kw.get("lam0"), kw.get("lam1"))
        assert O.rel_diff(y3.cpu().numpy(), want) <= TOL, (eq, src)
        for c in range(3):
            y1 = op1.apply(torch.as_tensor(x[:, :, c : c + 1].copy(), device=DEV))
            assert torch.equal(y3[:, :, c], y1[:, :, 0]), (eq, src, c)


def test_low_order_kernel_rejects_higher_orders():
    mesh = _random_box(3, 2, 2, 2)
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, "trilinear", 3), mesh, hx.SpectralBasis.build(3))
    op.kernel = 3
    with pytest.raises(ValueError):
        op.apply(torch.zeros((8, 64, 1), dtype=torch.float64, device=DEV))


@pytest.mark.parametrize("kernel", KERNELS)
def test_ncol3_bitwise_equals_three_ncol1(kernel):
    """test_axlocal.py:206-225: factor reuse must not change per-column bits."""
    order = 7
    _need(kernel, order)
    mesh = _random_box(order, 4, 3, 2, seed=9)
    rng = np.random.default_rng(1)
    x = torch.as_tensor(rng.standard_normal((mesh.n_elements, 512, 3)), device=DEV)
    shear = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
    ppd = torch.as_tensor(hx.box_mesh(4, 3, 2, order).vertices @ shear.T, device=DEV)
    E = mesh.n_elements
    kw = {"lam0": rng.uniform(0.5, 2.0, (E, 512)), "lam1": rng.uniform(0.5, 2.0, (E, 512))}
    for eq, src in (("poisson", "trilinear"), ("poisson", "stored"), ("helmholtz", "trilinear-merged"),
                    ("poisson", "trilinear-partial"), ("helmholtz", "trilinear"), ("helmholtz", "stored"),
                    ("poisson", "parallelepiped"), ("helmholtz", "parallelepiped")):
        els = ppd if src == "parallelepiped" else mesh
        k = kw if eq == "helmholtz" else {}
        op3 = hx.LocalOperator(hx.KernelSpec(eq, 3, src, order), els, hx.SpectralBasis.build(order), **k)
        op1 = hx.LocalOperator(hx.KernelSpec(eq, 1, src, order), els, hx.SpectralBasis.build(order), **k)
        op3.kernel = op1.kernel = kernel
        y3 = op3.apply(x)
        for c in range(3):
            y1 = op1.apply(x[:, :, c : c + 1].contiguous())
            assert torch.equal(y3[:, :, c], y1[:, :, 0]), (src, c)


@pytest.mark.parametrize("kernel", [0, 5])
@pytest.mark.parametrize("order", [2, 3])
def test_ncol3_bitwise_small_orders(order, kernel):
    """The j-plane kernel (and the default routing at orders 2, 3): n_col=3 == three
    n_col=1 applies for every source and equation, and the oracle to 1e-12."""
    mesh = _random_box(order, 5, 3, 2, seed=order)
    E, n3 = mesh.n_elements, (order + 1) ** 3
    rng = np.random.default_rng(order)
    x = torch.as_tensor(rng.standard_normal((E, n3, 3)), device=DEV)
    shear = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
    ppd = hx.box_mesh(5, 3, 2, order).vertices @ shear.T
    kw = {"lam0": rng.uniform(0.5, 2.0, (E, n3)), "lam1": rng.uniform(0.5, 2.0, (E, n3))}
    for eq, src in (("poisson", "trilinear"), ("poisson", "trilinear-partial"), ("poisson", "stored"),
                    ("poisson", "parallelepiped"), ("helmholtz", "trilinear"), ("helmholtz", "trilinear-merged"),
                    ("helmholtz", "stored"), ("helmholtz", "parallelepiped")):
        verts = ppd if src == "parallelepiped" else mesh.vertices
        k = kw if eq == "helmholtz" else {}
        op3 = hx.LocalOperator(hx.KernelSpec(eq, 3, src, order), torch.as_tensor(verts, device=DEV),
                               hx.SpectralBasis.build(order), **k)
        op1 = hx.LocalOperator(hx.KernelSpec(eq, 1, src, order), torch.as_tensor(verts, device=DEV),
                               hx.SpectralBasis.build(order), **k)
        op3.kernel = op1.kernel = kernel
        y3 = op3.apply(x)
        want = O.apply(src, eq, order, verts, x.cpu().numpy(), k.get("lam0"), k.get("lam1"))
        assert O.rel_diff(y3.cpu().numpy(), want) <= TOL, (eq, src)
        for c in range(3):
            y1 = op1.apply(x[:, :, c : c + 1].contiguous())
            assert torch.equal(y3[:, :, c], y1[:, :, 0]), (eq, src, c)


@pytest.mark.parametrize("kernel", KERNELS)
def test_run_to_run_bitwise(kernel):
    order = 7
    _need(kernel, order)
    mesh = _random_box(order, 8, 8, 8, seed=4)
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, "trilinear", order), mesh, hx.SpectralBasis.build(order))
    op.kernel = kernel
    x = torch.randn((mesh.n_elements, 512, 1), dtype=torch.float64, device=DEV)
    a = op.apply(x)
    b = op.apply(x)
    assert torch.equal(a, b)


@pytest.mark.parametrize("order", [2, 3, 4, 5, 6, 8, 9, 11, 12, 13, 14, 15])
@pytest.mark.parametrize("dims", [(3, 2, 2), (7, 1, 1), (1, 1, 1)])
def test_role_table_layouts_every_source(order, dims):
    """The order-generic kernel's role-table layouts (fastn_roles.cuh: row / column
    tasks dealt across the elements of a CTA, padding lanes) for every source,
    equation and n_col, at element counts that leave CTAs partly empty; the
    default kernel (0) and the fast kernel (2), against the oracle."""
    mesh = hx.box_mesh(*dims, order, perturbation=0.15, seed=order)
    shear = np.array([[0.9, 0.2, -0.1], [0.0, 1.1, 0.3], [0.15, 0.0, 0.8]])
    ppd_verts = hx.box_mesh(*dims, order).vertices @ shear.T
    E, n3 = mesh.n_elements, (order + 1) ** 3
    rng = np.random.default_rng(order + 100 * dims[0])
    x = rng.standard_normal((E, n3, 3))
    lam0 = rng.uniform(0.5, 2.0, (E, n3))
    lam1 = rng.uniform(0.5, 2.0, (E, n3))
    cases = [("poisson", s) for s in ("trilinear", "trilinear-partial", "stored", "parallelepiped")]
    cases += [("helmholtz", s) for s in ("trilinear", "trilinear-merged", "stored", "parallelepiped")]
    for eq, src in cases:
        verts = ppd_verts if src == "parallelepiped" else mesh.vertices
        kw = {"lam0": lam0, "lam1": lam1} if eq == "helmholtz" else {}
        for n_col in (1, 3):
            xc = np.ascontiguousarray(x[..., :n_col])
            want = O.apply(src, eq, order, verts, xc, **kw)
            for kernel in (0, 2):
                op = hx.LocalOperator(hx.KernelSpec(eq, n_col, src, order), torch.as_tensor(verts, device=DEV),
                                      hx.SpectralBasis.build(order), **kw)
                op.kernel = kernel
                got = op.apply(torch.as_tensor(xc, device=DEV)).cpu().numpy()
                assert O.rel_diff(got, want) <= TOL, (order, dims, eq, src, n_col, kernel)


@pytest.mark.parametrize("E", [1, 2, 3, 5, 7, 33, 149, 300])
def test_ragged_element_counts(E):
    """Element counts that do not fill a CTA / wave (tail handling)."""
    order = 7
    verts = O.box_vertices(E, 1, 1, 0.0, 0)
    verts[..., 0] *= E  # unit cubes in a row
    verts = verts @ np.array([[1.0, 0.1, 0], [0, 1.0, 0.2], [0.05, 0, 1.0]]).T
    verts = verts + np.random.default_rng(E).uniform(-0.05, 0.05, verts.shape)  # make them trilinear
    rng = np.random.default_rng(E)
    x = rng.standard_normal((E, 512, 1))
    for src in ("trilinear", "stored"):
        op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), torch.as_tensor(verts, device=DEV),
                              hx.SpectralBasis.build(order))
        got = op.apply(torch.as_tensor(x, device=DEV)).cpu().numpy()
        assert O.rel_diff(got, O.apply(src, "poisson", order, verts, x)) <= TOL


def test_c2_config_subset_parity():
    """C2 (E=32768 trilinear, 32^3 pert 0.1 seed 0): full GPU apply, oracle on a
    random element subset (elements are independent)."""
    order = 7
    mesh = hx.box_mesh(32, 32, 32, order, perturbation=0.1, seed=0)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((mesh.n_elements, 512, 1))
    sub = np.sort(rng.choice(mesh.n_elements, 512, replace=False))
    for src in ("trilinear", "stored", "trilinear-partial"):
        op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), mesh, hx.SpectralBasis.build(order))
        y = op.apply(torch.as_tensor(x, device=DEV)).cpu().numpy()
        want = O.apply(src, "poisson", order, mesh.vertices[sub], x[sub])
        assert O.rel_diff(y[sub], want) <= TOL, src


@pytest.mark.parametrize("order,counts", [(7, (128, 128, 96)), (15, (58, 58, 58)), (2, (215, 215, 215))])
def test_benchmark_scale_subset_parity(order, counts):
    """At the benchmark scale (C4: 1.57 M elements = 805 M DOF at N=7; ~800 M DOF
    at N=15 and 2) every large-index path runs: full GPU applies, the oracle on a
    random 256-element subset."""
    mesh = hx.box_mesh(*counts, order, perturbation=0.1, seed=0)
    E, n3 = mesh.n_elements, (order + 1) ** 3
    rng = np.random.default_rng(order)
    sub = np.sort(rng.choice(E, 256, replace=False))
    x = torch.randn((E, n3, 1), dtype=torch.float64, device=DEV)
    xs = x[torch.as_tensor(sub, device=DEV)].cpu().numpy()
    verts = mesh.vertices[sub]
    for src in ("trilinear", "stored"):
        op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), mesh, hx.SpectralBasis.build(order))
        y = op.apply(x)
        got = y[torch.as_tensor(sub, device=DEV)].cpu().numpy()
        assert O.rel_diff(got, O.apply(src, "poisson", order, verts, xs)) <= TOL, src
        del op, y
        torch.cuda.empty_cache()


def test_full_size_properties():
    """Size-independent properties at a large size: Poisson annihilates
    constants; the operator is linear and symmetric (u.Av = v.Au per element)."""
    order = 7
    mesh = hx.box_mesh(40, 40, 40, order, perturbation=0.1, seed=0)
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, "trilinear", order), mesh, hx.SpectralBasis.build(order))
    E = mesh.n_elements
    ones = torch.full((E, 512, 1), 3.7, dtype=torch.float64, device=DEV)
    assert op.apply(ones).abs().max().item() <= 1e-10 * 3.7 * 64
    u = torch.randn((E, 512, 1), dtype=torch.float64, device=DEV)
    v = torch.randn((E, 512, 1), dtype=torch.float64, device=DEV)
    au, av = op.apply(u), op.apply(v)
    lin = op.apply(2.0 * u - 0.5 * v)
    assert ((lin - (2.0 * au - 0.5 * av)).abs().max() / lin.abs().max()).item() <= 1e-13
    uav = (u * av).sum(dim=(1, 2))
    vau = (v * au).sum(dim=(1, 2))
    assert ((uav - vau).abs().max() / uav.abs().max()).item() <= 1e-12


def test_geometry_errors():
    order = 3
    bad = O.box_vertices(2, 1, 1, 0.0, 0)
    bad[1, 7] = bad[1, 0] - 0.5  # fold a corner through the element
    for src in ("trilinear", "trilinear-partial"):
        with pytest.raises(hx.GeometryError, match="degenerate element 1"):
            hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), torch.as_tensor(bad, device=DEV),
                             hx.SpectralBasis.build(order))
    with pytest.raises(hx.GeometryError, match="non-positive Jacobian determinant at element 1"):
        hx.LocalOperator(hx.KernelSpec("poisson", 1, "stored", order), torch.as_tensor(bad, device=DEV),
                         hx.SpectralBasis.build(order))


def test_api_errors():
    order = 2
    basis = hx.SpectralBasis.build(order)
    el = hx.make_element(hx.REFERENCE_CUBE + 0.05 * np.random.default_rng(0).uniform(-1, 1, (8, 3)))
    with pytest.raises(ValueError):
        hx.LocalOperator(hx.KernelSpec("poisson", 1, "stored", order), [el], basis, lam1=1.0)
    with pytest.raises(ValueError):
        hx.LocalOperator(hx.KernelSpec("poisson", 1, "parallelepiped", order), [el], basis)
    with pytest.raises(ValueError):
        hx.LocalOperator(hx.KernelSpec("poisson", 1, "stored", 3), [el], basis)
    with pytest.raises(ValueError):
        hx.LocalOperator(hx.KernelSpec("poisson", 1, "stored", order), [], basis)
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, "stored", order), [el], basis)
    with pytest.raises(ValueError):
        op.apply(hx.LocalField(np.zeros((2, 27, 1)), order))
    with pytest.raises(ValueError):
        op.apply(hx.LocalField(np.zeros((1, 27, 3)), order))
    with pytest.raises(ValueError):
        op.apply(hx.LocalField(np.zeros((1, 64, 1)), 3))


def test_mass_limit_reference_cube():
    """lam0=0, lam1=1 on the identity element leaves w_i w_j w_k x (test_axlocal.py:136-150)."""
    order = 3
    basis = hx.SpectralBasis.build(order)
    el = hx.make_element(hx.REFERENCE_CUBE)
    x = np.random.default_rng(0).standard_normal((1, 64, 1))
    for src in ("stored", "trilinear", "trilinear-merged"):
        op = hx.LocalOperator(hx.KernelSpec("helmholtz", 1, src, order), [el], basis, lam0=0.0, lam1=1.0)
        got = op.apply(hx.LocalField(x, order)).data[0, :, 0]
        assert np.abs(got - basis.tensor_weights() * x[0, :, 0]).max() <= 1e-13


def test_apply_inplace_validates_buffers():
    mesh = _random_box(3, 2, 2, 2)
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, "trilinear", 3), mesh, hx.SpectralBasis.build(3))
    x = torch.randn((8, 64, 1), dtype=torch.float64, device=DEV)
    y = torch.empty_like(x)
    op.apply_(x, y)
    assert torch.equal(y, op.apply(x))
    strided = torch.randn((8, 64, 2), dtype=torch.float64, device=DEV)[:, :, :1]  # not contiguous
    for bad in (x.float(), x.cpu(), strided, torch.randn((7, 64, 1), dtype=torch.float64, device=DEV)):
        with pytest.raises(ValueError):
            op.apply_(bad, y)
        with pytest.raises(ValueError):
            op.apply_(x, bad)


@pytest.mark.parametrize("order", [1, 2, 3, 5, 6, 7, 8, 9, 12, 15])
def test_every_family_is_deterministic(order):
    """Shared-memory races show up as run-to-run differences: every kernel family,
    n_col 1 and 3, three applies each, bitwise equal (and all families agree to 1e-12)."""
    mesh = _random_box(order, 5, 3, 2, pert=0.15, seed=order)
    n3 = (order + 1) ** 3
    kernels = (0, 1, 2, 3) if order <= 2 else (0, 1, 2, 4) if order == 7 else (0, 1, 2)
    kernels += (5,) if order in (2, 3) else ()
    for eq, src, ncol in (("poisson", "trilinear", 1), ("helmholtz", "stored", 3), ("poisson", "trilinear-partial", 3)):
        kw = {"lam0": 1.1, "lam1": 0.7} if eq == "helmholtz" else {}
        x = torch.randn((mesh.n_elements, n3, ncol), dtype=torch.float64, device=DEV)
        ref = None
        for kernel in kernels:
            op = hx.LocalOperator(hx.KernelSpec(eq, ncol, src, order), mesh, hx.SpectralBasis.build(order), **kw)
            op.kernel = kernel
            ys = [op.apply(x) for _ in range(3)]
            assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2]), (eq, src, ncol, kernel)
            if ref is None:
                ref = ys[0]
            else:
                assert O.rel_diff(ys[0].cpu().numpy(), ref.cpu().numpy()) <= TOL, (eq, src, ncol, kernel)


@pytest.mark.parametrize("eq", ["poisson", "helmholtz"])
@pytest.mark.parametrize("order", [2, 3])
def test_dense_local_matrix_golden(golden, eq, order):
    """dense_local_matrix (axlocal.py:277-310) against the reference's own matrices."""
    verts = golden[f"dense_{eq}_{order}_verts"]
    got = hx.dense_local_matrix(hx.KernelSpec(eq, 1, "stored", order), hx.make_element(verts),
                                hx.SpectralBasis.build(order))
    assert got.shape == ((order + 1) ** 3,) * 2
    assert O.rel_diff(got, golden[f"dense_{eq}_{order}"]) <= TOL
    with pytest.raises(ValueError):
        hx.dense_local_matrix(hx.KernelSpec("poisson", 1, "stored", order), hx.make_element(verts),
                              hx.SpectralBasis.build(order), lam0=2.0)


def test_sharded_operator_is_bitwise_one_operator():
    """ShardedLocalOperator (devices= wrapper): chunks on several devices (here the one
    GPU twice / three times) give the single operator's result bit for bit."""
    from paper_2504_07042_b200.sharding import ShardedLocalOperator

    order = 5
    mesh = _random_box(order, 5, 4, 3, pert=0.1, seed=6)
    n3 = (order + 1) ** 3
    rng = np.random.default_rng(3)
    lam0 = rng.uniform(0.5, 2.0, (mesh.n_elements, n3))
    spec = hx.KernelSpec("helmholtz", 1, "trilinear", order)
    one = hx.LocalOperator(spec, mesh, hx.SpectralBasis.build(order), lam0=lam0, lam1=0.3)
    x = rng.standard_normal((mesh.n_elements, n3, 1))
    want = one.apply(torch.as_tensor(x, device=DEV))
    for parts in (2, 3):
        sh = ShardedLocalOperator(spec, mesh, hx.SpectralBasis.build(order), lam0=lam0, lam1=0.3,
                                  devices=[DEV] * parts)
        assert torch.equal(sh.apply(torch.as_tensor(x, device=DEV)), want)
        got = sh.apply(hx.LocalField(x, order))
        assert np.array_equal(got.data, want.cpu().numpy())


def test_graphed_apply_matches_eager():
    mesh = hx.box_mesh(512, 1, 1, 7)  # C1: 512 small elements, launch-overhead bound
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, "parallelepiped", 7), mesh, hx.SpectralBasis.build(7))
    x = torch.randn((512, 512, 1), dtype=torch.float64, device=DEV)
    y = torch.empty_like(x)
    replay = op.graphed(x, y, applies=3)
    want = op.apply(x)
    y.zero_()
    replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)
    x.copy_(torch.randn_like(x))  # the graph reads the buffer's current contents
    replay()
    torch.cuda.synchronize()
    assert torch.equal(y, op.apply(x))


def test_order7_setup_kernels_match_the_generic_order(monkeypatch):
    """The N=7 setup kernels (stored factors at a compile-time order, trilinear
    route one thread per k-fibre) produce bit for bit the generic-order
    kernels' fields, and report the same first bad node."""
    mesh = hx.box_mesh(9, 7, 5, 7, perturbation=0.15, seed=11)
    verts = mesh.vertices_device(DEV)
    E = verts.shape[0]
    rng = np.random.default_rng(12)
    l0 = torch.as_tensor(rng.uniform(0.5, 2.0, (E, 512)), device=DEV)
    l1 = torch.as_tensor(rng.uniform(0.5, 2.0, (E, 512)), device=DEV)
    basis = hx.SpectralBasis.build(7)

    def fields():
        st = hx.LocalOperator(hx.KernelSpec("helmholtz", 1, "stored", 7), verts, basis, lam0=1.1, lam1=0.4)
        pa = hx.LocalOperator(hx.KernelSpec("poisson", 1, "trilinear-partial", 7), verts, basis)
        me = hx.LocalOperator(hx.KernelSpec("helmholtz", 1, "trilinear-merged", 7), verts, basis, lam0=l0, lam1=l1)
        return [st._g.clone(), st._gwj.clone(), pa._lam_geo.clone(), me._lam2.clone(), me._lam3.clone()]

    def first_bad():
        bad = mesh.vertices.copy()
        bad[23] = bad[23][[1, 0, 3, 2, 5, 4, 7, 6]]
        msgs = []
        for src in ("trilinear", "stored"):
            with pytest.raises(hx.GeometryError) as ex:
                hx.LocalOperator(hx.KernelSpec("poisson", 1, src, 7), torch.as_tensor(bad, device=DEV), basis)
            msgs.append(str(ex.value))
        return msgs

    fast, fast_bad = fields(), first_bad()
    monkeypatch.setenv("HX_SETUP_GENERIC", "1")
    generic, generic_bad = fields(), first_bad()
    for a, b in zip(fast, generic):
        assert torch.equal(a, b)
    assert fast_bad == generic_bad
