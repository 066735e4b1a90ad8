"""Host-side checks that need no GPU: API validation, input generation, work
model, and the C-ABI library's exported surface."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2504_07042_b200 as hx
from paper_2504_07042_b200 import _native
from paper_2504_07042_b200.axlocal import Equation, FactorSource, KernelSpec

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "hx_axlocal.h")


def test_spec_validation():
    """KernelSpec pairing rules (axlocal.py:67-81; test_axlocal.py:56-66)."""
    with pytest.raises(ValueError):
        KernelSpec(Equation.POISSON, 2, FactorSource.STORED, 3)
    with pytest.raises(ValueError):
        KernelSpec(Equation.POISSON, 1, FactorSource.TRILINEAR_MERGED, 3)
    with pytest.raises(ValueError):
        KernelSpec(Equation.HELMHOLTZ, 1, FactorSource.TRILINEAR_PARTIAL, 3)
    with pytest.raises(ValueError):
        KernelSpec(Equation.POISSON, 1, FactorSource.STORED, 0)
    assert KernelSpec(Equation.HELMHOLTZ, 3, FactorSource.STORED, 4).n1 == 5
    # string and foreign-enum values are accepted like the reference's enums
    s = KernelSpec("poisson", 1, "trilinear", 7)
    assert s.equation is Equation.POISSON and s.factor_source is FactorSource.TRILINEAR_RECOMPUTE


@pytest.mark.parametrize("order", range(1, 16))
def test_product_basis_bitwise_golden(golden, order):
    b = hx.SpectralBasis.build(order)
    assert np.array_equal(b.points, golden[f"basis{order}_points"])
    assert np.array_equal(b.weights, golden[f"basis{order}_weights"])
    assert np.array_equal(b.diff_matrix, golden[f"basis{order}_dmat"])
    assert np.array_equal(b.tensor_weights(), golden[f"basis{order}_tw"])


@pytest.mark.parametrize("name", ["boxA", "boxB", "boxC"])
def test_box_mesh_bitwise_golden(golden, name):
    ex, ey, ez, order, pert, seed = golden[f"{name}_args"]
    m = hx.box_mesh(int(ex), int(ey), int(ez), int(order), perturbation=pert, seed=int(seed))
    assert np.array_equal(m.vertices, golden[f"{name}_verts"])
    assert np.array_equal(m.element_kinds(), golden[f"{name}_kinds"])
    assert np.array_equal(m.local_to_global, golden[f"{name}_l2g"])
    kinds = [el.kind is hx.ElementKind.PARALLELEPIPED for el in m.elements]
    assert kinds == list(golden[f"{name}_kinds"])


def test_box_mesh_slabs_concatenate():
    m = hx.box_mesh(3, 2, 4, 2, perturbation=0.1, seed=1)
    parts = [m.vertices_slab(z, z + 1) for z in range(4)]
    assert np.array_equal(np.concatenate(parts), m.vertices)


def test_box_mesh_rejects_bad_inputs():
    with pytest.raises(ValueError):
        hx.box_mesh(0, 1, 1, 2)
    with pytest.raises(ValueError):
        hx.box_mesh(1, 1, 1, 2, perturbation=0.5)


def test_workload_integers():
    """Hand-evaluated values of the paper's Table 2 (test_workload.py:79-91)."""
    P, H = Equation.POISSON, Equation.HELMHOLTZ
    spec = KernelSpec(P, 1, FactorSource.TRILINEAR_RECOMPUTE, 7)
    wc = hx.workload_count(spec)
    assert (wc.f_ax, wc.f_geo) == (56832, 44416)
    assert hx.workload_count(spec, include_dmat_traffic=False).m_bytes == 8384
    st = hx.workload_count(KernelSpec(P, 1, FactorSource.STORED, 7), include_dmat_traffic=False)
    assert st.m_bytes == 32768 and st.f_geo == 0
    pa = hx.workload_count(KernelSpec(P, 1, FactorSource.TRILINEAR_PARTIAL, 7), include_dmat_traffic=False)
    assert pa.m_bytes == 12480 and pa.f_geo == 72 * 8 + 45 * 64 + 60 * 512
    pp = hx.workload_count(KernelSpec(P, 1, FactorSource.PARALLELEPIPED_RECOMPUTE, 7), include_dmat_traffic=False)
    assert pp.m_bytes == 8240 and pp.f_geo == 7 * 512
    hm = hx.workload_count(KernelSpec(H, 3, FactorSource.TRILINEAR_MERGED, 7))
    assert hm.f_ax == 3 * (12 * 8**4 + 20 * 512)


def test_workload_matches_reference(reference):
    from hosfem.axlocal import Equation as RE, FactorSource as RF, KernelSpec as RK
    from hosfem.workload import workload_count as rwc

    for eq in ("poisson", "helmholtz"):
        for src in ("stored", "trilinear", "trilinear-merged", "trilinear-partial", "parallelepiped"):
            for n_col in (1, 3):
                for order in (1, 3, 7, 15):
                    try:
                        rs = RK(RE(eq), n_col, RF(src), order)
                    except ValueError:
                        continue
                    ours = hx.workload_count(KernelSpec(eq, n_col, src, order), include_dmat_traffic=False)
                    assert ours == type(ours)(**vars(rwc(rs, include_dmat_traffic=False)))


def test_b200_profile_roofline():
    hw = hx.resolve_profile("b200")
    assert hw.peak_general == 37.0e12
    b = hx.roofline_bounds(hx.KernelModel.from_spec(KernelSpec("poisson", 1, "stored", 7)), hw)
    assert b.bound == "memory"
    t = hx.roofline_bounds(hx.KernelModel.from_spec(KernelSpec("poisson", 1, "trilinear", 7)), hw)
    assert t.bound == "compute"


def _header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(hx_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    """The C-ABI .so loads without a GPU and exports exactly what the header declares."""
    declared = _header_functions()
    assert set(declared) == set(_native.SYMBOLS)
    so = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert _native.lib().hx_version().decode().startswith("hx_axlocal")


def test_library_rejects_bad_args_without_gpu():
    """Argument validation happens before any CUDA call (axlocal.py:67-81)."""
    L = _native.lib()
    a = _native.AxArgs(order=7, n_col=2, equation=0, factor_source=1, n_elements=1)
    with pytest.raises(ValueError, match="n_col"):
        _native.check(L.hx_axlocal(ctypes.byref(a), None))
    a = _native.AxArgs(order=7, n_col=1, equation=0, factor_source=2, n_elements=1)
    with pytest.raises(ValueError, match="Helmholtz only"):
        _native.check(L.hx_axlocal(ctypes.byref(a), None))
    a = _native.AxArgs(order=16, n_col=1, equation=0, factor_source=1, n_elements=1)
    with pytest.raises(ValueError, match="order"):
        _native.check(L.hx_axlocal(ctypes.byref(a), None))
    a = _native.AxArgs(order=7, n_col=1, equation=0, factor_source=1, n_elements=0)
    _native.check(L.hx_axlocal(ctypes.byref(a), None))  # E = 0 is a no-op
    if os.environ.get("HX_TUNING", "0") in ("", "0"):
        # the tuning hook field is rejected unless the A/B tools enable it
        a = _native.AxArgs(order=7, n_col=1, equation=0, factor_source=1, n_elements=4, reserved=3)
        with pytest.raises(ValueError, match="reserved"):
            _native.check(L.hx_axlocal(ctypes.byref(a), None))


def test_product_does_not_import_oracle():
    pkg = os.path.dirname(hx.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                assert "oracle" not in open(os.path.join(root, f)).read().replace("no oracle", ""), f


def test_compat_patch_rebinds_reference_entry_points():
    """compat.patch_hosfem swaps hosfem's AxLocal names in every loaded module and restores them."""
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "hosfem")):
        pytest.skip("reference not installed in baseline/_ref")
    import sys

    sys.path.insert(0, ref)
    try:
        import hosfem
        import hosfem.solver

        from paper_2504_07042_b200.compat import patch_hosfem

        orig = hosfem.axlocal.LocalOperator
        restore = patch_hosfem(hosfem)
        assert hosfem.axlocal.LocalOperator is hx.LocalOperator
        assert hosfem.solver.LocalOperator is hx.LocalOperator
        assert hosfem.LocalOperator is hx.LocalOperator
        assert hosfem.axlocal.dense_local_matrix is hx.dense_local_matrix
        restore()
        assert hosfem.axlocal.LocalOperator is orig and hosfem.solver.LocalOperator is orig
        # the reference's own spec objects are accepted as they are
        spec = hosfem.KernelSpec(hosfem.Equation.HELMHOLTZ, 3, hosfem.FactorSource.TRILINEAR_MERGED, 4)
        from paper_2504_07042_b200.axlocal import _as_spec

        ours = _as_spec(spec)
        assert (ours.equation.value, ours.n_col, ours.factor_source.value, ours.order) == ("helmholtz", 3,
                                                                                           "trilinear-merged", 4)
    finally:
        sys.path.remove(ref)
