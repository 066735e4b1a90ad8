"""Pin the CPU oracle: golden vectors produced by the reference itself, and the
live reference where it is present.  (No GPU needed.)"""

import numpy as np
import pytest

from conftest import golden_case, n_golden_cases
from oracle import hosfem_oracle as O


@pytest.mark.parametrize("order", range(1, 16))
def test_basis_bitwise(golden, order):
    pts, w, d = O.gll_basis(order)
    assert np.array_equal(pts, golden[f"basis{order}_points"])
    assert np.array_equal(w, golden[f"basis{order}_weights"])
    assert np.array_equal(d, golden[f"basis{order}_dmat"])
    assert np.array_equal(O.tensor_weights(w), golden[f"basis{order}_tw"])


@pytest.mark.parametrize("name", ["boxA", "boxB", "boxC"])
def test_box_vertices_bitwise(golden, name):
    ex, ey, ez, order, pert, seed = golden[f"{name}_args"]
    verts = O.box_vertices(int(ex), int(ey), int(ez), pert, int(seed))
    assert np.array_equal(verts, golden[f"{name}_verts"])
    kinds = np.array([O.is_parallelepiped(v) for v in verts])
    assert np.array_equal(kinds, golden[f"{name}_kinds"])


@pytest.mark.parametrize("idx", range(n_golden_cases()))
def test_oracle_matches_reference_golden(golden, idx):
    c = golden_case(golden, idx)
    got = O.apply(c["source"], c["equation"], c["order"], c["verts"], c["x"], c["lam0"], c["lam1"])
    # the restatement keeps the reference's operation order: agreement is
    # bitwise on this machine; allow a few ulps for other BLAS builds
    assert O.rel_diff(got, c["y"]) <= 1e-14, c


@pytest.mark.parametrize("eq", ["poisson", "helmholtz"])
@pytest.mark.parametrize("order", [2, 3])
def test_dense_matrix_golden(golden, eq, order):
    got = O.dense_matrix(eq, order, golden[f"dense_{eq}_{order}_verts"])
    assert O.rel_diff(got, golden[f"dense_{eq}_{order}"]) <= 1e-14


def test_oracle_threads_bitwise():
    rng = np.random.default_rng(3)
    verts = O.box_vertices(3, 2, 2, 0.2, 1)
    x = rng.standard_normal((len(verts), 4**3, 1))
    one = O.apply("trilinear", "poisson", 3, verts, x, threads=1)
    four = O.apply("trilinear", "poisson", 3, verts, x, threads=4)
    assert np.array_equal(one, four)


def test_oracle_vs_dense_every_variant():
    """matrix-free oracle vs the assembled matrix (test_axlocal.py:85-103)."""
    rng = np.random.default_rng(11)
    order = 3
    verts = O.box_vertices(2, 2, 1, 0.2, 4)
    x = rng.standard_normal((len(verts), 64, 1))
    for eq, srcs in (("poisson", ("stored", "trilinear", "trilinear-partial")),
                     ("helmholtz", ("stored", "trilinear", "trilinear-merged"))):
        want = np.stack([O.dense_matrix(eq, order, v) @ x[e] for e, v in enumerate(verts)])
        for s in srcs:
            assert O.rel_diff(O.apply(s, eq, order, verts, x), want) <= 1e-12


def test_oracle_live_reference_random(reference):
    """Fresh random cases against the live reference (build container only)."""
    from hosfem.axlocal import Equation, FactorSource, KernelSpec, LocalOperator
    from hosfem.basis import SpectralBasis
    from hosfem.mesh import LocalField, box_mesh

    rng = np.random.default_rng(99)
    for order, src, eq in ((4, "trilinear", "helmholtz"), (6, "trilinear-partial", "poisson"), (8, "stored", "helmholtz")):
        mesh = box_mesh(2, 2, 2, order, perturbation=0.15, seed=order)
        verts = np.stack([el.vertices for el in mesh.elements])
        x = rng.standard_normal((len(verts), (order + 1) ** 3, 3))
        kw = {"lam0": 1.3, "lam1": 0.7} if eq == "helmholtz" else {}
        op = LocalOperator(KernelSpec(Equation(eq), 3, FactorSource(src), order), mesh.elements,
                           SpectralBasis.build(order), **kw)
        want = op.apply(LocalField(x, order)).data
        got = O.apply(src, eq, order, verts, x, kw.get("lam0"), kw.get("lam1"))
        assert np.array_equal(got, want)


def test_mutation_is_detected(golden):
    """A 1e-6 corruption of one factor must fail the parity bar (test_cli.py:32-51 pattern)."""
    c = golden_case(golden, 3)
    y = O.apply(c["source"], c["equation"], c["order"], c["verts"], c["x"], c["lam0"], c["lam1"])
    bad = y * (1 + 1e-6)
    assert O.rel_diff(bad, c["y"]) > 1e-12


@pytest.mark.parametrize("order", [3, 7])
def test_oracle_c1_fixture(order):
    """C1 (512 x 1 x 1 high-aspect box) against the reference's own run: ppd to
    round-off; stored within the level at which numpy / BLAS builds differ on this
    ill-conditioned input (bitwise in the build container)."""
    import os

    fx = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_c1.npz"))
    verts = O.box_vertices(512, 1, 1, 0.0, 0)
    x = np.random.default_rng(0).standard_normal((512, (order + 1) ** 3, 1))[::8]
    assert O.rel_diff(O.apply("parallelepiped", "poisson", order, verts[::8], x), fx[f"n{order}_parallelepiped"]) <= 1e-14
    assert O.rel_diff(O.apply("stored", "poisson", order, verts[::8], x), fx[f"n{order}_stored"]) <= 2e-11
