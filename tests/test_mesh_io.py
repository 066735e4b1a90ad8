"""Mesh container and the reference's text mesh format (reference mesh.py:185-211,
336-402; its tests test_mesh.py:177-198), against files written by the reference
itself (tests/golden/make_mesh_golden.py)."""

import os

import numpy as np
import pytest

import paper_2504_07042_b200 as hx
from oracle import hosfem_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = {
    "mesh_box_2x1x1_n3.txt": ((2, 1, 1, 3), dict(perturbation=0.17, seed=4)),
    "mesh_box_3x2x2_n2.txt": ((3, 2, 2, 2), dict(perturbation=0.2, seed=5)),
    "mesh_box_2x2x1_n1_affine.txt": ((2, 2, 1, 1), dict(extents=((0.0, 2.0), (-1.0, 1.0), (0.0, 0.5)))),
}


@pytest.mark.parametrize("name", sorted(FILES))
def test_reads_reference_file_and_writes_same_bytes(name, tmp_path):
    path = os.path.join(GOLDEN, name)
    mesh = hx.load_mesh(path)
    out = tmp_path / "m.txt"
    hx.save_mesh(mesh, out)
    assert out.read_bytes() == open(path, "rb").read()


@pytest.mark.parametrize("name", sorted(FILES))
def test_box_mesh_saves_like_reference(name, tmp_path):
    args, kw = FILES[name]
    out = tmp_path / "m.txt"
    hx.save_mesh(hx.box_mesh(*args, **kw), out)
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()
    back = hx.load_mesh(out)
    ex, ey, ez, order = args
    assert back.lattice_shape == (ex * order + 1, ey * order + 1, ez * order + 1)
    assert np.array_equal(back.local_to_global, O.box_l2g(ex, ey, ez, order))
    assert np.array_equal(back.vertices, hx.box_mesh(*args, **kw).vertices)  # repr round-trips exactly


def test_round_trip_like_reference(tmp_path):
    box = hx.box_mesh(2, 1, 1, 3, perturbation=0.17, seed=4)
    path = tmp_path / "mesh.txt"
    hx.save_mesh(box, path)
    back = hx.load_mesh(path)
    assert back.order == box.order
    assert back.global_node_count == box.global_node_count
    assert back.lattice_shape == box.lattice_shape
    assert np.array_equal(back.local_to_global, box.local_to_global)
    for a, b in zip(back.elements, box.elements):
        assert a.kind is b.kind
        assert np.array_equal(a.vertices, b.vertices)
    assert np.array_equal(back.multiplicity(), np.bincount(box.local_to_global.ravel()))


def test_rejects_garbage(tmp_path):
    path = tmp_path / "bad.txt"
    path.write_text("not a mesh\n")
    with pytest.raises(hx.MeshFormatError):
        hx.load_mesh(path)
    path.write_text("hosfem-mesh v1\norder 2\nelements 1\nnodes 27\n")
    with pytest.raises(hx.MeshFormatError):
        hx.load_mesh(path)
    good = open(os.path.join(GOLDEN, "mesh_box_2x1x1_n3.txt")).read().splitlines()
    for bad in (
        good[:-1],                                    # truncated connectivity
        [ln for ln in good if ln != "connectivity"],  # missing section
        [ln.replace("element 1", "element 7") for ln in good],
        [ln.replace("parallelepiped", "prism") for ln in good],
    ):
        path.write_text("\n".join(bad) + "\n")
        with pytest.raises(hx.MeshFormatError):
            hx.load_mesh(path)
    path.write_text("")
    with pytest.raises(hx.MeshFormatError):
        hx.load_mesh(path)


def test_mesh_validation():
    box = hx.box_mesh(2, 1, 1, 2)
    m = hx.Mesh.from_box(box)
    with pytest.raises(ValueError):
        hx.Mesh(m.vertices, m.kinds, 3, m.local_to_global, m.global_node_count)
    with pytest.raises(ValueError):
        hx.Mesh(m.vertices, m.kinds, 2, m.local_to_global, 5)
    with pytest.raises(ValueError):
        hx.Mesh(m.vertices[:, :7], m.kinds, 2, m.local_to_global, m.global_node_count)
    m2 = hx.Mesh.from_elements(m.elements, 2, m.local_to_global, m.global_node_count, m.lattice_shape)
    assert m2.kinds == m.kinds and np.array_equal(m2.vertices, m.vertices)


@pytest.mark.gpu
def test_operator_accepts_loaded_mesh():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mesh = hx.load_mesh(os.path.join(GOLDEN, "mesh_box_3x2x2_n2.txt"))
    order = mesh.order
    x = np.random.default_rng(0).standard_normal((mesh.n_elements, (order + 1) ** 3, 1))
    for src in ("trilinear", "stored"):
        op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, order), mesh, hx.SpectralBasis.build(order))
        got = op.apply(hx.LocalField(x, order)).data
        want = O.apply(src, "poisson", order, mesh.vertices, x)
        assert O.rel_diff(got, want) <= 1e-12
