"""Element containers and the synthetic box-mesh generator (operator inputs).

Mirrors the reference containers the AxLocal operator consumes
(pkg/src/hosfem/mesh.py): ``Element`` (67-78), ``ElementKind`` (61-64),
``make_element`` (97-107), ``parallelepiped_defect`` (81-94), ``LocalField``
(140-176) and ``box_mesh`` (214-283), with the same conventions:

* node (i, j, k) of an element is flat index i + j n1 + k n1^2;
* vertex b sits at reference corner (bit0 -> r, bit1 -> s, bit2 -> t);
* box elements are ordered cx fastest, then cy, then cz (so contiguous element
  ranges are z-slabs, the unit of multi-GPU sharding);
* ``box_mesh`` reproduces the reference's corner jitter draw exactly:
  one ``default_rng(seed).uniform(-1, 1, (ex+1, ey+1, ez+1, 3))`` scaled by
  ``perturbation * h`` and masked to interior corners (mesh.py:245-251).

Unlike the reference, a box mesh here is array-backed: vertices live in one
(E, 8, 3) fp64 array (built vectorised, optionally straight on the GPU),
``elements`` and ``local_to_global`` are materialised only on demand — the
reference's O(E) Python loop cannot build the 1.5 M-element configuration.

``Mesh`` / ``save_mesh`` / ``load_mesh`` read and write the reference's
plain-text mesh format (mesh.py:185-211, 336-402) byte for byte, array-backed
as well (tests/test_mesh_io.py checks files written by the reference).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "ElementKind",
    "Element",
    "LocalField",
    "BoxMesh",
    "REFERENCE_CUBE",
    "parallelepiped_defect",
    "parallelepiped_defects",
    "make_element",
    "element_node_coords",
    "box_mesh",
    "box_corners",
    "Mesh",
    "MeshFormatError",
    "save_mesh",
    "load_mesh",
]

REFERENCE_CUBE = np.array(
    [[(1.0 if b & 1 else -1.0), (1.0 if b & 2 else -1.0), (1.0 if b & 4 else -1.0)] for b in range(8)]
)
REFERENCE_CUBE.flags.writeable = False


class ElementKind(enum.Enum):
    GENERAL = "general"
    TRILINEAR = "trilinear"
    PARALLELEPIPED = "parallelepiped"


@dataclass(frozen=True)
class Element:
    """One hexahedron: (8, 3) fp64 vertices plus its shape class."""

    vertices: np.ndarray
    kind: ElementKind

    def __post_init__(self):
        v = np.asarray(self.vertices, dtype=float)
        if v.shape != (8, 3):
            raise ValueError("element vertices must form an (8, 3) array")
        object.__setattr__(self, "vertices", v)


def parallelepiped_defects(verts: np.ndarray) -> np.ndarray:
    """Per-element max deviation from v3=v1+v2-v0, v5=v1+v4-v0, v6=v2+v4-v0,
    v7=v1+v2+v4-2v0 for a (E, 8, 3) batch (reference mesh.py:81-94)."""
    v = np.asarray(verts, dtype=float)
    v0, v1, v2, v4 = v[:, 0], v[:, 1], v[:, 2], v[:, 4]
    preds = (
        np.abs(v[:, 3] - (v1 + v2 - v0)),
        np.abs(v[:, 5] - (v1 + v4 - v0)),
        np.abs(v[:, 6] - (v2 + v4 - v0)),
        np.abs(v[:, 7] - (v1 + v2 + v4 - 2.0 * v0)),
    )
    return np.max(np.stack([p.max(axis=-1) for p in preds]), axis=0)


def parallelepiped_defect(vertices: np.ndarray) -> float:
    return float(parallelepiped_defects(np.asarray(vertices, dtype=float)[None])[0])


def _kinds_from_defects(verts: np.ndarray, tol: float = 1e-12) -> np.ndarray:
    """True where the element classifies as a parallelepiped (mesh.py:105-106)."""
    scale = np.maximum(1.0, np.abs(verts).reshape(len(verts), -1).max(axis=1))
    return parallelepiped_defects(verts) <= tol * scale


def make_element(vertices: np.ndarray, tol: float = 1e-12) -> Element:
    v = np.asarray(vertices, dtype=float)
    if v.shape != (8, 3):
        raise ValueError("an element needs 8 vertices with 3 coordinates each")
    ppd = bool(_kinds_from_defects(v[None], tol)[0])
    return Element(vertices=v, kind=ElementKind.PARALLELEPIPED if ppd else ElementKind.TRILINEAR)


def element_node_coords(element: Element, basis) -> np.ndarray:
    """(n1^3, 3) physical coordinates of the GLL nodes under the trilinear map."""
    xi = basis.points
    lo, hi = 0.5 * (1.0 - xi), 0.5 * (1.0 + xi)
    n1 = len(xi)
    out = np.zeros((n1, n1, n1, 3))
    for b in range(8):
        fr = hi if b & 1 else lo
        fs = hi if b & 2 else lo
        ft = hi if b & 4 else lo
        out += (ft[:, None, None] * fs[None, :, None] * fr[None, None, :])[..., None] * element.vertices[b]
    return out.reshape(n1**3, 3)


@dataclass
class LocalField:
    """Element-local nodal data of shape (E, n1**3, n_col) (reference mesh.py:140-176).

    ``data`` is a numpy array (host) as in the reference; the GPU operator also
    accepts and returns torch CUDA tensors of the same shape directly.
    """

    data: np.ndarray
    order: int

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=float)
        if self.data.ndim == 2:
            self.data = self.data[:, :, None]
        if self.data.ndim != 3:
            raise ValueError("local field data must have shape (E, n1**3, n_col)")
        n3 = (self.order + 1) ** 3
        if self.data.shape[1] != n3:
            raise ValueError(f"expected {n3} nodes per element, got {self.data.shape[1]}")

    @property
    def n_elements(self) -> int:
        return self.data.shape[0]

    @property
    def n_col(self) -> int:
        return self.data.shape[2]

    @property
    def n1(self) -> int:
        return self.order + 1

    @classmethod
    def zeros(cls, n_elements: int, order: int, n_col: int = 1) -> "LocalField":
        return cls(np.zeros((n_elements, (order + 1) ** 3, n_col)), order)

    def cube(self, e: int, col: int = 0) -> np.ndarray:
        n1 = self.n1
        return self.data[e, :, col].reshape(n1, n1, n1)


def box_corners(ex, ey, ez, extents=((0.0, 1.0), (0.0, 1.0), (0.0, 1.0)), perturbation=0.0, seed=0):
    """(ex+1, ey+1, ez+1, 3) corner lattice with the reference's jitter draw."""
    if min(ex, ey, ez) < 1:
        raise ValueError("element counts must be at least 1")
    if not 0.0 <= perturbation:
        raise ValueError("perturbation must be nonnegative")
    if perturbation >= 0.5:
        raise ValueError("perturbation must be below 0.5 (inverted-element risk)")
    counts = (ex, ey, ez)
    lows = [float(lo) for lo, _ in extents]
    span = [float(hi) - float(lo) for lo, hi in extents]
    axes = [lows[d] + span[d] * np.arange(counts[d] + 1) / counts[d] for d in range(3)]
    corners = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)
    if perturbation > 0.0:
        rng = np.random.default_rng(seed)
        h = np.array([span[d] / counts[d] for d in range(3)])
        jitter = rng.uniform(-1.0, 1.0, corners.shape) * (perturbation * h)
        interior = np.zeros(corners.shape[:3], dtype=bool)
        interior[1:-1, 1:-1, 1:-1] = True
        corners = corners + jitter * interior[..., None]
    return corners


def _element_vertices_np(corners: np.ndarray, z0: int = 0, z1: int | None = None) -> np.ndarray:
    ex, ey, ez = (s - 1 for s in corners.shape[:3])
    z1 = ez if z1 is None else z1
    cx, cy, cz = np.meshgrid(np.arange(ex), np.arange(ey), np.arange(z0, z1), indexing="ij")
    # element order cx fastest, then cy, then cz
    cx, cy, cz = (a.transpose(2, 1, 0).ravel() for a in (cx, cy, cz))
    verts = np.empty((cx.size, 8, 3))
    for b in range(8):
        verts[:, b] = corners[cx + (b & 1), cy + ((b >> 1) & 1), cz + ((b >> 2) & 1)]
    return verts


@dataclass
class BoxMesh:
    """Structured ex x ey x ez box of order-N hexahedra, array-backed."""

    counts: tuple
    order: int
    corners: np.ndarray
    perturbation: float = 0.0
    _vertices: np.ndarray | None = field(default=None, repr=False)

    @property
    def n_elements(self) -> int:
        ex, ey, ez = self.counts
        return ex * ey * ez

    @property
    def lattice_shape(self) -> tuple:
        ex, ey, ez = self.counts
        n = self.order
        return (ex * n + 1, ey * n + 1, ez * n + 1)

    @property
    def global_node_count(self) -> int:
        nx, ny, nz = self.lattice_shape
        return nx * ny * nz

    @property
    def vertices(self) -> np.ndarray:
        """(E, 8, 3) fp64 vertex array (host)."""
        if self._vertices is None:
            self._vertices = _element_vertices_np(self.corners)
        return self._vertices

    def vertices_slab(self, z0: int, z1: int) -> np.ndarray:
        """Vertices of the contiguous element range of z-layers [z0, z1)."""
        return _element_vertices_np(self.corners, z0, z1)

    def vertices_device(self, device, z0: int = 0, z1: int | None = None):
        """(E_slab, 8, 3) vertices assembled on the GPU from the corner lattice."""
        import torch

        ex, ey, ez = self.counts
        z1 = ez if z1 is None else z1
        c = torch.as_tensor(self.corners[:, :, z0 : z1 + 1], dtype=torch.float64, device=device)
        cz, cy, cx = torch.meshgrid(
            torch.arange(z1 - z0, device=device),
            torch.arange(ey, device=device),
            torch.arange(ex, device=device),
            indexing="ij",
        )
        cx, cy, cz = cx.reshape(-1), cy.reshape(-1), cz.reshape(-1)
        parts = [c[cx + (b & 1), cy + ((b >> 1) & 1), cz + ((b >> 2) & 1)] for b in range(8)]
        return torch.stack(parts, dim=1).contiguous()

    def element_kinds(self) -> np.ndarray:
        """True where an element is a parallelepiped (make_element's rule)."""
        return _kinds_from_defects(self.vertices)

    @property
    def elements(self) -> tuple:
        """Reference-style tuple of Element objects (built on demand)."""
        verts = self.vertices
        ppd = _kinds_from_defects(verts)
        return tuple(
            Element(vertices=verts[e], kind=ElementKind.PARALLELEPIPED if ppd[e] else ElementKind.TRILINEAR)
            for e in range(len(verts))
        )

    @property
    def local_to_global(self) -> np.ndarray:
        """(E, n1^3) int64 lattice numbering (reference mesh.py:271-274)."""
        ex, ey, ez = self.counts
        n = self.order
        n1 = n + 1
        nx, ny, _ = self.lattice_shape
        li = np.arange(n1)
        kk, jj, ii = np.meshgrid(li, li, li, indexing="ij")
        cz, cy, cx = np.meshgrid(np.arange(ez), np.arange(ey), np.arange(ex), indexing="ij")
        cx, cy, cz = cx.ravel()[:, None], cy.ravel()[:, None], cz.ravel()[:, None]
        gx = cx * n + ii.ravel()[None]
        gy = cy * n + jj.ravel()[None]
        gz = cz * n + kk.ravel()[None]
        return ((gz * ny + gy) * nx + gx).astype(np.int64)


def box_mesh(ex, ey, ez, order, extents=((0.0, 1.0), (0.0, 1.0), (0.0, 1.0)), perturbation=0.0, seed=0) -> BoxMesh:
    """Same inputs and jitter draw as the reference's box_mesh (mesh.py:214-283)."""
    if order < 1:
        raise ValueError("order must be at least 1")
    corners = box_corners(ex, ey, ez, extents, perturbation, seed)
    return BoxMesh(counts=(ex, ey, ez), order=order, corners=corners, perturbation=perturbation)


_KIND_BY_NAME = {k.value: k for k in ElementKind}


class MeshFormatError(ValueError):
    """A malformed mesh file (reference mesh.py:336-337)."""


@dataclass(frozen=True, eq=False)
class Mesh:
    """A conforming hexahedral mesh plus its local-to-global node map (reference mesh.py:185-211).

    Array-backed: ``vertices`` (E, 8, 3) fp64 and ``kinds`` (E,) of ``ElementKind``
    values; ``elements`` builds the reference's Element tuple on demand.
    """

    vertices: np.ndarray
    kinds: tuple
    order: int
    local_to_global: np.ndarray
    global_node_count: int
    lattice_shape: tuple | None = None

    def __post_init__(self):
        v = np.ascontiguousarray(self.vertices, dtype=np.float64)
        if v.ndim != 3 or v.shape[1:] != (8, 3):
            raise ValueError("vertices must have shape (E, 8, 3)")
        kinds = tuple(ElementKind(k) for k in self.kinds)
        if len(kinds) != v.shape[0]:
            raise ValueError("one kind per element")
        l2g = np.asarray(self.local_to_global, dtype=np.int64)
        n3 = (self.order + 1) ** 3
        if l2g.shape != (v.shape[0], n3):
            raise ValueError("local_to_global must have shape (E, n1**3)")
        if l2g.min(initial=0) < 0 or (l2g.size and l2g.max() >= self.global_node_count):
            raise ValueError("local_to_global entries out of range")
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "kinds", kinds)
        object.__setattr__(self, "local_to_global", l2g)
        if self.lattice_shape is not None:
            object.__setattr__(self, "lattice_shape", tuple(int(n) for n in self.lattice_shape))

    @classmethod
    def from_elements(cls, elements, order, local_to_global, global_node_count, lattice_shape=None) -> "Mesh":
        elements = tuple(elements)
        verts = np.stack([el.vertices for el in elements]) if elements else np.zeros((0, 8, 3))
        return cls(verts, tuple(el.kind for el in elements), order, local_to_global, global_node_count, lattice_shape)

    @classmethod
    def from_box(cls, box: "BoxMesh") -> "Mesh":
        ppd = _kinds_from_defects(box.vertices)
        kinds = tuple(ElementKind.PARALLELEPIPED if p else ElementKind.TRILINEAR for p in ppd)
        return cls(box.vertices, kinds, box.order, box.local_to_global, box.global_node_count, box.lattice_shape)

    @property
    def n_elements(self) -> int:
        return self.vertices.shape[0]

    @property
    def elements(self) -> tuple:
        return tuple(Element(vertices=self.vertices[e], kind=k) for e, k in enumerate(self.kinds))

    def multiplicity(self) -> np.ndarray:
        """How many element-local nodes map onto each global node (reference mesh.py:209-211)."""
        return np.bincount(self.local_to_global.ravel(), minlength=self.global_node_count)


def save_mesh(mesh, path) -> None:
    """Write ``mesh`` (a Mesh or BoxMesh) in the reference's text format (mesh.py:340-353).

    Floats are written with Python's shortest round-trip ``repr`` like the
    reference, so files are byte-identical and reload bit-exactly.
    """
    if isinstance(mesh, BoxMesh):
        mesh = Mesh.from_box(mesh)
    lines = ["hosfem-mesh v1", f"order {mesh.order}", f"elements {mesh.n_elements}", f"nodes {mesh.global_node_count}"]
    if mesh.lattice_shape is not None:
        lines.append("lattice {} {} {}".format(*mesh.lattice_shape))
    rows = mesh.vertices.reshape(-1, 3).tolist()
    for e, kind in enumerate(mesh.kinds):
        lines.append(f"element {e} {kind.value}")
        lines.extend(" ".join(map(repr, r)) for r in rows[8 * e : 8 * e + 8])
    lines.append("connectivity")
    lines.extend(" ".join(map(str, r)) for r in mesh.local_to_global.tolist())
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def load_mesh(path) -> Mesh:
    """Parse a mesh written by ``save_mesh`` (either implementation; reference mesh.py:356-402).

    Same acceptance rules and error type (``MeshFormatError``) as the reference.
    """
    with open(path) as fh:
        raw = [ln.strip() for ln in fh if ln.strip()]
    pos = 0

    def take():
        nonlocal pos
        if pos >= len(raw):
            return ""
        pos += 1
        return raw[pos - 1]

    if (raw[0] if raw else None) != "hosfem-mesh v1":
        raise MeshFormatError("not a hosfem mesh file")
    pos = 1

    def expect(key):
        parts = (line := take()).split()
        if not parts or parts[0] != key:
            raise MeshFormatError(f"expected '{key}' line, got {line!r}")
        return parts[1:]

    try:
        order = int(expect("order")[0])
        n_elements = int(expect("elements")[0])
        n_nodes = int(expect("nodes")[0])
        lattice = None
        line = take()
        if line.startswith("lattice"):
            lattice = tuple(int(v) for v in line.split()[1:4])
            line = take()
        verts = np.empty((n_elements, 8, 3))
        kinds = []
        for e in range(n_elements):
            head = line.split()
            if len(head) != 3 or head[0] != "element" or int(head[1]) != e:
                raise MeshFormatError(f"malformed element header for element {e}")
            if head[2] not in _KIND_BY_NAME:
                raise MeshFormatError(f"unknown element kind {head[2]!r}")
            kinds.append(_KIND_BY_NAME[head[2]])
            if pos + 8 > len(raw):
                raise MeshFormatError(f"truncated vertices for element {e}")
            block = [r.split() for r in raw[pos : pos + 8]]
            if any(len(r) != 3 for r in block):
                raise MeshFormatError(f"malformed vertex line in element {e}")
            verts[e] = np.array(block, dtype=np.float64)
            pos += 8
            line = take()
        if line != "connectivity":
            raise MeshFormatError("missing connectivity section")
        if pos + n_elements > len(raw):
            raise MeshFormatError("truncated connectivity section")
        conn = raw[pos : pos + n_elements]
        l2g = np.array([r.split() for r in conn], dtype=np.int64) if n_elements else np.zeros((0, (order + 1) ** 3))
    except (IndexError, ValueError) as exc:
        if isinstance(exc, MeshFormatError):
            raise
        raise MeshFormatError(str(exc)) from exc
    return Mesh(verts, tuple(kinds), order, l2g, n_nodes, lattice)
