"""B200-native AxLocal (CEED BK5) — drop-in for the reference ``hosfem`` operator path.

Public names follow ``hosfem`` (reference pkg/src/hosfem/__init__.py): the
operator (``LocalOperator``, ``ax_local_apply``, ``KernelSpec``, ``Equation``,
``FactorSource``), its inputs (``SpectralBasis``, ``Element``, ``ElementKind``,
``LocalField``, ``make_element``, ``box_mesh``), and the work model used for
roofline reporting (``workload_count``, ``roofline_bounds``).
"""

from .axlocal import (
    Equation,
    FactorSource,
    GeometryError,
    KernelSpec,
    LocalOperator,
    ax_local_apply,
    dense_local_matrix,
)
from .basis import SpectralBasis
from .mesh import (
    REFERENCE_CUBE,
    BoxMesh,
    Element,
    ElementKind,
    LocalField,
    Mesh,
    MeshFormatError,
    box_mesh,
    element_node_coords,
    load_mesh,
    save_mesh,
    make_element,
    parallelepiped_defect,
)
from .sharding import ShardedLocalOperator
from .workload import WorkloadCount, ax_flops, geo_flops, workload_count
from .roofline import (
    HardwareProfile,
    KernelModel,
    RooflineBounds,
    load_profile,
    machine_balance,
    mbp_crossing,
    measured_performance,
    operational_intensity,
    preset_names,
    resolve_profile,
    roofline_bounds,
)

__version__ = "0.1.0"

__all__ = [
    "Equation",
    "FactorSource",
    "GeometryError",
    "KernelSpec",
    "LocalOperator",
    "ax_local_apply",
    "dense_local_matrix",
    "SpectralBasis",
    "REFERENCE_CUBE",
    "BoxMesh",
    "Element",
    "ElementKind",
    "LocalField",
    "Mesh",
    "MeshFormatError",
    "load_mesh",
    "save_mesh",
    "box_mesh",
    "element_node_coords",
    "make_element",
    "parallelepiped_defect",
    "ShardedLocalOperator",
    "WorkloadCount",
    "ax_flops",
    "geo_flops",
    "workload_count",
    "HardwareProfile",
    "KernelModel",
    "RooflineBounds",
    "load_profile",
    "resolve_profile",
    "roofline_bounds",
    "machine_balance",
    "mbp_crossing",
    "measured_performance",
    "operational_intensity",
    "preset_names",
]
