"""Algorithmic work per element — the numerator of every roofline fraction.

Same integer model as the reference (pkg/src/hosfem/workload.py:52-120, the
paper's Table 2): effective operator flops F_ax, factor flops F_geo and bytes
M per element and apply.  ``roofline.achieved`` in bench.py is
E * (F_ax + F_geo) / t for compute-bound variants and E * M / t for
memory-bound ones, with M counted without the D-matrix term (D sits in the
``__constant__`` bank, ``include_dmat_traffic=False``).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["FP_SIZE", "WorkloadCount", "ax_flops", "geo_flops", "geo_memory_reals", "base_memory_reals",
           "stored_memory_reals", "workload_count", "matrix_unit_split"]

FP_SIZE = 8


@dataclass(frozen=True)
class WorkloadCount:
    f_ax: int
    f_geo: int
    m_bytes: int


def _src(spec_or_source):
    from .axlocal import FactorSource, _coerce_enum

    return _coerce_enum(FactorSource, spec_or_source)


def _helm(equation) -> bool:
    return getattr(equation, "value", equation) == "helmholtz"


def ax_flops(equation, n_col: int, n1: int) -> int:
    """12 n1^4 (six contractions) + 15 n1^3 (factor stage) per column, +5 n1^3 mass."""
    per = 12 * n1**4 + (20 if _helm(equation) else 15) * n1**3
    return n_col * per


def geo_flops(source, equation, n1: int) -> int:
    name = _src(source).value
    if name == "stored":
        return 0
    if name == "parallelepiped":
        return (8 if _helm(equation) else 7) * n1**3
    tail = 80 if name == "trilinear" else 60  # merged / partial skip the divide tail
    return 72 * n1 + 45 * n1**2 + tail * n1**3


def geo_memory_reals(source, equation, n1: int) -> int:
    name = _src(source).value
    helm = _helm(equation)
    if name == "stored":
        return (7 if helm else 6) * n1**3
    if name == "parallelepiped":
        return 7 if helm else 6
    if name == "trilinear-partial":
        return 24 + n1**3
    return 24


def base_memory_reals(equation, n_col: int, n1: int, include_dmat: bool = True) -> int:
    reals = 2 * n_col * n1**3 + (2 * n1**3 if _helm(equation) else 0)
    return reals + (n1**2 if include_dmat else 0)


def stored_memory_reals(equation, n_col: int, n1: int) -> int:
    """Full traffic of the stored-factor baseline in reals (reference workload.py:101-105)."""
    return base_memory_reals(equation, n_col, n1) + geo_memory_reals("stored", equation, n1)


def matrix_unit_split(spec) -> int:
    """Flops a matrix unit could take: the r and s contractions, forward and
    transposed, 8 n1^4 per column (reference workload.py:123-127).  On B200 the
    FP64 matrix path (DMMA) shares the DFMA pipe, so the b200 profile's
    peak_matrix equals peak_general."""
    return spec.n_col * 8 * (spec.order + 1) ** 4


def workload_count(spec, include_dmat_traffic: bool = True, fp_size: int = FP_SIZE) -> WorkloadCount:
    n1 = spec.order + 1
    reals = base_memory_reals(spec.equation, spec.n_col, n1, include_dmat_traffic) + geo_memory_reals(
        spec.factor_source, spec.equation, n1
    )
    return WorkloadCount(
        f_ax=ax_flops(spec.equation, spec.n_col, n1),
        f_geo=geo_flops(spec.factor_source, spec.equation, n1),
        m_bytes=reals * fp_size,
    )
