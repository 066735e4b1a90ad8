"""Gauss-Lobatto-Legendre constants for one polynomial order.

Host-side setup data, not the hot path: the points, weights and the nodal
differentiation matrix are computed once here in fp64 and uploaded into the
kernel library's ``__constant__`` bank (``hx_set_basis``), where the unrolled
contractions read D as a compile-time-offset operand.

Mirrors ``hosfem.basis.SpectralBasis`` (reference pkg/src/hosfem/basis.py:110-136):
same attributes (``order``, ``points``, ``weights``, ``diff_matrix``, ``n1``,
``tensor_weights()``), same conventions (ascending points on [-1, 1], entry
[i][j] of D is the derivative of cardinal j at point i, corner entries
-/+ N(N+1)/4, flat tensor weights with i fastest).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = ["SpectralBasis", "MAX_ORDER"]

#: Largest order the CUDA library is instantiated for (n1 = 16).
MAX_ORDER = 15


def _legendre(n: int, x: np.ndarray):
    """L_n(x) and L_n'(x) by the Bonnet recurrence (valid at +-1)."""
    p_prev = np.ones_like(x)
    dp_prev = np.zeros_like(x)
    if n == 0:
        return p_prev, dp_prev
    p, dp = x.copy(), np.ones_like(x)
    for k in range(1, n):
        # coefficients rounded once, as the reference does, so the constants
        # uploaded to the GPU are bit-identical to hosfem's
        a, b = (2.0 * k + 1.0) / (k + 1.0), k / (k + 1.0)
        p_next = a * x * p - b * p_prev
        dp_next = a * (p + x * dp) - b * dp_prev
        p_prev, dp_prev, p, dp = p, dp, p_next, dp_next
    return p, dp


def _gll_points(n: int) -> np.ndarray:
    # interior nodes are the roots of L_n'; Newton on L_n' with the Legendre
    # ODE for L_n'', started from the Chebyshev-Lobatto nodes
    x = -np.cos(np.pi * np.arange(n + 1) / n)
    for idx in range(1, n):
        # per-node Newton loop with its own stopping test (a node that has
        # converged must not take further steps)
        t = x[idx]
        for _ in range(100):
            p, dp = _legendre(n, np.array(t))
            d2p = (2.0 * t * dp - n * (n + 1) * p) / (1.0 - t * t)
            step = float(dp / d2p)
            t -= step
            if abs(step) < 1e-15:
                break
        else:
            raise RuntimeError(f"GLL root refinement did not converge for order {n}")
        x[idx] = t
    x[0], x[-1] = -1.0, 1.0
    return 0.5 * (x - x[::-1])


def _gll_weights(n: int, pts: np.ndarray) -> np.ndarray:
    ln, _ = _legendre(n, pts)
    w = 2.0 / (n * (n + 1) * ln * ln)
    return 0.5 * (w + w[::-1])


def _diff_matrix(n: int, pts: np.ndarray) -> np.ndarray:
    ln, _ = _legendre(n, pts)
    diff = pts[:, None] - pts[None, :]
    np.fill_diagonal(diff, 1.0)
    d = ln[:, None] / (ln[None, :] * diff)
    np.fill_diagonal(d, 0.0)
    d[0, 0] = -0.25 * n * (n + 1)
    d[n, n] = 0.25 * n * (n + 1)
    return d


@dataclass(frozen=True)
class SpectralBasis:
    """Immutable GLL data for one order (drop-in for hosfem.basis.SpectralBasis)."""

    order: int
    points: np.ndarray
    weights: np.ndarray
    diff_matrix: np.ndarray

    @classmethod
    def build(cls, order: int) -> "SpectralBasis":
        return _build_cached(int(order))

    @property
    def n1(self) -> int:
        return self.order + 1

    def tensor_weights(self) -> np.ndarray:
        """Flat (n1**3,) w_i w_j w_k, node (i, j, k) at i + j n1 + k n1^2."""
        w = self.weights
        # (w_k w_j) w_i: the product order of the reference's einsum and of the
        # kernels' cW(k) * cW(j) * cW(i), so all three agree bit for bit
        return ((w[:, None, None] * w[None, :, None]) * w[None, None, :]).ravel()


@lru_cache(maxsize=None)
def _build_cached(order: int) -> SpectralBasis:
    if order < 1:
        raise ValueError("order must be at least 1")
    pts = _gll_points(order)
    wts = _gll_weights(order, pts)
    dmat = _diff_matrix(order, pts)
    for arr in (pts, wts, dmat):
        arr.flags.writeable = False
    return SpectralBasis(order=order, points=pts, weights=wts, diff_matrix=dmat)
