"""CPU stand-in for the BP5 C-ABI kernels (TEST INFRASTRUCTURE ONLY).

Lets the solver's host logic — slab layout, interface exchange, rank-ordered
reductions, the CG driver — run under the gloo backend on CPU, with the
oracle as the element-local operator.  Vectors are CPU torch tensors.
"""

import numpy as np
import torch

from oracle import hosfem_oracle as O


class _OracleLocal:
    def __init__(self, spec, verts, basis, lam0, lam1):
        self.st = O.setup(spec.factor_source.value, spec.equation.value, spec.order, np.asarray(verts),
                          lam0=lam0, lam1=lam1)

    def apply_(self, x, y):
        y.copy_(torch.as_tensor(O.apply_setup(self.st, x.numpy())))
        return y


class NumpyBackend:
    def local_operator(self, spec, verts, basis, lam0, lam1):
        if isinstance(lam0, torch.Tensor):
            lam0 = lam0.numpy()
        if isinstance(lam1, torch.Tensor):
            lam1 = lam1.numpy()
        return _OracleLocal(spec, verts, basis, lam0, lam1)

    @staticmethod
    def _slab_l2g(layout):
        ex, ey, _ = layout.counts
        return O.box_l2g(ex, ey, layout.nz_el, layout.order)

    def gather(self, layout, u, xl, n_col=1, col=0):
        xl[:, :, col] = torch.as_tensor(u.numpy()[self._slab_l2g(layout)])

    def scatter(self, layout, yl, v, n_col=1, col=0):
        y = yl[:, :, col].numpy()
        v.copy_(torch.as_tensor(O.scatter_add(y, self._slab_l2g(layout), layout.n_local)))

    def mask(self, layout, v):
        ex, ey, ez = layout.counts
        m = O.interior_mask(ex, ey, ez, layout.order)[layout.global_slice()]
        v[torch.as_tensor(~m)] = 0.0

    def dot(self, a, b, n, out):
        out[0] = float(np.sum(a.numpy()[:n] * b.numpy()[:n]))

    def update_xr(self, scal, x, p, r, ap):
        alpha = float(scal[0] / scal[1])
        x += alpha * p
        r -= alpha * ap

    def update_p(self, scal, p, r):
        beta = float(scal[2] / scal[0])
        p.copy_(r + beta * p)
