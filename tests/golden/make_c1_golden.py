"""C1 fixtures (box_mesh(512, 1, 1, N), BASELINE configs[0]) from the REFERENCE.

    python tests/golden/make_c1_golden.py

Runs hosfem's own LocalOperator.apply (stored and parallelepiped) on the C1 mesh
with x = default_rng(0).standard_normal((512, n1^3, 1)) (cli.py:194-197) and keeps
y for every 8th element (elements are independent).  C1's elements are 1/512 x 1 x 1:
the stored route's exact-zero Jacobian entries are rounding noise that the aspect
ratio amplifies to ~1e-12 of y, so y depends on the host's numpy / BLAS kernels at
that level -- the fixture pins the values of THIS reference run, not whatever the
GPU box's numpy would compute.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_c1.npz")


def main():
    sys.path.insert(0, REF)
    from hosfem.axlocal import Equation, FactorSource, KernelSpec, LocalOperator
    from hosfem.basis import SpectralBasis
    from hosfem.mesh import LocalField, box_mesh

    arrays = {}
    for order in (3, 7):
        n1 = order + 1
        mesh = box_mesh(512, 1, 1, order)
        x = np.random.default_rng(0).standard_normal((512, n1**3, 1))
        for src in ("stored", "parallelepiped"):
            spec = KernelSpec(Equation("poisson"), 1, FactorSource(src), order)
            y = LocalOperator(spec, mesh.elements, SpectralBasis.build(order)).apply(LocalField(x, order)).data
            arrays[f"n{order}_{src}"] = y[::8]
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
