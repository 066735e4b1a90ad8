"""Generate the golden AxLocal vectors by running the REFERENCE package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports hosfem read-only from /root/reference/pkg/src, runs its own public
API (SpectralBasis.build, box_mesh, LocalOperator.apply, dense_local_matrix)
on seeded inputs and writes tests/golden/golden_v1.npz.  The GPU box has no
/root/reference, so the parity tests read these fixtures instead.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def main():
    sys.path.insert(0, REF)
    from hosfem.axlocal import Equation, FactorSource, KernelSpec, LocalOperator, dense_local_matrix
    from hosfem.basis import SpectralBasis
    from hosfem.mesh import REFERENCE_CUBE, LocalField, box_mesh, make_element

    arrays: dict[str, np.ndarray] = {}
    cases: list[dict] = []

    for n in range(1, 16):
        b = SpectralBasis.build(n)
        arrays[f"basis{n}_points"] = b.points
        arrays[f"basis{n}_weights"] = b.weights
        arrays[f"basis{n}_dmat"] = b.diff_matrix
        arrays[f"basis{n}_tw"] = b.tensor_weights()

    for name, args in (("boxA", (3, 2, 2, 2, 0.2, 5)), ("boxB", (4, 4, 4, 7, 0.1, 0)), ("boxC", (5, 1, 1, 3, 0.0, 0))):
        ex, ey, ez, order, pert, seed = args
        m = box_mesh(ex, ey, ez, order, perturbation=pert, seed=seed)
        arrays[f"{name}_verts"] = np.stack([el.vertices for el in m.elements])
        arrays[f"{name}_kinds"] = np.array([el.kind.value == "parallelepiped" for el in m.elements])
        arrays[f"{name}_l2g"] = m.local_to_global
        arrays[f"{name}_args"] = np.array(args, dtype=float)

    rng = np.random.default_rng(20240817)

    def tri_elements(k):
        return [make_element(REFERENCE_CUBE + rng.uniform(-0.2, 0.2, (8, 3))) for _ in range(k)]

    def ppd_elements(k):
        out = []
        while len(out) < k:
            a = np.eye(3) + rng.uniform(-0.3, 0.3, (3, 3))
            if np.linalg.det(a) > 0.1:
                out.append(make_element(REFERENCE_CUBE @ a.T + rng.uniform(-1.0, 1.0, 3)))
        return out

    def add_case(order, equation, source, n_col, elements, coeff_mode):
        basis = SpectralBasis.build(order)
        E, n3 = len(elements), basis.n1**3
        x = rng.standard_normal((E, n3, n_col))
        lam0 = lam1 = None
        if equation == "helmholtz":
            if coeff_mode == "field":
                lam0 = rng.uniform(0.5, 2.0, (E, n3))
                lam1 = rng.uniform(0.5, 2.0, (E, n3))
            elif coeff_mode == "scalar":
                lam0, lam1 = 1.7, 0.3
        spec = KernelSpec(Equation(equation), n_col, FactorSource(source), order)
        y = LocalOperator(spec, elements, basis, lam0=lam0, lam1=lam1).apply(LocalField(x, order)).data
        idx = len(cases)
        key = f"case{idx}"
        arrays[f"{key}_verts"] = np.stack([el.vertices for el in elements])
        arrays[f"{key}_x"] = x
        arrays[f"{key}_y"] = y
        meta = dict(order=order, equation=equation, source=source, n_col=n_col, coeff=coeff_mode, E=E)
        if lam0 is not None and np.ndim(lam0) == 2:
            arrays[f"{key}_lam0"] = lam0
            arrays[f"{key}_lam1"] = lam1
        elif lam0 is not None:
            meta["lam0"], meta["lam1"] = lam0, lam1
        cases.append(meta)

    poisson = ("stored", "trilinear", "trilinear-partial")
    helm = ("stored", "trilinear", "trilinear-merged")
    for order in (1, 2, 3, 5, 7):
        els = tri_elements(3)
        for n_col in (1, 3):
            for src in poisson:
                add_case(order, "poisson", src, n_col, els, "none")
            for src, mode in zip(helm, ("field", "none", "field")):
                add_case(order, "helmholtz", src, n_col, els, mode)
        add_case(order, "helmholtz", "trilinear", 1, els, "scalar")
    for order in (3, 7):
        els = ppd_elements(2)
        add_case(order, "poisson", "parallelepiped", 1, els, "none")
        add_case(order, "helmholtz", "parallelepiped", 1, els, "field")
        add_case(order, "poisson", "stored", 1, els, "none")
    for order in (9, 11, 15):
        els = tri_elements(2)
        add_case(order, "poisson", "trilinear", 1, els, "none")
        add_case(order, "poisson", "stored", 1, els, "none")
    add_case(15, "helmholtz", "trilinear", 3, tri_elements(1), "field")
    boxb = box_mesh(3, 3, 3, 7, perturbation=0.1, seed=0).elements
    for src in poisson:
        add_case(7, "poisson", src, 1, boxb, "none")
    add_case(7, "helmholtz", "trilinear-merged", 1, boxb, "scalar")
    add_case(4, "poisson", "parallelepiped", 3, box_mesh(5, 1, 1, 4).elements, "none")

    # dense element matrices (axlocal.py:277-310)
    for order in (2, 3):
        el = tri_elements(1)[0]
        for eq in ("poisson", "helmholtz"):
            spec = KernelSpec(Equation(eq), 1, FactorSource.STORED, order)
            arrays[f"dense_{eq}_{order}_verts"] = el.vertices
            arrays[f"dense_{eq}_{order}"] = dense_local_matrix(spec, el, SpectralBasis.build(order))

    # Nekbone CG protocol (solver.py:240-308): iterations and max-norm error per variant
    from hosfem.solver import NekboneConfig, nekbone_benchmark

    nek = []
    for cfg in (
        dict(order=5, elements=(3, 3, 3), equation="poisson", n_col=1, perturbation=0.0),
        dict(order=3, elements=(4, 3, 2), equation="poisson", n_col=1, perturbation=0.15),
        dict(order=4, elements=(2, 2, 3), equation="helmholtz", n_col=1, perturbation=0.1),
        dict(order=3, elements=(2, 2, 2), equation="poisson", n_col=3, perturbation=0.1),
    ):
        res, _ = nekbone_benchmark(NekboneConfig(order=cfg["order"], elements=cfg["elements"],
                                                 equation=Equation(cfg["equation"]), n_col=cfg["n_col"],
                                                 perturbation=cfg["perturbation"], tol=1e-8, max_iter=300))
        nek.append(dict(cfg, results=[dict(variant=r.variant, iterations=r.iterations, error=r.error) for r in res]))
    arrays["nekbone_json"] = np.frombuffer(json.dumps(nek).encode(), dtype=np.uint8)

    arrays["cases_json"] = np.frombuffer(json.dumps(cases).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(cases)} operator cases, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
