"""Mesh files written by the REFERENCE's save_mesh (reference mesh.py:340-353).

    python tests/golden/make_mesh_golden.py

Runs in the build container (where /root/reference exists) and writes
tests/golden/mesh_*.txt; tests/test_mesh_io.py checks that this package reads
them and writes the same bytes.
"""

import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from hosfem.mesh import box_mesh, save_mesh

    for name, args, kw in (
        ("mesh_box_2x1x1_n3.txt", (2, 1, 1, 3), dict(perturbation=0.17, seed=4)),
        ("mesh_box_3x2x2_n2.txt", (3, 2, 2, 2), dict(perturbation=0.2, seed=5)),
        ("mesh_box_2x2x1_n1_affine.txt", (2, 2, 1, 1), dict(extents=((0.0, 2.0), (-1.0, 1.0), (0.0, 0.5)))),
    ):
        save_mesh(box_mesh(*args, **kw), os.path.join(HERE, name))
        print("wrote", name)


if __name__ == "__main__":
    main()
