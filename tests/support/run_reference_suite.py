"""Run the reference's own operator tests with hosfem's AxLocal entry points
rebound to the B200 operator (paper_2504_07042_b200.compat.patch_hosfem).

    python tests/support/run_reference_suite.py [pytest node ids relative to hosfem_tests]

Test infrastructure: the reference package and its tests come from
baseline/_ref (tools/install_reference.sh); nothing here is product code.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "hosfem_tests")

DEFAULT = [
    "test_axlocal.py",
    "test_acceptance.py::test_criterion_2_operator_oracle",
    "test_acceptance.py::test_criterion_7_solver_invariance",
    "test_acceptance.py::test_criterion_8_nullspace_and_mass",
]


def main(argv):
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    import hosfem
    import hosfem.cli  # noqa: F401 - load every module that imports the entry points
    import hosfem.solver  # noqa: F401
    import hosfem.verify  # noqa: F401

    import paper_2504_07042_b200 as hx
    from paper_2504_07042_b200.compat import patch_hosfem

    patch_hosfem(hosfem)
    assert hosfem.axlocal.LocalOperator is hx.LocalOperator
    assert hosfem.solver.LocalOperator is hx.LocalOperator
    print("hosfem AxLocal entry points -> paper_2504_07042_b200 (GPU)", flush=True)
    import pytest

    nodes = [os.path.join(TESTS, n) for n in (argv or DEFAULT)]
    return pytest.main([*nodes, "-q", "-rA", "-p", "no:cacheprovider", "-c", os.devnull, "--rootdir", TESTS])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
