"""Drop-in proof: the reference's own operator tests on the B200 operator.

hosfem's LocalOperator / ax_local_apply / dense_local_matrix are rebound to
this package's (paper_2504_07042_b200.compat.patch_hosfem) and the reference's
pkg/tests/test_axlocal.py (dense Kronecker oracle, null space, mass limit,
coefficient fields, n_col bitwise, threads bitwise, shape errors) plus
acceptance criteria 2, 7 and 8 (test_acceptance.py:91-130, 269-300, 302-337)
run unmodified -- criterion 7 through the reference's own CG solver, whose
GlobalOperator then applies the GPU AxLocal.  Needs baseline/_ref from
tools/install_reference.sh (it travels with gpurun); skipped without it.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "hosfem_tests", "test_axlocal.py")
RUNNER = os.path.join(ROOT, "tests", "support", "run_reference_suite.py")


def test_reference_operator_suite_runs_on_the_gpu_operator():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SUITE):
        pytest.skip("baseline/_ref has no reference test suite (tools/install_reference.sh)")
    out = subprocess.run([sys.executable, RUNNER], capture_output=True, text=True, timeout=1200, cwd=ROOT)
    tail = (out.stdout + out.stderr)[-4000:]
    assert "paper_2504_07042_b200 (GPU)" in out.stdout, tail
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and " failed" not in out.stdout, tail
