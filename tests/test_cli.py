"""The command-line front end: `roofline` prints the reference CLI's bytes for
every golden flag combination (tests/golden/roofline_cli.json, written by the
reference CLI itself, tests/golden/make_cli_golden.py); error exit status."""

import contextlib
import io
import json
import os

import pytest

from paper_2504_07042_b200 import cli

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "roofline_cli.json")


def _run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def _cases():
    with open(GOLDEN) as fh:
        return sorted(json.load(fh).items())


@pytest.mark.parametrize("argv,want", _cases())
def test_roofline_matches_reference_cli(argv, want):
    rc, out = _run(argv.split())
    if "--list-profiles" in argv:
        assert rc == 0 and set(want["stdout"].split()) <= set(out.split()) and "b200" in out.split()
        return
    assert rc == want["rc"]
    assert out == want["stdout"]


def test_roofline_b200_profile():
    rc, out = _run(["roofline", "--profile", "b200", "--format", "json"])
    assert rc == 0
    rows = {r["variant"]: r for r in json.loads(out)}
    assert rows["stored"]["bound"] == "memory" and rows["trilinear"]["bound"] == "compute"
    # D-matrix traffic included by default, like the reference: 8896 B for trilinear N=7
    assert rows["trilinear"]["m_bytes"] == 8896


def test_errors_exit_2(capsys):
    assert cli.main(["roofline", "--profile", "no-such-device"]) == 2
    assert "error:" in capsys.readouterr().err


def test_model_api():
    """The reference's roofline functions behave as documented (roofline.py)."""
    from paper_2504_07042_b200 import roofline as R

    hw = R.resolve_profile("a100")
    assert R.machine_balance(hw) == pytest.approx(9.7e12 / 1.360e12)
    assert hw.peak("matrix") == 19.5e12 and hw.bandwidth("theoretical") == 1.555e12
    for bad in (lambda: hw.peak("tensor"), lambda: hw.bandwidth("peak"), lambda: R.resolve_profile("k100").peak("matrix"),
                lambda: R.HardwareProfile("x", 1.0, 2.0, 1.0), lambda: R.KernelModel(1, 1, 1, 5),
                lambda: R.measured_performance(1, 1, 0.0)):
        with pytest.raises(ValueError):
            bad()
    m = R.KernelModel(100, 50, 10, matrix_unit_flops=60)
    b_sum, b_max = R.roofline_bounds(m, hw), R.roofline_bounds(m, hw, overlap=True)
    assert b_sum.t_cmp == pytest.approx(90 / 9.7e12 + 60 / 19.5e12)
    assert b_max.t_cmp == pytest.approx(max(90 / 9.7e12, 60 / 19.5e12))
    assert R.measured_performance(10.0, 5.0, 2.0) == (5.0, 7.5)
