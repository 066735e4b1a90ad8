"""The command-line front end (reference cli.py): `roofline` prints the reference's
bytes for every golden flag combination (tests/golden/roofline_cli.json, written
by the reference CLI itself); bench CSV round trip; error exit status."""

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


def test_bench_csv_round_trip():
    rec = cli.BenchRecord("poisson", 1, 7, "trilinear", 512, 5, 1.5e-5, 1.9e12, 3.4e12, 2.0e13, 95.0)
    text = cli.bench_records_to_csv([rec, rec])
    assert cli.parse_bench_csv(text) == [rec, rec]
    with pytest.raises(ValueError):
        cli.parse_bench_csv("bad header\n")


def test_errors_exit_2(capsys):
    assert cli.main(["roofline", "--profile", "no-such-device"]) == 2
    assert "error:" in capsys.readouterr().err
    assert cli.main(["bench", "--elements", "4x4"]) == 2


@pytest.mark.gpu
def test_bench_and_nekbone_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rc, out = _run(["bench", "--variant", "trilinear", "--elements", "8x8x8", "--perturbation", "0.1",
                    "--format", "json", "--repeats", "3"])
    assert rc == 0
    rec = json.loads(out)
    assert rec["E"] == 512 and rec["best_time_s"] > 0 and rec["roofline_R_eff"] > 0
    rc, out = _run(["nekbone", "--elements", "3x3x3", "--order", "5", "--format", "csv", "--variants", "trilinear"])
    assert rc == 0
    lines = out.strip().splitlines()
    assert lines[0] == "variant,iterations,error,wall_time_s,gflops_effective,axlocal_share"
    assert lines[1].startswith("trilinear,")
