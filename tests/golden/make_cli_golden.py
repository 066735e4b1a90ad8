"""Outputs of the REFERENCE's `hosfem roofline` subcommand (reference cli.py:260-312).

    python tests/golden/make_cli_golden.py

Runs the reference CLI in this container for a grid of flags and stores
{args: stdout} in tests/golden/roofline_cli.json; tests/test_cli.py checks this
package's `roofline` prints the same bytes.
"""

import contextlib
import io
import json
import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "roofline_cli.json")

CASES = [
    [],
    ["--profile", "k100"],
    ["--format", "csv", "--order", "3"],
    ["--format", "json", "--order", "11", "--equation", "helmholtz"],
    ["--tensor-core", "--order", "7"],
    ["--tensor-core", "--overlap", "--format", "csv", "--ncol", "3"],
    ["--crossing"],
    ["--crossing", "--profile", "k100", "--equation", "helmholtz", "--ncol", "3"],
    ["--order", "1", "--format", "csv"],
    ["--order", "15", "--equation", "helmholtz", "--format", "json", "--overlap", "--tensor-core"],
    ["--list-profiles"],
]


def main():
    sys.path.insert(0, REF)
    from hosfem.cli import main as ref_main

    out = {}
    for extra in CASES:
        argv = ["roofline", "--profile", "a100"] + extra if "--profile" not in extra else ["roofline"] + extra
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = ref_main(argv)
        out[" ".join(argv)] = {"rc": rc, "stdout": buf.getvalue()}
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {OUT}: {len(out)} cases")


if __name__ == "__main__":
    main()
