import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        data = {k: z[k] for k in z.files}
    data["cases"] = json.loads(bytes(data.pop("cases_json")).decode())
    return data


def golden_case(golden, idx):
    meta = dict(golden["cases"][idx])
    key = f"case{idx}"
    meta["verts"] = golden[f"{key}_verts"]
    meta["x"] = golden[f"{key}_x"]
    meta["y"] = golden[f"{key}_y"]
    if f"{key}_lam0" in golden:
        meta["lam0"] = golden[f"{key}_lam0"]
        meta["lam1"] = golden[f"{key}_lam1"]
    else:
        meta.setdefault("lam0", None)
        meta.setdefault("lam1", None)
    return meta


def n_golden_cases():
    with np.load(GOLDEN) as z:
        return len(json.loads(bytes(z["cases_json"]).decode()))


@pytest.fixture(scope="session")
def reference():
    """The live reference package, only where /root/reference exists (build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference tree not present (GPU box); golden fixtures cover parity")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import hosfem

    return hosfem
