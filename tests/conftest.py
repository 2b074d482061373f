import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"
PROGRAMS = ROOT / "paper_1604_04997_b200" / "programs"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    return json.loads((GOLDEN / name).read_text())


def hexf(s):
    return float.fromhex(s)


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def suite_alpha():
    """Weights fitted by the reference on the 390 measurement cases."""
    import kc_oracle
    d = load_golden("fit_suite.json")
    a = [0.0] * len(kc_oracle.SCHEMA)
    for k, v in d["alpha"].items():
        a[kc_oracle.SCHEMA_INDEX[k]] = hexf(v[1])
    return a
