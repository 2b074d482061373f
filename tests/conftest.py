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


# fitted-weight tolerance (north star: 1e-9 relative in fp64). Weights are
# compared in the equilibrated coordinates the solve works in
# (x_j = alpha_j * max|col_j|, model.cpp:71-76): relative 1e-9, plus an
# absolute 1e-13 for numerically-zero weights (a weight whose true value is
# 0 comes out of the double data as ~1e-16 in those units; relative error
# is meaningless there)
FIT_REL = 1e-9
FIT_ABS_SCALED = 1e-13


def fit_errors(got, want, colmax):
    """per-weight |got - want| / (FIT_REL |want| + FIT_ABS_SCALED / colmax): <= 1 passes"""
    out = []
    for g, w, c in zip(got, want, colmax):
        out.append(abs(g - w) / (FIT_REL * abs(w) + FIT_ABS_SCALED / c) if c > 0 else (0.0 if g == 0 else 1e300))
    return out


def exact_fit(name):
    """the exact min-norm LS solution of a golden fit design (tests/gen/gen_fit_exact.py)"""
    for f in load_golden("fit_exact.json")["fits"]:
        if f["name"] == name:
            return f
    raise KeyError(name)
