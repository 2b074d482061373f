"""The C++ host path (include/kcg.hpp -> C ABI -> kernels) without Python in
the loop: tests/cpp/kcg_host_driver evaluates bindings and fits a design,
results are compared here with the oracle / the reference fit."""
import math
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

import kc_oracle as ko
from conftest import GOLDEN, PROGRAMS, hexf, load_golden

ROOT = Path(__file__).resolve().parent.parent
DRIVER = ROOT / "paper_1604_04997_b200" / "_lib" / "kcg_host_driver"


def test_driver_is_built():
    assert DRIVER.exists(), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_cpp_host_eval_matches_oracle(tmp_path, suite_alpha):
    kid = "matmul_skinny_g16x16"
    text = (PROGRAMS / f"{kid}.kcp").read_text()
    oprog = ko.Program(text)
    rng = np.random.default_rng(1)
    us = rng.integers(1, 300000, size=3000)
    bs = [{"n": 16 * int(u), "m": 128 * int(u), "l": 16 * int(u)} for u in us]
    bs += [{"n": 17, "m": 128, "l": 16}, {"n": -16, "m": 128, "l": 16}]
    n = len(bs)
    cols = [[b[p] for b in bs] for p in oprog.params]
    (tmp_path / "b.bin").write_bytes(struct.pack("<qq", n, len(cols)) +
                                     b"".join(struct.pack(f"<{n}q", *c) for c in cols))
    r = subprocess.run([str(DRIVER), "eval", str(PROGRAMS / f"{kid}.kcp"), str(GOLDEN / "weights_suite.json"),
                        str(tmp_path / "b.bin"), str(tmp_path / "o.bin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    raw = (tmp_path / "o.bin").read_bytes()
    F = len(oprog.props)
    pred = struct.unpack_from(f"<{n}d", raw, 0)
    st = raw[8 * n:9 * n]
    lo = struct.unpack_from(f"<{F * n}q", raw, 9 * n)
    hi = struct.unpack_from(f"<{F * n}q", raw, 9 * n + 8 * F * n)
    for i, b in enumerate(bs):
        try:
            want = oprog.evaluate_properties(b)
        except ko.AssumptionViolated:
            assert st[i] == 1 and math.isnan(pred[i])
            continue
        assert st[i] == 0
        for j, (k, _) in enumerate(oprog.props):
            assert (hi[j * n + i] << 64) | (lo[j * n + i] & ((1 << 64) - 1)) == want[k]
        assert pred[i] == ko.predict(suite_alpha, want)


@pytest.mark.gpu
def test_cpp_host_fit_matches_reference(tmp_path):
    fit = [f for f in load_golden("fit_synthetic.json")["fits"] if f["name"] == "config3_f40_n4000"][0]
    X = np.array(fit["counts"], dtype=np.float64) / np.array([hexf(t) for t in fit["times"]])[:, None]
    n, F = X.shape
    (tmp_path / "x.bin").write_bytes(struct.pack("<qq", n, F) + X.astype("<f8").tobytes())
    r = subprocess.run([str(DRIVER), "fit", str(tmp_path / "x.bin"), str(tmp_path / "o.bin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    raw = (tmp_path / "o.bin").read_bytes()
    alpha = struct.unpack_from(f"<{F}d", raw, 0)
    rank, obj = struct.unpack_from("<qd", raw, 8 * F)
    ref = [hexf(a) for a in fit["alpha"]]
    assert rank == F
    for a, b in zip(alpha, ref):
        assert abs(a - b) <= 1e-6 * abs(b)
    assert obj <= 1e-18


@pytest.mark.gpu
def test_cpp_host_grid_and_columns(tmp_path):
    """kcg::predict_grid == kcg::grid_bindings -> kcg-columns file ->
    kcg::Columns::load -> kcg::predict, bitwise, from C++."""
    r = subprocess.run([str(DRIVER), "grid", str(PROGRAMS / "matmul_tiled_g16x16.kcp"),
                        str(GOLDEN / "weights_suite.json"), str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "grid ok" in r.stdout


@pytest.mark.gpu
def test_cpp_host_enumerate_matches_golden():
    """kcg::EnumProgram from C++ reproduces a reference enumerate_points tally."""
    c = next(c for c in load_golden("enum_points.json")["cases"]
             if c["kernel"] == "fd_stencil_g16x16" and c["status"] == "ok")
    n = int(c["binding"]["n"])
    r = subprocess.run([str(DRIVER), "enum", str(PROGRAMS / "enum" / "fd_stencil_g16x16.kce"), str(n)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.split("\n")
    assert lines[0] == f"points {c['points']}"
    got = dict(l.split(" ") for l in lines[1:] if l)
    assert got == c["counts"]
