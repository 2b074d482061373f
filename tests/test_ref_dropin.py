"""The reference-side drop-in compiled and run for real (verdict: "the
reference callers never reach the GPU in any test"): oracle/_ref/ref_dropin
is tests/cpp/ref_dropin.cpp + tests/cpp/kernelcost_gpu.hpp (INTEGRATION.md
§2: predict_batch, evaluate_properties_batch, predict_batch_host,
fit_weights_gram) built against the reference's own headers and library
(the sources compiled in place) and linked with libkcg.so. In one process
it parses every suite kernel with the reference parser, extracts the
symbolic PV, hands program_text to kcg and compares the GPU with the
reference's scalar evaluate_properties / predict / fit_weights on the 406
manifest cases, a host-vector sweep of the six matmul variants and the
simulated 390-case campaign fit."""
import json
import subprocess

import pytest

from conftest import ROOT

EXE = ROOT / "oracle" / "_ref" / "ref_dropin"


@pytest.mark.gpu
def test_reference_callers_through_the_gpu_drop_in():
    if not EXE.exists():
        pytest.skip("oracle/_ref/ref_dropin not built (build() builds it where /root/reference exists)")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=900)
    assert r.stdout.strip(), r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["manifest_cases"] == 406
    assert d["symbolic_kernels"] >= 59 and d["gpu_checked_points"] > 350
    assert d["count_mismatches"] == 0 and d["prediction_mismatches"] == 0 and d["status_mismatches"] == 0
    assert d["host_batch_points"] == 30000 and d["host_batch_mismatches"] == 0
    assert d["fit_cases"] == 390 and d["fit_worst_in_tolerance_units"] <= 1.0 and d["fit_covered_mismatches"] == 0
    assert d["ok"] is True and r.returncode == 0
