"""`kernelcost simulate` on the GPU: run_campaign (campaign.cpp:11-45) with
simulate_time / simulate_runs (simdevice.cpp:96-128) over the reference's
390 measurement cases, written with the reference's CSV writers
(csvio.cpp:104-155). sigma 0: the file is byte-identical to the reference's
meas_sigma0.csv; 8 noisy runs (sigma 0.02, seed 7): every field identical
and every time within 2 ulp of the reference's raw_runs_sigma002.csv (CUDA's
exp/log/cos vs glibc). The CLI fit on the GPU-written file equals the fit
on the reference's file."""
import csv
import io

import pytest

from conftest import GOLDEN, hexf, load_golden

pytestmark = pytest.mark.gpu

import kc_oracle as ko  # noqa: E402
import paper_1604_04997_b200 as kc  # noqa: E402


def _cases():
    out = []
    for c in load_golden("suite_cases.json")["cases"]:
        if c["role"] != "measurement":
            continue
        out.append((c["kernel"], {k: int(v) for k, v in c["binding"].items()}, c["kernel"].rsplit("_g", 1)[1]))
    return out


def test_campaign_sigma0_csv_is_byte_identical(tmp_path):
    recs, diags = kc.run_campaign(_cases(), ko.simdev_reference_alpha())
    assert not diags and len(recs) == 390
    kc.write_measurements_csv(tmp_path / "m.csv", recs)
    assert (tmp_path / "m.csv").read_bytes() == (GOLDEN / "meas_sigma0.csv").read_bytes()
    w1, r1 = kc.fit_from_csv(tmp_path / "m.csv", device="gpu")
    w2, r2 = kc.fit_from_csv(GOLDEN / "meas_sigma0.csv", device="gpu")
    assert w1.alpha == w2.alpha and r1["objective"] == r2["objective"]


def test_campaign_noisy_raw_runs_match_the_reference(tmp_path):
    recs, diags = kc.run_campaign(_cases(), ko.simdev_reference_alpha(), sigma=0.02, seed=7, runs=8)
    assert not diags and len(recs) == 8 * 390
    kc.write_raw_runs_csv(tmp_path / "r.csv", recs)
    got = list(csv.reader(io.StringIO((tmp_path / "r.csv").read_text())))
    want = list(csv.reader(io.StringIO((GOLDEN / "raw_runs_sigma002.csv").read_text())))
    assert got[0] == want[0] and len(got) == len(want)
    worst = 0.0
    for g, w in zip(got[1:], want[1:]):
        assert g[:4] == w[:4]
        worst = max(worst, abs(float(g[4]) - float(w[4])) / float(w[4]))
    assert worst <= 5e-16, worst


def test_campaign_reports_inadmissible_cases_as_diagnostics(tmp_path):
    cases = _cases()[:3] + [("matmul_tiled_g16x16", {"n": 17, "m": 16, "l": 16}, "16x16")]
    recs, diags = kc.run_campaign(cases, ko.simdev_reference_alpha())
    assert len(recs) == 3 and len(diags) == 1
    assert diags[0].startswith("matmul_tiled_g16x16 [l=16;m=16;n=17]: E_ASSUMPTION_VIOLATED")
    one = [r for r in recs if r.kernel == recs[0].kernel]
    kc.write_campaign_columns(tmp_path / "c.kcgcol", one)
    cols = kc.read_columns(tmp_path / "c.kcgcol")
    assert list(cols.numpy("time_s")) == [r.time_s for r in one]
