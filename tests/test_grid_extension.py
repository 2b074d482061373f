"""SURVEY 8(f) row 1 as a rule: the front-end extension
(oracle/kcref_extract.hpp: stride-0/1 accesses classified without the
footprint, classify.cpp:15-17; contained-box footprint union) makes kernels
symbolic that the reference's extract_properties rejects for their
footprint (props.cpp:136-159, footprint.cpp:421-430). On the suite it equals
extract_properties on all 59 symbolic kernels and regenerates fd_stencil /
nbody (programs/derived.json); here two new halo kernels
(tests/gen/halo_kernels.txt: a 1D halo stencil with guarded edge loads and
an interleaved [2, n] column-major array read through a component loop)
are checked: the extension's programs against the reference's own
bound-mode extraction at every n the 2e7 cap admits (tests/golden/
halo_kernels.json, oracle/_ref/kcref_grid), and on the GPU against the
brute-force enumeration far past that cap."""
import json

import pytest

from conftest import PROGRAMS, load_golden

import kc_oracle as ko
import paper_1604_04997_b200 as kc


def _kernels():
    return load_golden("halo_kernels.json")["kernels"]


def test_halo_kernels_are_rejected_by_the_reference_and_extended():
    ks = _kernels()
    assert [k["id"] for k in ks] == ["halo1d_g256", "cplx_sum_g128"]
    for k in ks:
        assert k["reference_symbolic"] is False and len(k["bound_mode"]) >= 30


@pytest.mark.parametrize("k", _kernels(), ids=lambda k: k["id"])
def test_extension_programs_equal_reference_bound_mode(k):
    """oracle restatement of the extension's program == the reference's
    bound-mode counts (no GPU)"""
    prog = ko.Program(k["program"])
    for case in k["bound_mode"]:
        want = {ko.SCHEMA_INDEX[key]: int(v) for key, v in case["counts"].items()}
        assert prog.evaluate_properties({"n": case["n"]}) == want, (k["id"], case["n"])


def test_fd_stencil_nbody_programs_come_from_the_extension():
    d = json.loads((PROGRAMS / "derived.json").read_text())["derived"]
    assert {e["id"] for e in d if "file" in e} == {"fd_stencil_g16x16", "nbody_g256"}
    for e in d:
        assert e["method"].startswith("symbolic: oracle/kcref_extract.hpp") and e["verified_points"] >= 10
        text = (PROGRAMS / e["file"]).read_text()
        assert "kcref_extract.hpp" in text and "interpolation" not in text


@pytest.mark.gpu
@pytest.mark.parametrize("k", _kernels(), ids=lambda k: k["id"])
def test_extension_programs_on_gpu_bound_mode_and_beyond_the_cap(k):
    import torch
    prog = kc.Program(k["program"])
    ns = [c["n"] for c in k["bound_mode"]]
    bb = kc.evaluate_properties(prog, {"n": torch.tensor(ns, dtype=torch.int64, device="cuda")}, wide=True)
    torch.cuda.synchronize()
    keys = kc.schema_keys()
    for i, c in enumerate(k["bound_mode"]):
        got = {keys[key]: bb.counts_int(j, i) for j, key in enumerate(prog.props) if bb.counts_int(j, i)}
        assert got == {key: int(v) for key, v in c["counts"].items()}, (k["id"], c["n"])
    ep = kc.EnumProgram(k["enum_text"])
    for n in (1 << 16, 1 << 20, 1 << 24):
        counts, points = ep.enumerate_points({"n": n})
        one = kc.evaluate_properties(prog, {"n": torch.tensor([n], dtype=torch.int64, device="cuda")}, wide=True)
        torch.cuda.synchronize()
        sym = {keys[key]: one.counts_int(j, 0) for j, key in enumerate(prog.props) if one.counts_int(j, 0)}
        assert points > 0 and counts == sym, (k["id"], n)
