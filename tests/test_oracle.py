"""Pin the CPU restatement (oracle/kc_oracle.py) against the golden vectors
the reference itself produced (oracle/_ref/kcref_export, reference sources
compiled in place against oracle/shim). Mirrors test_countexpr.cpp,
test_props.cpp, test_model.cpp, test_simdevice.cpp and acceptance.cpp."""
import math

import numpy as np
import pytest

import kc_oracle as ko
from conftest import PROGRAMS, hexf, load_golden


def _binding(d):
    return {k: int(v) for k, v in d.items()}


def _counts(d):
    return {ko.SCHEMA_INDEX[k]: int(v) for k, v in d.items()}


@pytest.fixture(scope="module")
def programs():
    return {p.stem: ko.Program(p.read_text()) for p in PROGRAMS.glob("*.kcp")}


def test_schema_has_149_keys_in_reference_order():
    assert len(ko.SCHEMA) == 149
    assert ko.SCHEMA[0] == "mem.global.load.s32.uniform"
    assert ko.SCHEMA[-3:] == ["sync.barrier", "launch.groups", "launch.const"]
    w = load_golden("weights_suite.json")
    assert list(w["weights"].keys()) == sorted(ko.SCHEMA)  # nlohmann sorts keys


def test_exact_evaluation_at_large_magnitudes():
    # test_countexpr.cpp:27-32
    e = ko.CountExpr("(+ (* 7 n) (^ n 3))")
    assert e.evaluate({"n": 10**10}) == 1000000000000000000070000000000


def test_floordiv_min_max_atoms():
    # test_countexpr.cpp:43-61
    fd = ko.CountExpr("(floordiv n 16)")
    assert [fd.evaluate({"n": v}) for v in (32, 33, 47, 48)] == [2, 2, 2, 3]
    assert ko.CountExpr("(min m n)").evaluate({"n": 5, "m": 9}) == 5
    assert ko.CountExpr("(max m n)").evaluate({"n": 5, "m": 9}) == 9
    assert ko.CountExpr("(floordiv (+ -3 n) 4)").evaluate({"n": 0}) == -1


def test_suite_cases_match_reference_bound_extraction(programs):
    """symbolic -> evaluate_properties == bound extraction (acceptance.cpp
    criterion 2) and noiseless_time bits, for all 406 manifest cases whose
    kernel extracts symbolically."""
    sim = ko.simdev_reference_alpha()
    cases = load_golden("suite_cases.json")["cases"]
    assert len(cases) == 406
    checked = 0
    for c in cases:
        want = _counts(c["counts"])
        # the stored timing is the reference's noiseless_time
        assert ko.noiseless_time(sim, want) == hexf(c["time_s"][1])
        prog = programs[c["kernel"]]  # fd_stencil / nbody: derived programs (§8f row 1)
        got = prog.evaluate_properties(_binding(c["binding"]))
        assert {k: v for k, v in got.items() if v} == want, c
        checked += 1
    assert checked == 406


def test_oracle_draws_match(programs):
    draws = load_golden("oracle_draws.json")["draws"]
    assert len(draws) == 61 * 20
    for d in draws:
        if "symbolic_equal" in d:
            assert d["symbolic_equal"], d
        # every kernel, incl. the derived fd_stencil / nbody programs, must
        # reproduce the reference's bound-mode extraction on its oracle lattice
        got = programs[d["kernel"]].evaluate_properties(_binding(d["binding"]))
        assert {k: v for k, v in got.items() if v} == _counts(d["counts"])


def _check_samples(samples, progs, alpha):
    n_ok = n_bad = 0
    for s in samples:
        prog = progs[s["kernel"]]
        b = _binding(s["binding"])
        if s["status"] == "ok":
            got = prog.evaluate_properties(b)
            assert {k: v for k, v in got.items() if v} == _counts(s["counts"])
            assert ko.predict(alpha, got) == hexf(s["predicted_s"][1])
            n_ok += 1
        else:
            with pytest.raises(ko.AssumptionViolated):
                prog.evaluate_properties(b)
            assert s["status"] == "E_ASSUMPTION_VIOLATED"
            n_bad += 1
    return n_ok, n_bad


def test_grid_samples_bitwise(programs, suite_alpha):
    ok, bad = _check_samples(load_golden("grid_samples.json")["samples"], programs, suite_alpha)
    assert ok > 1000 and bad > 50
    wide = [s for s in load_golden("grid_samples.json")["samples"]
            if s["status"] == "ok" and any(abs(int(v)) >= 2**64 for v in s["counts"].values())]
    assert wide, "golden set must exercise counts beyond 64 bits"


def test_extra_programs_with_atoms(suite_alpha):
    d = load_golden("extra_programs.json")
    progs = {p["id"]: ko.Program(p["program"]) for p in d["programs"] if "program" in p}
    assert {"x_minmax", "x_floordiv", "x_floordiv2", "x_triangle", "x_simplex"} <= set(progs)
    ok, bad = _check_samples(d["samples"], progs, suite_alpha)
    assert ok > 200 and bad > 10


def test_fit_suite_predictions_bitwise(suite_alpha):
    d = load_golden("fit_suite.json")
    sim = ko.simdev_reference_alpha()
    cases = {(c["kernel"], tuple(sorted(c["binding"].items()))): c
             for c in load_golden("suite_cases.json")["cases"]}
    assert len(d["test_predictions"]) == 16
    for p in d["test_predictions"]:
        c = cases[(p["kernel"], tuple(sorted(p["binding"].items())))]
        counts = _counts(c["counts"])
        assert ko.predict(suite_alpha, counts) == hexf(p["predicted_s"][1])
        assert ko.predict(sim, counts) == hexf(p["predicted_simdev_s"][1])


def test_reference_fit_recovers_table2_weights(suite_alpha):
    # acceptance.cpp:190-230 (noiseless recovery, rel 1e-6)
    sim = ko.simdev_reference_alpha()
    d = load_golden("fit_suite.json")
    assert hexf(d["objective"][1]) <= 1e-10
    for k in d["covered"]:
        i = ko.SCHEMA_INDEX[k]
        if sim[i] != 0.0:
            assert abs(suite_alpha[i] - sim[i]) <= 1e-6 * abs(sim[i]), k
        else:
            assert abs(suite_alpha[i]) <= 1e-15, k


def test_numpy_fit_matches_reference_cod():
    for fit in load_golden("fit_synthetic.json")["fits"]:
        keys = fit["keys"]
        cases = []
        for row, t in zip(fit["counts"], fit["times"]):
            cases.append(({ko.SCHEMA_INDEX[k]: c for k, c in zip(keys, row)}, hexf(t)))
        X, cov = ko.build_design_matrix(cases)
        alpha, obj, _ = ko.fit_weights(X, cov)
        ref = [hexf(a) for a in fit["alpha"]]
        for k, r in zip(keys, ref):
            got = alpha[ko.SCHEMA_INDEX[k]]
            assert abs(got - r) <= 1e-6 * abs(r), (fit["name"], k, got, r)
        assert obj <= max(1e-18, 10 * hexf(fit["objective"][1]))


def test_fit_never_beats_zero_model():
    # test_model.cpp:111-120
    X, cov = ko.build_design_matrix([({0: 100}, 1.0), ({0: 100}, 2.0)])
    alpha, obj, resid = ko.fit_weights(X, cov)
    assert 0.0 < obj < 2.0 and len(resid) == 2


def test_geomean_fixtures():
    # test_model.cpp:175-183
    assert ko.geometric_mean_error([(1.1, 1.0), (0.9, 1.0)]) == pytest.approx(0.10, rel=1e-12)
    assert ko.geometric_mean_error([(1.0, 1.0), (2.0, 1.0)]) == pytest.approx(math.sqrt(1e-12), rel=1e-9)


def test_keyed_gaussian_properties():
    # test_simdevice.cpp:47-69
    a = ko.keyed_gaussian(1, "k|n=64", 0)
    assert a == ko.keyed_gaussian(1, "k|n=64", 0)
    assert a != ko.keyed_gaussian(2, "k|n=64", 0)
    assert a != ko.keyed_gaussian(1, "k|n=65", 0)
    assert a != ko.keyed_gaussian(1, "k|n=64", 1)
    g = np.array([ko.keyed_gaussian(42, "moment-check", i) for i in range(4000)])
    assert abs(g.mean()) < 0.08 and abs(g.var() - 1.0) < 0.08


def test_admits_semantics():
    p = ko.Program((PROGRAMS / "matmul_tiled_g16x16.kcp").read_text())
    assert p.admits({"n": 16, "m": 32, "l": 48})
    assert not p.admits({"n": 17, "m": 32, "l": 48})
    assert not p.admits({"n": 0, "m": 32, "l": 48})
    assert not p.admits({"n": -16, "m": 32, "l": 48})


def test_derived_programs_match_survey_appendix_a():
    """fd_stencil / nbody closed forms recovered from
    the reference's bound-mode counts."""
    import json
    d = json.loads((PROGRAMS / "derived.json").read_text())["derived"]
    assert {e["id"] for e in d if "file" in e} == {"fd_stencil_g16x16", "nbody_g256"}
    fd = ko.Program((PROGRAMS / "fd_stencil_g16x16.kcp").read_text())
    c = fd.evaluate_properties({"n": 4096})
    assert c[ko.SCHEMA_INDEX["mem.global.load.s32.1/1"]] == 9 * 4096 ** 2 // 8
    assert c[ko.SCHEMA_INDEX["mem.local.load"]] == 6 * 4096 ** 2
    nb = ko.Program((PROGRAMS / "nbody_g256.kcp").read_text())
    c = nb.evaluate_properties({"n": 1 << 20})
    assert c[ko.SCHEMA_INDEX["mem.global.load.s32.3/3"]] == 3 * 4 ** 20 + 3 * 4 ** 20 // 256
    assert c[ko.SCHEMA_INDEX["launch.groups"]] == (1 << 20) // 256


def test_keyed_gaussian_and_simulate_match_reference_bitwise():
    """The Python restatement of simdevice.cpp:13-46 / 96-127 reproduces the
    reference's noisy stored timings bit for bit (same libm)."""
    import math
    d = load_golden("simulate.json")
    sim = ko.simdev_reference_alpha()
    for c in d["cases"][:120]:
        g = ko.keyed_gaussian(d["seed"], c["key"], 0)
        assert g == hexf(c["gaussian"])
        t0 = hexf(c["noiseless"])
        for run, r in enumerate(c["runs"]):
            assert t0 * math.exp(d["sigma"] * ko.keyed_gaussian(d["seed"], c["key"], run)) == hexf(r)
    for gm in d["geomean"]:
        assert ko.geometric_mean_error(gm["pairs"]) == hexf(gm["geomean"])


def test_markstein_division_is_correctly_rounded():
    """The GPU's row formation kcg_div (q = RN(c r), e = RN(c - q t) exact by
    FMA, RN(q + e r), r = RN(1/t)) equals IEEE division on random and
    all-ones-mantissa operands (exact rational FMA emulation here; the full
    300,000-case run is tests/gen/check_markstein_division.py)."""
    import random
    import struct
    from fractions import Fraction as Fr

    def fma(x, y, z):
        return float(Fr(x) * Fr(y) + Fr(z))

    def div_m(a, b):
        r = float(Fr(1) / Fr(b))
        q = a * r
        return fma(fma(-q, b, a), r, q)

    rng = random.Random(7)
    for i in range(20000):
        a = struct.unpack("<d", struct.pack("<Q", ((1023 + rng.randint(-60, 60)) << 52) | rng.getrandbits(52)))[0]
        m = ((1 << 52) - 1 - rng.randint(0, 3)) if i % 3 == 0 else rng.getrandbits(52)
        b = struct.unpack("<d", struct.pack("<Q", ((1023 + rng.randint(-60, 60)) << 52) | m))[0]
        assert div_m(a, b) == a / b, (a, b)
