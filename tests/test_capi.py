"""CPU-side checks of the C ABI (no kernel launches): the library loads and
exports every symbol include/kcg.h declares, programs parse and lower like
the reference front end printed them, errors map to the reference's Errc
codes, the weights file round-trips byte-identically, the host solve
reproduces the reference fit, and launches fail loudly without a GPU."""
import ctypes
import json
import math

import numpy as np
import pytest

import kc_oracle as ko
from conftest import FIT_ABS_SCALED, FIT_REL, GOLDEN, PROGRAMS, exact_fit, fit_errors, hexf, load_golden
import paper_1604_04997_b200 as kc
from paper_1604_04997_b200 import _capi


def test_library_exports_every_header_symbol():
    L = _capi.lib()
    names = _capi.header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n


def test_schema_matches_reference_order():
    assert kc.schema_keys() == ko.SCHEMA
    assert kc.schema_index("launch.const") == 148
    with pytest.raises(kc.KcgError) as e:
        kc.schema_index("mem.bogus")
    assert e.value.code == _capi.E_SCHEMA_MISMATCH


def test_every_suite_program_lowers():
    idx = {k["id"]: k for k in kc.suite_index()}
    n = 0
    for path in sorted(PROGRAMS.glob("*.kcp")):
        p = kc.Program.from_file(path)
        o = ko.Program(path.read_text())
        assert p.params == idx[path.stem]["params"] == o.params
        assert p.props == [k for k, _ in o.props]
        b64, b128 = p.safe_bounds()
        assert 0 < b64 <= b128
        n += 1
    assert n == 61  # 59 symbolic + fd_stencil / nbody derived (programs/derived.json)
    assert not idx["fd_stencil_g16x16"]["symbolic"] and not idx["nbody_g256"]["symbolic"]


def test_safe_bounds_are_sound_for_matmul():
    p = kc.load_program("matmul_tiled_g16x16")
    b64, b128 = p.safe_bounds()
    # largest count 4608 q^3 (q = n/16) must fit int63 at the bound
    assert 4608 * (b64 // 16) ** 3 < 2**63
    assert (b128 // 16) ** 3 * 4608 < 2**127


@pytest.mark.parametrize("text,code", [
    ("", _capi.E_PARSE),
    ("kernelcost-program v1\nkernel k\nparam n\nprop launch.const 1\n", _capi.E_PARSE),
    ("kernelcost-program v1\nkernel k\nparam n\nprop bogus.key n\nend\n", _capi.E_SCHEMA_MISMATCH),
    ("kernelcost-program v1\nkernel k\nparam n\nprop launch.const (* m 2)\nend\n", _capi.E_PARSE),
    ("kernelcost-program v1\nkernel k\nparam n\nassume n ~ 3\nend\n", _capi.E_PARSE),
    ("kernelcost-program v1\nkernel k\nparam n\nprop launch.const (floordiv n 0)\nend\n", _capi.E_PARSE),
])
def test_parse_errors(text, code):
    with pytest.raises(kc.KcgError) as e:
        kc.Program(text)
    assert e.value.code == code


def test_program_with_atoms_and_rationals_lowers():
    d = load_golden("extra_programs.json")
    for p in d["programs"]:
        if "program" in p:
            prog = kc.Program(p["program"])
            src = prog.jit_source()
            assert "kcg_fasti_0" in src and "kcg_wide_0" in src and "_tma" in src


def test_jit_source_has_no_divisions_after_congruence_substitution():
    src = kc.load_program("matmul_tiled_g16x16").jit_source()
    fast = src[src.index("kcg_fastd_0"):src.index("kcg_wide_0")]
    assert " % " not in fast and "4608" in fast


def test_launches_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = kc.load_program("conv_g16x16")
    rc = _capi.lib().kcg_eval_predict(p.handle, (ctypes.c_void_p * 1)(0), 4, None, None, None,
                                      None, None, 0, None)
    assert rc == _capi.E_CUDA
    assert b"no CUDA device" in _capi.lib().kcg_last_error()


def test_pipe_peak_probe_arguments_and_no_gpu():
    out = ctypes.c_double()
    assert _capi.lib().kcg_measure_pipe_peak(4, 16, ctypes.byref(out)) == _capi.E_INVALID_ARGUMENT
    assert _capi.lib().kcg_measure_pipe_peak(0, 0, ctypes.byref(out)) == _capi.E_INVALID_ARGUMENT
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _capi.lib().kcg_measure_pipe_peak(0, 16, ctypes.byref(out)) == _capi.E_CUDA


@pytest.mark.gpu
def test_pipe_peaks_are_plausible():
    """The instruction-roofline denominators (csrc/peaks.cu) on this device:
    every pipe below the issue bound (4 warp-instructions per clock per SM),
    the IMAD + LOP3 mix above either pipe alone."""
    import torch
    p = torch.cuda.get_device_properties(0)
    clock = 2.1e9  # above the B200's 1965 MHz boost
    issue_bound = p.multi_processor_count * 4 * 32 * clock
    r = {k: kc.measure_pipe_peak(k) for k in ("imad", "lop3", "dfma", "issue")}
    for k, v in r.items():
        assert 1e12 < v < issue_bound, (k, v)
    assert r["issue"] > 1.2 * max(r["imad"], r["lop3"]), r


def test_weights_json_round_trip_is_byte_identical(tmp_path):
    src = GOLDEN / "weights_suite.json"
    w = kc.read_weights_json(src)
    fit = load_golden("fit_suite.json")
    for k, v in fit["alpha"].items():
        assert w.alpha[ko.SCHEMA_INDEX[k]] == hexf(v[1])
    assert w.device == "simdev-v1" and w.n_cases == 390
    out = tmp_path / "w.json"
    kc.write_weights_json(out, w)
    assert out.read_bytes() == src.read_bytes()


def test_weights_json_errors(tmp_path):
    with pytest.raises(kc.KcgError) as e:
        kc.read_weights_json(tmp_path / "missing.json")
    assert e.value.code == _capi.E_IO
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"schema_version": "v0", "weights": {}}))
    with pytest.raises(kc.KcgError) as e:
        kc.read_weights_json(bad)
    assert e.value.code == _capi.E_SCHEMA_MISMATCH
    bad.write_text("{not json")
    with pytest.raises(kc.KcgError) as e:
        kc.read_weights_json(bad)
    assert e.value.code == _capi.E_PARSE


def _solve(X):
    F = X.shape[1]
    G = np.ascontiguousarray(X.T @ X)
    s1 = np.ascontiguousarray(X.sum(0))
    cm = np.ascontiguousarray(np.abs(X).max(0))
    out = (ctypes.c_double * F)()
    rank = ctypes.c_int()
    dp = lambda a: a.ctypes.data_as(_capi.DP)
    _capi.check(_capi.lib().kcg_solve_gram(F, dp(G), dp(s1), dp(cm), out, ctypes.byref(rank)))
    alpha = np.array(list(out))
    # two semi-normal refinement steps as fit_weights() does on the GPU: the
    # residual in extended precision (the GPU forms it in double-double)
    for _ in range(2):
        r = (1 - X.astype(np.longdouble) @ alpha.astype(np.longdouble)).astype(np.float64)
        g = np.ascontiguousarray(X.T @ r)
        arr = (ctypes.c_double * F)(*alpha)
        _capi.check(_capi.lib().kcg_refine_gram(F, dp(G), dp(cm), dp(g), arr))
        alpha = np.array(list(arr))
    return alpha, rank.value


def test_host_solve_reproduces_reference_fits():
    """The host solve + two refinement steps land within 1e-9 (relative, in
    the equilibrated coordinates; conftest.fit_errors) of the EXACT min-norm
    least-squares solution of each reference fixture's double design, and
    therefore within the reference COD's own distance from it plus 1e-9."""
    for fit in load_golden("fit_synthetic.json")["fits"]:
        counts = np.array(fit["counts"], dtype=np.float64)
        times = np.array([hexf(t) for t in fit["times"]])
        X = counts / times[:, None]
        alpha, rank = _solve(X)
        ref = [hexf(a) for a in fit["alpha"]]
        ex = [hexf(a) for a in exact_fit(fit["name"])["alpha_exact"]]
        cm = np.abs(X).max(axis=0)
        err = fit_errors(alpha, ex, cm)
        assert max(err) <= 1.0, (fit["name"], err)
        for k, got, r, e, c in zip(fit["keys"], alpha, ref, ex, cm):
            assert abs(got - r) <= abs(r - e) + FIT_REL * abs(e) + FIT_ABS_SCALED / c, (fit["name"], k, got, r)
        if fit["name"] == "duplicate_columns":
            assert rank == 2  # min-norm split of the two identical columns
        r = 1.0 - X @ alpha
        assert float(r @ r) <= max(1e-18, 10 * hexf(fit["objective"][1]))


def test_host_solve_suite_design_matches_reference(suite_alpha):
    cases = [c for c in load_golden("suite_cases.json")["cases"] if c["role"] == "measurement"]
    rows = [({ko.SCHEMA_INDEX[k]: int(v) for k, v in c["counts"].items()}, hexf(c["time_s"][1])) for c in cases]
    X, cov = ko.build_design_matrix(rows)
    cols = np.flatnonzero(cov)
    Xc = np.ascontiguousarray(X[:, cols])
    alpha, rank = _solve(Xc)
    ex = exact_fit("suite_measurement_390")
    assert ex["keys"] == [ko.SCHEMA[c] for c in cols]
    exa = [hexf(a) for a in ex["alpha_exact"]]
    err = fit_errors(alpha, exa, np.abs(Xc).max(axis=0))
    assert max(err) <= 1.0, err
    sim = ko.simdev_reference_alpha()
    for c, got in zip(cols, alpha):
        if sim[c] != 0.0:
            assert abs(got - suite_alpha[c]) <= 1e-9 * abs(suite_alpha[c]), ko.SCHEMA[c]
        else:
            assert abs(got) <= 1e-15


@pytest.mark.parametrize("kid", ["matmul_tiled_g16x16", "matmul_skinny_g16x16", "conv_g16x16",
                                 "arith_div_g16x12", "stride2_fill_g192", "transpose_tile_g16x16"])
def test_generated_kernels_compile_for_sm100a(kid):
    """NVRTC (sm_100a) accepts every specialised kernel family for the
    program -- eval (+ _gen, _tma), fused Gram (DMMA), fused residual and
    its refinement gradient."""
    p = kc.load_program(kid)
    L = _capi.lib()
    for kind, base in ((0, "kcg_eval_"), (1, "kcg_gram_"), (2, "kcg_resid_"), (3, "kcg_argmin"), (5, "kcg_rgrad_")):
        src = L.kcg_program_jit_source_kind(p.handle, kind)
        rc = L.kcg_jit_compile_check(src, (base + (kid if kind != 3 else "")).encode())
        assert rc == 0, L.kcg_last_error().decode()[:3000]


def test_generated_kernels_compile_for_atom_programs():
    d = load_golden("extra_programs.json")
    L = _capi.lib()
    for q in d["programs"]:
        if "program" not in q:
            continue
        p = kc.Program(q["program"])
        for kind in (0, 1):
            rc = L.kcg_jit_compile_check(L.kcg_program_jit_source_kind(p.handle, kind), b"k")
            assert rc == 0, L.kcg_last_error().decode()[:3000]


@pytest.mark.parametrize("name", ["meas_sigma0.csv", "raw_runs_sigma002.csv"])
def test_measurement_csv_reader_matches_oracle(name):
    """kcg_measurements_read_csv == the restated read_any_csv /
    reduce_raw_runs of the reference CLI (bitwise times, exact bindings)."""
    recs = ko.read_any_csv(GOLDEN / name)
    got = {}
    for km in kc.read_measurements(GOLDEN / name):
        for i in range(len(km.times)):
            key = (km.kernel, tuple(sorted((p, int(km.columns[p][i])) for p in km.params)))
            got.setdefault(key, []).append(float(km.times[i]))
    want = {}
    for k, b, t in recs:
        want.setdefault((k, tuple(sorted(b.items()))), []).append(t)
    assert got == want
    assert sum(len(v) for v in got.values()) == 390


def test_measurement_csv_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("kernel,binding,time_s\n")
    with pytest.raises(kc.KcgError) as e:
        kc.read_measurements(bad)
    assert e.value.code == _capi.E_PARSE
    bad.write_text("kernel,binding,group_config,time_s\nk,n=12,1,abc\n")
    with pytest.raises(kc.KcgError) as e:
        kc.read_measurements(bad)
    assert e.value.code == _capi.E_PARSE
    bad.write_text("kernel,binding,group_config,run_index,time_s\nk,n=12,1,0,1.0\n")
    with pytest.raises(kc.KcgError) as e:
        kc.read_measurements(bad)  # fewer runs than the 4 discarded warm-ups
    assert e.value.code == _capi.E_INVALID_ARGUMENT
    with pytest.raises(kc.KcgError) as e:
        kc.read_measurements(tmp_path / "missing.csv")
    assert e.value.code == _capi.E_IO


def test_host_build_of_generated_evaluator_matches_goldens():
    """The generated evaluator compiled for the host (source kind 4, g++
    -ffp-contract=off) reproduces the reference's golden grid samples bit for
    bit -- counts beyond 2^64 included: a CPU-side check of the code
    generator. (Baseline/cross-check tooling only; the package never falls
    back to it.)"""
    import collections

    import numpy as np

    from tools.hostbuild import HostEvaluator
    d = load_golden("grid_samples.json")["samples"]
    fit = load_golden("fit_suite.json")
    alpha = [0.0] * 149
    for k, v in fit["alpha"].items():
        alpha[ko.SCHEMA_INDEX[k]] = hexf(v[1])
    by = collections.defaultdict(list)
    for s in d:
        by[s["kernel"]].append(s)
    checked = 0
    for kid, ss in by.items():
        p = kc.load_program(kid)
        pred, st = HostEvaluator(p).predict(alpha, {q: np.array([int(s["binding"][q]) for s in ss], dtype=np.int64)
                                                    for q in p.params}, threads=2)
        for i, s in enumerate(ss):
            if s["status"] == "ok":
                assert st[i] == 0 and pred[i] == hexf(s["predicted_s"][1]), (kid, s["binding"])
                checked += 1
            else:
                assert st[i] != 0, (kid, s["binding"])
    assert checked > 1000


def test_design_and_time_inputs_are_validated():
    """gram_accumulate / fit_weights / gram_fused / residual_fused refuse
    inputs the kernels would mis-read (CPU, wrong dtype) before any launch."""
    import torch
    X = torch.zeros((8, 3), dtype=torch.float64)
    for f in (kc.gram_accumulate, kc.fit_weights):
        with pytest.raises(kc.KcgError) as e:
            f(X)
        assert e.value.code == _capi.E_INVALID_ARGUMENT


@pytest.mark.gpu
def test_design_and_time_inputs_are_validated_on_device():
    import torch
    X = torch.rand((64, 6), dtype=torch.float64, device="cuda")
    bad = [X[:, ::2], X.float(), X.T]
    for Xb in bad:
        with pytest.raises(kc.KcgError) as e:
            kc.gram_accumulate(Xb)
        assert e.value.code == _capi.E_INVALID_ARGUMENT
    prog = kc.load_program("matmul_tiled_g16x16")
    cols = {p: torch.full((32,), 64, dtype=torch.int64, device="cuda") for p in prog.params}
    a = [0.0] * kc.schema_size()
    for T in (torch.ones(31, dtype=torch.float64, device="cuda"), torch.ones(32, dtype=torch.float32, device="cuda"),
              torch.ones(64, dtype=torch.float64, device="cuda")[::2], torch.ones(32, dtype=torch.float64)):
        with pytest.raises(kc.KcgError):
            kc.gram_fused(prog, cols, T)
        with pytest.raises(kc.KcgError):
            kc.residual_fused(prog, cols, T, a)


def test_refinement_gradient_groups_power_of_two_keys():
    """kcg_rgrad_<k> forms one design-column division per group of keys whose
    counts differ by powers of two (tiled matmul: 9 keys -> 4 divisions)."""
    L = _capi.lib()
    for kid, want in (("matmul_tiled_g16x16", 4), ("conv_g16x16", 3), ("transpose_tile_g16x16", 2)):
        prog = kc.load_program(kid)  # the returned text is owned by the program: keep it alive
        src = L.kcg_program_jit_source_kind(prog.handle, 5).decode()
        i = src.index("kcg_xrow(const T* c")
        assert src[i:src.index("}", i)].count("__ddiv_rn") == want, kid
