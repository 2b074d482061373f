"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors. Counts bit-exact, predictions bitwise, statuses
equal. Both engines (NVRTC-specialised and table interpreter) are checked."""
import math
import random

import numpy as np
import pytest

import kc_oracle as ko
from conftest import FIT_ABS_SCALED, FIT_REL, GOLDEN, PROGRAMS, exact_fit, fit_errors, hexf, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_1604_04997_b200 as kc  # noqa: E402
from paper_1604_04997_b200 import _capi  # noqa: E402

ENGINES = ["jit", "interp"]
ST_NAME = {0: "ok", 1: "E_ASSUMPTION_VIOLATED", 2: "NONINTEGRAL", 3: "OVERFLOW", 4: "COUNT_WIDE"}


def _weights(alpha):
    return kc.ModelWeights(device="t", alpha=list(alpha), covered=[a != 0 for a in alpha])


def _cols(prog, bindings):
    return {p: torch.tensor([b[p] for b in bindings], dtype=torch.int64, device="cuda")
            for p in prog.params}


def _run(prog, bindings, alpha, engine):
    prog.set_engine(engine)
    cols = _cols(prog, bindings)
    bb = kc.evaluate_properties(prog, cols, wide=True)
    pred, st = kc.predict(_weights(alpha), prog, cols, with_status=True)
    torch.cuda.synchronize()
    lo = bb.counts_lo.cpu().numpy()
    hi = bb.counts_hi.cpu().numpy()
    return lo, hi, bb.status.cpu().numpy(), pred.cpu().numpy(), st.cpu().numpy()


def _as_int(lo, hi):
    return (int(hi) << 64) | (int(lo) & ((1 << 64) - 1))


def _compare(prog, oprog, bindings, alpha, engine, expect=None):
    lo, hi, st, pred, st2 = _run(prog, bindings, alpha, engine)
    assert (st == st2).all()
    for i, b in enumerate(bindings):
        try:
            want = oprog.evaluate_properties(b)
            want_st = 0
        except ko.AssumptionViolated:
            want_st = 1
        except ko.NonIntegral:
            want_st = 2
        if expect is not None and expect[i] is not None:
            assert ST_NAME[want_st] == expect[i] or expect[i] == "ok" and want_st == 0
        assert st[i] == want_st, (prog.name, engine, b, st[i], want_st)
        if want_st == 0:
            for j, k in enumerate(prog.props):
                assert _as_int(lo[j, i], hi[j, i]) == want[k], (prog.name, b, k)
            assert pred[i] == ko.predict(alpha, want), (prog.name, b)
        else:
            assert math.isnan(pred[i])


@pytest.fixture(scope="module")
def programs():
    return {p.stem: (kc.Program.from_file(p), ko.Program(p.read_text()))
            for p in sorted(PROGRAMS.glob("*.kcp"))}


@pytest.mark.parametrize("engine", ENGINES)
def test_suite_manifest_cases(programs, suite_alpha, engine):
    cases = load_golden("suite_cases.json")["cases"]
    by_kernel = {}
    for c in cases:
        by_kernel.setdefault(c["kernel"], []).append({k: int(v) for k, v in c["binding"].items()})
    for kid, (prog, oprog) in programs.items():
        bs = list(by_kernel[kid])
        # perturbations: inadmissible neighbours and negatives (props.cpp:263-266)
        bs += [{k: v + 1 for k, v in b.items()} for b in by_kernel[kid][:2]]
        bs += [{k: -v for k, v in b.items()} for b in by_kernel[kid][:1]]
        bs += [{k: 0 for k in b} for b in by_kernel[kid][:1]]
        _compare(prog, oprog, bs, suite_alpha, engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_golden_grid_samples(programs, suite_alpha, engine):
    samples = load_golden("grid_samples.json")["samples"]
    groups = {}
    for s in samples:
        groups.setdefault(s["kernel"], []).append(s)
    for kid, ss in groups.items():
        prog, oprog = programs[kid]
        bs = [{k: int(v) for k, v in s["binding"].items()} for s in ss]
        prog.set_engine(engine)
        lo, hi, st, pred, _ = _run(prog, bs, suite_alpha, engine)
        for i, s in enumerate(ss):
            if s["status"] == "ok":
                assert st[i] == 0, (kid, s["binding"])
                want = {ko.SCHEMA_INDEX[k]: int(v) for k, v in s["counts"].items()}
                for j, k in enumerate(prog.props):
                    assert _as_int(lo[j, i], hi[j, i]) == want.get(k, 0)
                assert pred[i] == hexf(s["predicted_s"][1]), (kid, s["binding"])
            else:
                assert st[i] == _capi.PT_ASSUMPTION_VIOLATED


@pytest.mark.parametrize("engine", ENGINES)
def test_extra_programs_atoms(suite_alpha, engine):
    d = load_golden("extra_programs.json")
    progs = {p["id"]: (kc.Program(p["program"]), ko.Program(p["program"]))
             for p in d["programs"] if "program" in p}
    groups = {}
    for s in d["samples"]:
        groups.setdefault(s["kernel"], []).append(s)
    for kid, ss in groups.items():
        prog, oprog = progs[kid]
        bs = [{k: int(v) for k, v in s["binding"].items()} for s in ss]
        _compare(prog, oprog, bs, suite_alpha, engine,
                 expect=[s["status"] if s["status"] != "E_ASSUMPTION_VIOLATED" else "E_ASSUMPTION_VIOLATED" for s in ss])


@pytest.mark.parametrize("engine", ENGINES)
def test_wide_and_overflow_paths(suite_alpha, engine):
    """Counts beyond 2^63 / 2^64 go through the int128 path bit-exactly;
    bindings beyond the 128-bit safe bound report OVERFLOW, never wrap."""
    for kid in ("matmul_skinny_g16x16", "matmul_tiled_g16x16", "conv_g16x16"):
        prog = kc.load_program(kid)
        oprog = ko.Program((PROGRAMS / f"{kid}.kcp").read_text())
        b64, b128 = prog.safe_bounds()
        rng = random.Random(7)
        bs = []
        for _ in range(300):
            n = 16 * rng.randint(1, b128 // 16 // (8 if "skinny" in kid else 1))
            b = {p: n for p in prog.params}
            if "skinny" in kid:
                b["m"] = 8 * n
            bs.append(b)
        for edge in (b64 - b64 % 16, b64 - b64 % 16 + 16, b128 - b128 % 16):
            bs.append({p: edge for p in prog.params})
        _compare(prog, oprog, [b for b in bs if max(b.values()) <= b128], suite_alpha, engine)
        over = [{p: b128 - b128 % 16 + 16 * k for p in prog.params} for k in (1, 2, 1000)]
        _, _, st, pred, _ = _run(prog, over, suite_alpha, engine)
        assert (st == _capi.PT_OVERFLOW).all() and np.isnan(pred).all()


def test_count_wide_status_without_hi_words(suite_alpha):
    prog = kc.load_program("matmul_skinny_g16x16")
    n = 1 << 24
    cols = _cols(prog, [{"n": n, "m": 8 * n, "l": n}, {"n": 16, "m": 128, "l": 16}])
    bb = kc.evaluate_properties(prog, cols, wide=False)
    st = bb.status.cpu().tolist()
    assert st == [_capi.PT_COUNT_WIDE, _capi.PT_OK]


def test_simulate_order_matches_noiseless_time(programs):
    sim = ko.simdev_reference_alpha()
    cases = load_golden("suite_cases.json")["cases"]
    for kid, (prog, oprog) in programs.items():
        bs = [{k: int(v) for k, v in c["binding"].items()} for c in cases if c["kernel"] == kid]
        t = kc.noiseless_time(sim, prog, _cols(prog, bs)).cpu().numpy()
        want = [hexf(c["time_s"][1]) for c in cases if c["kernel"] == kid]
        assert list(t) == want, kid


def test_argmin_over_matmul_variants(suite_alpha):
    ids = ["matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
           "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16"]
    progs = [kc.load_program(i) for i in ids]
    oprogs = [ko.Program((PROGRAMS / f"{i}.kcp").read_text()) for i in ids]
    rng = random.Random(3)
    bs = [{"n": 336 * rng.randint(1, 551), "m": 336 * rng.randint(1, 551), "l": 336 * rng.randint(1, 551)}
          for _ in range(500)]
    bs += [{"n": 16 * rng.randint(1, 200), "m": 16 * rng.randint(1, 200), "l": 16 * rng.randint(1, 200)}
           for _ in range(500)]  # g12/g14 variants often inadmissible here
    bs.append({"n": 17, "m": 17, "l": 17})  # nobody admissible
    cols = _cols(progs[0], bs)
    best, best_t, preds = kc.argmin(progs, _weights(suite_alpha), cols, return_preds=True)
    best, best_t, preds = best.cpu().numpy(), best_t.cpu().numpy(), preds.cpu().numpy()
    for i, b in enumerate(bs):
        ts = []
        for v, op in enumerate(oprogs):
            try:
                ts.append(ko.predict(suite_alpha, op.evaluate_properties(b)))
            except ko.AssumptionViolated:
                ts.append(math.nan)
        for v in range(len(ids)):
            assert (math.isnan(ts[v]) and math.isnan(preds[v, i])) or ts[v] == preds[v, i]
        fin = [(t, v) for v, t in enumerate(ts) if not math.isnan(t)]
        if fin:
            t, v = min(fin)
            assert best[i] == v and best_t[i] == t
        else:
            assert best[i] == -1 and math.isinf(best_t[i])


def test_gram_accumulate_matches_numpy():
    rng = np.random.default_rng(0)
    for F, N in ((1, 5001), (3, 5003), (9, 300_009), (18, 5018), (40, 5040), (47, 200_047), (64, 5064),
                 (100, 20_100), (149, 30_149)):
        X = rng.uniform(0.5, 2.0, size=(N, F)) * 10.0 ** rng.integers(-3, 3, size=F)
        X[rng.random((N, F)) < 0.1] = 0.0
        Xd = torch.tensor(X, device="cuda")
        st = kc.gram_accumulate(Xd)
        torch.cuda.synchronize()
        G = st.G.cpu().numpy()
        np.testing.assert_allclose(G, X.T @ X, rtol=1e-12, atol=0)
        np.testing.assert_allclose(st.xt1.cpu().numpy(), X.sum(axis=0), rtol=1e-12)
        assert (st.colmax.cpu().numpy() == np.abs(X).max(axis=0)).all()


def _synthetic_design(fit):
    keys = fit["keys"]
    counts = np.array(fit["counts"], dtype=np.float64)
    times = np.array([hexf(t) for t in fit["times"]])
    X = counts / times[:, None]
    return keys, X


def test_fit_weights_matches_reference_cod():
    """GPU Gram + host solve + two double-double refinement passes: within
    1e-9 (conftest.fit_errors) of the exact min-norm LS solution of every
    reference fixture, so within the reference COD's own distance from it
    (3.8e-9 on config3_f40_n4000, tests/golden/fit_exact.json) plus 1e-9."""
    for fit in load_golden("fit_synthetic.json")["fits"]:
        keys, X = _synthetic_design(fit)
        res = kc.fit_weights(torch.tensor(X, device="cuda"))
        ref = [hexf(a) for a in fit["alpha"]]
        ex = [hexf(a) for a in exact_fit(fit["name"])["alpha_exact"]]
        cm = np.abs(X).max(axis=0)
        err = fit_errors(res.alpha, ex, cm)
        assert max(err) <= 1.0, (fit["name"], err)
        for k, got, r, e, c in zip(keys, res.alpha, ref, ex, cm):
            assert abs(got - r) <= abs(r - e) + FIT_REL * abs(e) + FIT_ABS_SCALED / c, (fit["name"], k, got, r)
        assert res.objective <= max(1e-18, 10 * hexf(fit["objective"][1])) + 1e-20


def test_fit_suite_from_golden_counts(suite_alpha):
    """config 1: the measurement-suite design (390 x 149) through the GPU
    Gram + host solve reproduces the reference's fitted weights."""
    cases = [c for c in load_golden("suite_cases.json")["cases"] if c["role"] == "measurement"]
    rows = [({ko.SCHEMA_INDEX[k]: int(v) for k, v in c["counts"].items()}, hexf(c["time_s"][1])) for c in cases]
    X, cov = ko.build_design_matrix(rows)
    cols = np.flatnonzero(cov)
    Xc = np.ascontiguousarray(X[:, cols])
    res = kc.fit_weights(torch.tensor(Xc, device="cuda"), refine=2)
    exa = [hexf(a) for a in exact_fit("suite_measurement_390")["alpha_exact"]]
    err = fit_errors(res.alpha, exa, np.abs(Xc).max(axis=0))
    assert max(err) <= 1.0, err
    sim = ko.simdev_reference_alpha()
    for c, got in zip(cols, res.alpha):
        ref = suite_alpha[c]
        if sim[c] != 0.0:
            assert abs(got - ref) <= 1e-9 * abs(ref), ko.SCHEMA[c]
        else:
            assert abs(got) <= 1e-15
    assert res.objective <= 1e-10


def test_gram_fused_matches_oracle_rows():
    prog = kc.load_program("matmul_tiled_g16x16")
    oprog = ko.Program((PROGRAMS / "matmul_tiled_g16x16.kcp").read_text())
    rng = random.Random(11)
    bs = [{"n": 16 * rng.randint(1, 300), "m": 16 * rng.randint(1, 300), "l": 16 * rng.randint(1, 300)}
          for _ in range(4000)]
    bs += [{"n": 17, "m": 16, "l": 16}]  # inadmissible row is skipped and counted
    sim = ko.simdev_reference_alpha()
    T = []
    rows = []
    for b in bs:
        try:
            c = oprog.evaluate_properties(b)
            t = ko.noiseless_time(sim, c) * (1.0 + 0.01 * rng.random())
            rows.append([float(c[k]) / t for k in prog.props])
        except ko.AssumptionViolated:
            t = 1.0
        T.append(t)
    X = np.array(rows)
    cols = _cols(prog, bs)
    Td = torch.tensor(T, dtype=torch.float64, device="cuda")
    st = kc.gram_fused(prog, cols, Td)
    torch.cuda.synchronize()
    assert st.bad_rows == 1
    np.testing.assert_allclose(st.G.cpu().numpy(), X.T @ X, rtol=1e-11)
    np.testing.assert_allclose(st.xt1.cpu().numpy(), X.sum(axis=0), rtol=1e-11)
    # basis rows u_b = mono_b / T expanded by the exact key coefficients:
    # colmax within a few ulp of max |RN(count) / T|
    np.testing.assert_allclose(st.colmax.cpu().numpy(), np.abs(X).max(axis=0), rtol=1e-15, atol=0)
    # fused residual pass == numpy objective at some weights
    alpha = [0.0] * 149
    for j, k in enumerate(prog.props):
        alpha[k] = sim[k] * 1.001 + 1e-15
    got = kc.residual_fused(prog, cols, Td, alpha)
    a = np.array([alpha[k] for k in prog.props])
    r = 1.0 - X @ a
    assert got == pytest.approx(float(r @ r), rel=1e-9)


def test_no_silent_fallback_launches_counted():
    before = kc.launch_count()
    prog = kc.load_program("conv_g16x16")
    kc.evaluate_properties(prog, _cols(prog, [{"n": 16}]))
    torch.cuda.synchronize()
    assert kc.launch_count() == before + 1


@pytest.mark.parametrize("kid", ["matmul_tiled_g12x12", "conv_g16x16", "matmul_skinny_g16x16"])
def test_large_launch_tma_path_matches_interpreter(kid, suite_alpha):
    """Launches large enough for the TMA-staged persistent kernel (>= 148
    tiles of 1024 points, ragged tail) agree bitwise with the table
    interpreter and with the oracle on a sample, including inadmissible and
    wide-path points mixed into the stream."""
    prog = kc.load_program(kid)
    oprog = ko.Program((PROGRAMS / f"{kid}.kcp").read_text())
    g = torch.Generator(device="cpu").manual_seed(5)
    n = 148 * 1024 * 2 + 777
    unit = 12 if "g12" in kid else 16
    u = torch.randint(1, 20000, (len(prog.params), n), generator=g)
    cols = {p: (u[j] * unit).to(torch.int64) for j, p in enumerate(prog.params)}
    if "skinny" in kid:
        cols["m"] = cols["n"] * 8
    cols[prog.params[0]][::97] += 1                  # inadmissible
    cols[prog.params[0]][5::1013] = 16 * 3_000_000   # wide path
    cols = {k: v.cuda().contiguous() for k, v in cols.items()}
    w = _weights(suite_alpha)
    prog.set_engine("jit")
    pj, sj = kc.predict(w, prog, cols, with_status=True)
    prog.set_engine("interp")
    pi, si = kc.predict(w, prog, cols, with_status=True)
    torch.cuda.synchronize()
    assert torch.equal(sj, si)
    same = (pj == pi) | (torch.isnan(pj) & torch.isnan(pi))
    assert bool(same.all())
    for i in list(range(0, n, n // 97)) + [n - 1, n - 2, 5, 97]:
        b = {p: int(cols[p][i]) for p in prog.params}
        try:
            want = ko.predict(suite_alpha, oprog.evaluate_properties(b))
            assert float(pj[i]) == want and int(sj[i]) == 0
        except ko.AssumptionViolated:
            assert int(sj[i]) == 1


@pytest.mark.parametrize("in_off,out_off", [(0, 1), (1, 0), (1, 1)])
def test_unaligned_buffers_through_c_abi(suite_alpha, in_off, out_off):
    """Odd element offsets (8-byte but not 16-byte aligned) for the binding
    columns and/or the outputs select the scalar paths; results are
    identical to the aligned launch."""
    import ctypes
    prog = kc.load_program("matmul_tiled_g16x16")
    n = 148 * 1024 + 333
    g = torch.Generator(device="cpu").manual_seed(9)
    base = {p: (torch.randint(1, 5000, (n + 1,), generator=g) * 16).cuda() for p in prog.params}
    base["n"][::31] += 3
    w = _weights(suite_alpha)
    ref, ref_st = kc.predict(w, prog, {p: base[p][:n].contiguous() for p in prog.params}, with_status=True)
    cols = [base[p][in_off:in_off + n] for p in prog.params]
    arr = (ctypes.c_void_p * 3)(*[c.data_ptr() for c in cols])
    pred = torch.empty(n + 1, dtype=torch.float64, device="cuda")[out_off:out_off + n]
    st = torch.empty(n + 1, dtype=torch.uint8, device="cuda")[out_off:out_off + n]
    if in_off:
        ref, ref_st = kc.predict(w, prog, {p: base[p][1:n + 1].contiguous() for p in prog.params}, with_status=True)
    _capi.check(_capi.lib().kcg_eval_predict(prog.handle, arr, n, w.alpha_array(), pred.data_ptr(),
                                             st.data_ptr(), None, None, 0,
                                             torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(st, ref_st)
    assert bool(((pred == ref) | (torch.isnan(pred) & torch.isnan(ref))).all())


def test_fused_gram_large_matches_materialised_path():
    """>= 148 TMA tiles plus a ragged tail: the fused evaluate -> row -> Gram
    (DMMA) equals the Gram of rows materialised from evaluate_properties
    counts, and the fused residual equals the materialised residual."""
    prog = kc.load_program("matmul_tiled_g16x16")
    sim = ko.simdev_reference_alpha()
    n = 148 * 1024 * 2 + 555
    g = torch.Generator(device="cpu").manual_seed(21)
    cols = {p: (torch.randint(1, 3000, (n,), generator=g) * 16).cuda() for p in prog.params}
    cols["n"][::101] += 1  # inadmissible rows are skipped and counted
    T = kc.noiseless_time(sim, prog, cols) * (1.0 + 0.01 * torch.rand(n, generator=g, dtype=torch.float64).cuda())
    st = kc.gram_fused(prog, cols, T)
    bb = kc.evaluate_properties(prog, cols)
    ok = bb.status == 0
    X = (bb.counts_lo.to(torch.float64) / T).T[ok].contiguous()
    ref = kc.gram_accumulate(X)
    torch.cuda.synchronize()
    assert st.bad_rows == int((~ok).sum())
    torch.testing.assert_close(st.G, ref.G, rtol=1e-11, atol=0)
    torch.testing.assert_close(st.xt1, ref.xt1, rtol=1e-11, atol=0)
    torch.testing.assert_close(st.colmax, ref.colmax, rtol=1e-15, atol=0)
    alpha = [0.0] * 149
    for k in prog.props:
        alpha[k] = sim[k] * 0.999
    a = torch.tensor([alpha[k] for k in prog.props], dtype=torch.float64, device="cuda")
    want = float(((1.0 - X @ a) ** 2).sum())
    assert kc.residual_fused(prog, cols, T, alpha) == pytest.approx(want, rel=1e-9)


def test_simulate_time_with_noise_matches_reference(programs):
    """simulate_time / simulate_runs with sigma = 0.02, seed 7 for every
    measurement case of a symbolic kernel: the noise key "<kernel>|<binding>"
    is hashed on the GPU exactly like simdevice.cpp; exp/log/cos are CUDA's,
    so times agree to a few ulps (sigma = 0 is bitwise, see
    test_simulate_order_matches_noiseless_time)."""
    d = load_golden("simulate.json")
    sim = ko.simdev_reference_alpha()
    groups = {}
    for c in d["cases"]:
        groups.setdefault(c["kernel"], []).append(c)
    worst = 0.0
    for kid, cs in groups.items():
        prog, _ = programs[kid]
        cols = _cols(prog, [{k: int(v) for k, v in c["binding"].items()} for c in cs])
        for run in range(3):
            t = kc.simulate_time(sim, prog, cols, sigma=d["sigma"], seed=d["seed"], run=run).cpu().numpy()
            for i, c in enumerate(cs):
                want = hexf(c["runs"][run])
                worst = max(worst, abs(t[i] - want) / want)
        t0 = kc.simulate_time(sim, prog, cols, sigma=0.0).cpu().numpy()
        assert list(t0) == [hexf(c["noiseless"]) for c in cs]
    assert worst < 1e-14, worst


def test_geometric_mean_error_fixtures():
    for g in load_golden("simulate.json")["geomean"]:
        p = torch.tensor([x[0] for x in g["pairs"]], dtype=torch.float64, device="cuda")
        a = torch.tensor([x[1] for x in g["pairs"]], dtype=torch.float64, device="cuda")
        assert kc.geometric_mean_error(p, a) == pytest.approx(hexf(g["geomean"]), rel=1e-14)
    with pytest.raises(kc.KcgError):
        kc.geometric_mean_error(torch.ones(2, dtype=torch.float64, device="cuda"),
                                torch.zeros(2, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("name", ["meas_sigma0.csv", "raw_runs_sigma002.csv"])
def test_cli_fit_and_eval_from_csv(name, tmp_path):
    """`kernelcost fit` / `eval` on the reference's own campaign CSVs
    (noiseless and 8 noisy raw runs per case), on the GPU: weights within the
    reference's 1e-6, per-kernel geometric mean errors to 1e-6 (bitwise
    predictions when given the reference's weights)."""
    ref = load_golden("cli_fit_eval.json")[name]
    path = GOLDEN / name
    w, rep = kc.fit_from_csv(path, device="gpu-sim")
    assert rep["n_cases"] == ref["n_records"] == 390
    # against the exact min-norm LS solution of the CSV's design (1e-9,
    # conftest.fit_errors; colmax from the GPU Gram statistics' rows)
    ex = exact_fit(f"cli_{name}")
    recs = ko.read_any_csv(path)
    progs = {}
    rows = []
    for kernel, binding, t in recs:
        progs.setdefault(kernel, ko.Program((PROGRAMS / f"{kernel}.kcp").read_text()))
        rows.append((progs[kernel].evaluate_properties(binding), t))
    X, cov = ko.build_design_matrix(rows)
    cols = [ko.SCHEMA_INDEX[k] for k in ex["keys"]]
    cm = np.abs(X[:, cols]).max(axis=0)
    got = [w.alpha[c] for c in cols]
    err = fit_errors(got, [hexf(a) for a in ex["alpha_exact"]], cm)
    assert max(err) <= 1.0, (name, err)
    for k, v in ref["alpha"].items():
        r, got = hexf(v), w.alpha[ko.SCHEMA_INDEX[k]]
        if abs(r) > 1e-15:
            assert abs(got - r) <= 1e-9 * abs(r), (name, k, got, r)
    assert rep["objective"] == pytest.approx(hexf(ref["objective"]), rel=1e-6, abs=1e-20)
    # eval with the reference's weights: predictions are bitwise, geomeans ~ulp
    wref = kc.ModelWeights(device="ref", alpha=[0.0] * 149, covered=[False] * 149)
    for k, v in ref["alpha"].items():
        wref.alpha[ko.SCHEMA_INDEX[k]] = hexf(v)
        wref.covered[ko.SCHEMA_INDEX[k]] = True
    ev = kc.eval_from_csv(wref, path)
    for k, v in ref["geomean_per_kernel"].items():
        assert ev["per_kernel"][k] == pytest.approx(hexf(v), rel=1e-12), k
    assert ev["overall"] == pytest.approx(hexf(ref["geomean_overall"]), rel=1e-12)
    # and the weights file round-trips through the reference format
    kc.write_weights_json(tmp_path / "w.json", w)
    w2 = kc.read_weights_json(tmp_path / "w.json")
    assert w2.alpha == w.alpha and w2.n_cases == 390


def _extra_program(name):
    for q in load_golden("extra_programs.json")["programs"]:
        if "program" in q and f"kernel {name}\n" in q["program"]:
            return kc.Program(q["program"])
    raise KeyError(name)


@pytest.mark.parametrize("kid", ["matmul_tiled_g16x16", "matmul_naive_g16x12", "conv_g16x16",
                                 "fd_stencil_g16x16", "nbody_g256", "x_triangle", "x_simplex", "x_minmax",
                                 "x_floordiv2"])
def test_fused_gram_basis_matches_direct_and_materialised(kid):
    """The monomial-basis fused Gram (u_b = mono_b / T, G = A Gu A^T per
    CTA) and the one-column-per-key path both equal the Gram of the
    materialised design rows RN(count)/T: G and X^T 1 to 1e-11, colmax
    bitwise (direct) or within 1e-15 (basis); the fused residual agrees in
    both modes. Covers single-term keys (matmul, conv), compound keys with
    positive terms (x_triangle: n/2 + n^2/2, expanded in the basis) and
    with cancelling terms (x_simplex: kept per key), floordiv atoms."""
    prog = kc.load_program(kid) if not kid.startswith("x_") else _extra_program(kid)
    n = 148 * 1024 * 2 + 555
    g = torch.Generator(device="cpu").manual_seed(77)
    unit = {"nbody_g256": 256}.get(kid, 336 if not kid.startswith("x_") else 1)
    lo = 7 if kid.startswith("x_") else 1
    cols = {p: (torch.randint(lo, 3000, (n,), generator=g) * unit).cuda() for p in prog.params}
    cols[prog.params[0]][::101] += 1 if unit > 1 else 0   # inadmissible rows (aligned kernels)
    cols[prog.params[0]][7::211] = -3                      # inadmissible everywhere
    T = (0.001 + torch.rand(n, generator=g, dtype=torch.float64)).cuda()
    bb = kc.evaluate_properties(prog, cols)
    ok = bb.status == 0
    X = (bb.counts_lo.to(torch.float64) / T).T[ok].contiguous()
    ref = kc.gram_accumulate(X)
    alpha = [0.0] * 149
    for j, k in enumerate(prog.props):
        alpha[k] = 1e-9 * (1 + j)
    a = torch.tensor([alpha[k] for k in prog.props], dtype=torch.float64, device="cuda")
    want_obj = float(((1.0 - X @ a) ** 2).sum())
    for basis in (True, False):
        prog.set_gram_basis(basis)
        st = kc.gram_fused(prog, cols, T)
        obj = kc.residual_fused(prog, cols, T, alpha)
        torch.cuda.synchronize()
        assert st.bad_rows == int((~ok).sum())
        torch.testing.assert_close(st.G, ref.G, rtol=1e-11, atol=0)
        torch.testing.assert_close(st.xt1, ref.xt1, rtol=1e-11, atol=0)
        if basis:
            torch.testing.assert_close(st.colmax, ref.colmax, rtol=1e-15, atol=0)
        else:
            assert torch.equal(st.colmax, ref.colmax)
        assert obj == pytest.approx(want_obj, rel=1e-9)
    prog.set_gram_basis(True)


def test_fit_weights_full_schema_width():
    """A materialised design as wide as the schema (149 columns: the CUDA-core
    Gram with one 4x4 tile per thread, the 5-column-per-lane residual and
    gradient kernels) recovers the generating weights like the reference's
    noiseless fits (test_model.cpp:43-61: rel 1e-6)."""
    g = torch.Generator(device="cpu").manual_seed(149)
    F, N = 149, 60_000
    C = torch.randint(1, 10001, (N, F), generator=g).to(torch.float64)
    alpha = torch.exp(torch.empty(F, dtype=torch.float64).uniform_(math.log(1e-13), math.log(1e-9), generator=g))
    T = C @ alpha
    X = (C / T[:, None]).cuda()
    fit = kc.fit_weights(X, refine=2)
    got = torch.tensor(fit.alpha, dtype=torch.float64)
    assert float(((got - alpha).abs() / alpha).max()) < 1e-6
    assert fit.objective < 1e-18


def test_predict_detail_matches_reference_predictions():
    """Prediction{seconds, breakdown, warnings} (model.cpp:95-117) for the 16
    test cases with the reference-fitted weights: seconds bitwise, the same
    (empty) warnings as the reference, breakdown parts summing in schema
    order; with keys marked uncovered the warnings list exactly those keys
    that carry a nonzero count."""
    fit = load_golden("fit_suite.json")
    w = kc.ModelWeights(device="ref", alpha=[0.0] * 149, covered=[False] * 149)
    for k, v in fit["alpha"].items():
        w.alpha[ko.SCHEMA_INDEX[k]] = hexf(v[1])
    for k in fit["covered"]:
        w.covered[ko.SCHEMA_INDEX[k]] = True
    for t in fit["test_predictions"]:
        prog = kc.load_program(t["kernel"])
        b = {p: int(v) for p, v in t["binding"].items()}
        (pd,) = kc.predict_detail(w, prog, _cols(prog, [b]))
        assert pd.seconds == hexf(t["predicted_s"][1]), t["kernel"]
        assert pd.warnings == t["warnings"]
        s = 0.0
        for _, part in pd.breakdown:
            s += part
        assert s == pd.seconds
    prog = kc.load_program("matmul_tiled_g16x16")
    w2 = kc.ModelWeights(device="x", alpha=list(w.alpha), covered=[False] * 149)
    (pd,) = kc.predict_detail(w2, prog, _cols(prog, [{"n": 64, "m": 32, "l": 48}, {"n": 65, "m": 32, "l": 48}]), [0])
    assert pd.warnings == [ko.SCHEMA[k] for k in prog.props]
    assert kc.predict_detail(w2, prog, _cols(prog, [{"n": 65, "m": 32, "l": 48}]))[0] is None


def test_gram_accumulate_random_shapes():
    """Every Gram path (DMMA row-split for F <= 72 -- two CTAs per SM up to
    F = 40, one beyond --, the DMMA + DFMA hybrid for even F in 34..40, the
    row-per-lane DFMA kernel for F <= 6, 9..11, 17..19, per-width DMMA for
    73..160, CUDA-core for strided / unaligned X) against torch fp64 on
    random widths, row counts (tails included) and layouts."""
    rng = np.random.default_rng(123)
    widths = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 17, 18, 19, 20, 21, 22, 26, 31, 32, 34, 40, 41, 48, 49, 57, 64,
              65, 72, 73, 80, 81, 111, 131, 149, 160]
    for F in widths:
        N = int(rng.integers(1, 5000)) + (70_000 if F in (2, 9, 12, 18, 22, 32, 40, 41, 57, 72, 131) else 0)
        ld = F + (3 if F % 3 == 0 else 0)  # some strided layouts
        base = torch.tensor(rng.uniform(0.5, 2.0, size=(N, ld)) * 10.0 ** rng.integers(-2, 3, size=ld),
                            device="cuda")
        X = base[:, :F]
        st = kc.GramStats.zeros(F, X.device)
        _capi.check(_capi.lib().kcg_gram_accumulate(X.data_ptr(), N, F, ld, st.G.data_ptr(), st.xt1.data_ptr(),
                                                    st.colmax.data_ptr(), torch.cuda.current_stream().cuda_stream))
        ref = X.T @ X
        torch.testing.assert_close(st.G, ref, rtol=1e-12, atol=0, msg=f"F={F} N={N} ld={ld}")
        torch.testing.assert_close(st.xt1, X.sum(0), rtol=1e-12, atol=0)
        assert torch.equal(st.colmax, X.abs().max(0).values), F


def _wide_program(nkeys=60):
    keys = kc.schema_keys()
    lines = ["kernelcost-program v1", f"kernel wide{nkeys}", "param n", "param m", "assume n >= 1", "assume m >= 1"]
    k = 0
    for a in range(1, 9):
        for b in range(0, 8):
            if k < nkeys:
                lines.append(f"prop {keys[k]} (* (^ n {a}) (^ m {b}))" if b else f"prop {keys[k]} (^ n {a})")
                k += 1
    return kc.Program("\n".join(lines + ["end"]) + "\n")


def test_fused_gram_wide_rows_take_the_chunked_path():
    """60 keys over 60 distinct monomials (no narrower basis): the fused Gram
    and residual form rows in HBM chunk by chunk (exact counts -> RN(count)/T
    -> the per-width DMMA Gram) and equal the materialised statistics; bad
    rows are counted."""
    prog = _wide_program()
    g = torch.Generator(device="cpu").manual_seed(60)
    n = (1 << 18) + 1234  # two chunks
    cols = {p: torch.randint(1, 21, (n,), generator=g).cuda() for p in prog.params}
    cols["n"][::97] = -1  # inadmissible
    T = (0.5 + torch.rand(n, generator=g, dtype=torch.float64)).cuda()
    st = kc.gram_fused(prog, cols, T)
    bb = kc.evaluate_properties(prog, cols)
    ok = bb.status == 0
    X = (bb.counts_lo.to(torch.float64) / T).T[ok].contiguous()
    ref = kc.gram_accumulate(X)
    alpha = [1e-12 * (1 + (i % 5)) for i in range(149)]
    a = torch.tensor([alpha[k] for k in prog.props], dtype=torch.float64, device="cuda")
    want = float(((1.0 - X @ a) ** 2).sum())
    got = kc.residual_fused(prog, cols, T, alpha)
    torch.cuda.synchronize()
    assert st.bad_rows == int((~ok).sum())
    torch.testing.assert_close(st.G, ref.G, rtol=1e-12, atol=0)
    torch.testing.assert_close(st.xt1, ref.xt1, rtol=1e-12, atol=0)
    assert torch.equal(st.colmax, ref.colmax)
    assert got == pytest.approx(want, rel=1e-12)


def test_fit_fused_reaches_the_exact_min_norm_solution():
    """fit_fused (fused Gram over the monomial basis + solve + two fused
    double-double refinement passes) on rows formed from bindings and
    noisy times: within 1e-9 of the exact min-norm LS solution of the
    unrounded rows count/T (model.cpp:11-35; the tiled matmul's 9 keys span
    3 monomials, so this is the rank-deficient min-norm branch, which only
    the unrounded design defines -- see gen_fit_exact.py)."""
    import sys
    sys.path.insert(0, str(GOLDEN.parent / "gen"))
    from fractions import Fraction

    from gen_fit_exact import exact_min_norm_rational
    for kid in ("matmul_tiled_g16x16", "conv_g16x16", "transpose_tile_g16x16"):
        prog = kc.load_program(kid)
        oprog = ko.Program((PROGRAMS / f"{kid}.kcp").read_text())
        rng = np.random.default_rng(5)
        n = 1500
        bs = [{p: int(16 * rng.integers(1, 400)) for p in prog.params} for _ in range(n)]
        sim = ko.simdev_reference_alpha()
        cnt = [oprog.evaluate_properties(b) for b in bs]
        T = np.array([ko.noiseless_time(sim, c) for c in cnt]) * np.exp(0.05 * rng.standard_normal(n))
        X, cov = ko.build_design_matrix(list(zip(cnt, T)))
        cols = [k for k in prog.props]
        exa, rank = exact_min_norm_rational([[Fraction(c.get(k, 0)) / Fraction(float(t)) for k in cols]
                                             for c, t in zip(cnt, T)])
        dev = _cols(prog, bs)
        Td = torch.tensor(T, dtype=torch.float64, device="cuda")
        alpha, rk, obj, st = kc.fit_fused(prog, dev, Td)
        err = fit_errors(alpha, [float(a) for a in exa], np.abs(X[:, cols]).max(axis=0))
        assert max(err) <= 1.0, (kid, rank, err)


_OPT_IN_CHECK = r"""
import sys
import numpy as np, torch
import paper_1604_04997_b200 as kc
rng = np.random.default_rng(7)
for F in (int(f) for f in sys.argv[1].split(",")):
    for N in (47, 4813, 100_003):
        X = torch.tensor(rng.uniform(0.5, 2.0, size=(N, F)) * 10.0 ** rng.integers(-2, 3, size=F), device="cuda")
        st = kc.gram_accumulate(X)
        torch.testing.assert_close(st.G, X.T @ X, rtol=1e-12, atol=0, msg=f"F={F} N={N}")
        torch.testing.assert_close(st.xt1, X.sum(0), rtol=1e-12, atol=0)
        assert torch.equal(st.colmax, X.abs().max(0).values), F
print("ok")
"""


@pytest.mark.parametrize("env,widths", [
    # DMMA off-diagonal + DFMA diagonal blocks for every even F in 26..40
    ({"KCG_GRAM_HYBRID": "1"}, "26,28,32,34,40"),
    # the row-per-lane DFMA Gram at the widths where it is not the default
    ({"KCG_GRAM_DFMA": "2"}, "7,12,13,20,21,22"),
])
def test_gram_opt_in_kernels_match_torch(env, widths):
    """The opt-in Gram kernels against torch fp64, tails included. In a
    subprocess: the switches are read once per process."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    r = subprocess.run([sys.executable, "-c", _OPT_IN_CHECK, widths], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=900, cwd=str(Path(__file__).resolve().parent.parent))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
