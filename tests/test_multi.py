"""kcg_eval_predict_multi: every variant's evaluate_properties + predict
(props.cpp:259-271, model.cpp:95-117) over ONE binding stream in one pass.
Its predictions and status bytes must be bitwise those of one
kcg_eval_predict per program -- fast path, int128 path, inadmissible,
negative and overflowing points, ragged TMA tails, unaligned columns,
padded outputs -- and a sample is checked against the oracle directly."""
import ctypes

import numpy as np
import pytest

import kc_oracle as ko
from conftest import PROGRAMS
import paper_1604_04997_b200 as kc
from paper_1604_04997_b200 import _capi

MATMUL = ("matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
          "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16")
ONE_PARAM = ("conv_g16x16", "fd_stencil_g16x16", "nbody_g256", "matmul_skinny_g16x16")


def _weights(alpha=None):
    a = list(alpha) if alpha is not None else ko.simdev_reference_alpha()
    return kc.ModelWeights(alpha=a, covered=[x != 0 for x in a])


def test_multi_source_compiles_for_sm100a():
    """The generated one-pass kernels compile (NVRTC, sm_100a) without a GPU,
    for 3-parameter variants and for programs declaring parameters in
    another order."""
    progs = [kc.load_program(v) for v in MATMUL]
    for argmin, names in ((False, ("kcg_multi_v6", "kcg_multi_v6_tma_st")), (True, ("kcg_multiam_v6_tma", "kcg_multiam_v6_p"))):
        src = kc.multi_jit_source(progs, argmin=argmin)
        for name in names:
            assert name in src
            assert _capi.lib().kcg_jit_compile_check(src.encode(), name.encode()) == 0, _capi.lib().kcg_last_error()


def test_multi_argument_errors():
    p = kc.load_program("matmul_tiled_g16x16")
    q = kc.load_program("conv_g16x16")
    L = _capi.lib()
    h = (ctypes.c_void_p * 2)(p.handle.value, q.handle.value)
    w = _weights()
    out = (ctypes.c_double * 8)()
    assert L.kcg_eval_predict_multi(h, 0, None, 4, w.alpha_array(), out, 4, None, 0, None) == _capi.E_INVALID_ARGUMENT
    assert L.kcg_eval_predict_multi(h, 1, None, 4, None, out, 4, None, 0, None) == _capi.E_INVALID_ARGUMENT
    assert L.kcg_eval_predict_multi(h, 1, None, 4, w.alpha_array(), out, 3, None, 0, None) == _capi.E_INVALID_ARGUMENT
    with pytest.raises(kc.KcgError):  # parameter sets differ
        kc.multi_jit_source([p, q])


def _bindings(n, seed, scale=336):
    rng = np.random.default_rng(seed)
    b = {k: (rng.integers(1, 551, n) * scale).astype(np.int64) for k in "nml"}
    b["m"][::97] += 5           # inadmissible for every variant
    b["l"][::1013] = 0          # zero-sized (inadmissible: l >= G)
    b["n"][::4099] = -336       # negative
    b["n"][7::5003] = 336 * 10 ** 5          # past the int64-safe box: int128 counts
    b["m"][11::7001] = 336 * 10 ** 13        # past the int128 bound: OVERFLOW
    return b


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 1000, 3 * 4096 + 17, 148 * 3 * 1024 * 2 + 333, 148 * 3 * 1024 * 2 + 334])
def test_multi_bitwise_equals_per_program(n):
    """odd n: the 16-byte-store TMA kernel; even n (rows 16-byte aligned):
    the bulk-store kernel (kcg_multi_v6_tmab)"""
    import torch
    progs = [kc.load_program(v) for v in MATMUL]
    w = _weights()
    dev = {k: torch.from_numpy(v).cuda() for k, v in _bindings(n, n).items()}
    pred, st = kc.predict_multi(progs, w, dev, status=True)
    for i, p in enumerate(progs):
        want, wst = kc.predict(w, p, dev, with_status=True)
        assert torch.equal(pred[i].view(torch.int64), want.view(torch.int64)), (MATMUL[i], n)
        assert torch.equal(st[i], wst), (MATMUL[i], n)
    if n > 10000:
        for code in (0, 1, 3):
            assert int((st == code).sum()) > 0, code


@pytest.mark.gpu
def test_multi_against_oracle_sample():
    import torch
    progs = [kc.load_program(v) for v in MATMUL]
    oprogs = [ko.Program((PROGRAMS / f"{v}.kcp").read_text()) for v in MATMUL]
    alpha = ko.simdev_reference_alpha()
    b = _bindings(4000, 5)
    dev = {k: torch.from_numpy(v).cuda() for k, v in b.items()}
    pred, st = kc.predict_multi(progs, _weights(alpha), dev, status=True)
    pred, st = pred.cpu(), st.cpu()
    for i in range(0, 4000, 37):
        bi = {k: int(b[k][i]) for k in "nml"}
        for v, op in enumerate(oprogs):
            if not op.admits(bi):
                assert int(st[v, i]) == 1 and pred[v, i] != pred[v, i]
                continue
            if int(st[v, i]) == 3:  # beyond the 128-bit bound (documented divergence)
                continue
            want = ko.predict(alpha, op.evaluate_properties(bi))
            assert int(st[v, i]) == 0 and float(pred[v, i]) == want, (MATMUL[v], bi)


@pytest.mark.gpu
def test_multi_unaligned_columns_padded_output_and_pred_only():
    import torch
    progs = [kc.load_program(v) for v in MATMUL[:4]]
    w = _weights()
    n = 148 * 3 * 1024 + 999
    b = _bindings(n + 1, 9)
    base = {k: torch.from_numpy(v).cuda() for k, v in b.items()}
    dev = {k: v[1:] for k, v in base.items()}  # 8-byte aligned only: grid-stride kernel
    out = torch.full((len(progs), n + 64), 7.0, dtype=torch.float64, device="cuda")
    kc.predict_multi(progs, w, dev, out=out)
    for i, p in enumerate(progs):
        want = kc.predict(w, p, {k: v.contiguous() for k, v in dev.items()})
        assert torch.equal(out[i, :n].view(torch.int64), want.view(torch.int64))
        assert bool((out[i, n:] == 7.0).all())


@pytest.mark.gpu
def test_multi_one_parameter_programs_and_int128():
    """conv / fd_stencil / nbody / skinny matmul share the parameter n only
    when skinny is bound through its own columns -- so: the three one-
    parameter programs together, up to sizes with int128 counts."""
    import torch
    names = ONE_PARAM[:3]
    progs = [kc.load_program(v) for v in names]
    w = _weights()
    u = np.arange(1, 300001, dtype=np.int64)
    n_col = np.concatenate([16 * u, 256 * u[:1000] * 10 ** 9, [-16, 0, 17]]).astype(np.int64)
    dev = {"n": torch.from_numpy(n_col).cuda()}
    pred, st = kc.predict_multi(progs, w, dev, status=True)
    for i, p in enumerate(progs):
        want, wst = kc.predict(w, p, dev, with_status=True)
        assert torch.equal(pred[i].view(torch.int64), want.view(torch.int64)), names[i]
        assert torch.equal(st[i], wst), names[i]


@pytest.mark.gpu
def test_multi_nonfinite_weights_take_per_program_path():
    import torch
    alpha = ko.simdev_reference_alpha()
    alpha[ko.SCHEMA_INDEX["launch.const"]] = float("inf")
    w = _weights(alpha)
    progs = [kc.load_program(v) for v in MATMUL]
    dev = {k: torch.from_numpy(v).cuda() for k, v in _bindings(5000, 3).items()}
    pred = kc.predict_multi(progs, w, dev)
    for i, p in enumerate(progs):
        want = kc.predict(w, p, dev)
        assert torch.equal(pred[i].view(torch.int64), want.view(torch.int64))


def _argmin_ref(torch, preds, st):
    """lowest index among status-OK variants with the smallest prediction"""
    V, n = preds.shape
    big = torch.where(st == 0, preds, torch.full_like(preds, float("inf")))
    bt, _ = big.min(dim=0)
    first = torch.full((n,), -1, dtype=torch.int64, device=preds.device)
    for v in range(V - 1, -1, -1):
        hit = (st[v] == 0) & (preds[v] == bt)
        first = torch.where(hit, torch.full_like(first, v), first)
    return first, bt


@pytest.mark.gpu
@pytest.mark.parametrize("n", [777, 148 * 1024 * 3 + 4321])
def test_argmin_one_pass_equals_per_program_argmin(n):
    """kcg_argmin through the one-pass kernel (argmin epilogue): best variant,
    best time and every prediction equal the per-program predictions'
    lowest-index argmin, on the TMA path and the grid-stride path, with
    slow-path points (int128 counts, overflow, inadmissible, negative)."""
    import torch
    progs = [kc.load_program(v) for v in MATMUL]
    w = _weights()
    dev = {k: torch.from_numpy(v).cuda() for k, v in _bindings(n, n + 1).items()}
    best, bt, preds = kc.argmin(progs, w, dev, return_preds=True)
    best2, bt2 = kc.argmin(progs, w, dev)
    ref = [kc.predict(w, p, dev, with_status=True) for p in progs]
    P = torch.stack([r[0] for r in ref])
    S = torch.stack([r[1] for r in ref])
    assert torch.equal(preds.view(torch.int64), P.view(torch.int64))
    rb, rt = _argmin_ref(torch, P, S)
    assert torch.equal(best.to(torch.int64), rb) and torch.equal(best2.to(torch.int64), rb)
    assert torch.equal(bt.view(torch.int64), rt.view(torch.int64)) and torch.equal(bt2.view(torch.int64), rt.view(torch.int64))
    assert int((rb == -1).sum()) > 0 and int((rb >= 0).sum()) > 0


@pytest.mark.gpu
def test_argmin_ties_go_to_the_lowest_index():
    import torch
    p = kc.load_program("matmul_tiled_g16x16")
    q = kc.load_program("matmul_naive_g16x16")
    w = _weights()
    n = 148 * 1024 * 2
    dev = {k: torch.from_numpy(v).cuda() for k, v in _bindings(n, 2, scale=16).items()}
    best, bt = kc.argmin([q, p, p, q], w, dev)
    want = kc.predict(w, p, dev)
    wq = kc.predict(w, q, dev)
    ok = ~torch.isnan(want)
    exp = torch.where(wq <= want, torch.zeros_like(best), torch.ones_like(best))
    assert torch.equal(best[ok & (wq == wq)], exp[ok & (wq == wq)].to(best.dtype))


@pytest.mark.gpu
def test_multi_random_program_sets_bitwise_equal_per_program():
    """Fuzz: random programs (tests/fuzz_programs.py: floordiv / min / max
    atoms, rational and power-of-two coefficients, congruences) grouped by
    parameter set, up to six per launch, over random bindings incl. int128,
    overflowing and negative ones -- one pass == one kcg_eval_predict per
    program, predictions bitwise and status bytes equal. 36 seeds by default
    (NVRTC compiles dominate: ~1.5 min); round 2 ran 120 seeds clean
    (KCG_MULTI_FUZZ_SEEDS=120, 6 min)."""
    import os

    import torch
    from fuzz_programs import random_bindings, random_program
    alpha = [a if a != 0 else 1e-12 * (1 + i % 7) for i, a in enumerate(ko.simdev_reference_alpha())]
    w = _weights(alpha)
    groups = {}
    for seed in range(int(os.environ.get("KCG_MULTI_FUZZ_SEEDS", "36"))):
        p = kc.Program(random_program(seed))
        groups.setdefault(tuple(p.params), []).append((seed, p))
    checked = 0
    for params, members in groups.items():
        for c0 in range(0, len(members), 6):
            chunk = members[c0:c0 + 6]
            progs = [p for _, p in chunk]
            bs = random_bindings(chunk[0][0], list(params), 3000)
            cols = {q: torch.tensor([b[q] for b in bs], dtype=torch.int64, device="cuda") for q in params}
            pred, st = kc.predict_multi(progs, w, cols, status=True)
            for i, p in enumerate(progs):
                want, wst = kc.predict(w, p, cols, with_status=True)
                assert torch.equal(st[i], wst), (chunk[i][0],)
                assert torch.equal(pred[i].view(torch.int64), want.view(torch.int64)), (chunk[i][0],)
            checked += len(progs)
    assert checked >= 30
