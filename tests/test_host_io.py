"""kcg_eval_predict_host: the reference's calling convention (HOST bindings
in, HOST predictions out; predict, model.cpp:95-117) over the chunked
H2D / kernel / D2H pipeline. Results must be bitwise those of the
device-resident kcg_eval_predict, for pinned and pageable buffers, ragged
chunk tails, inadmissible points and several programs sharing one binding
stream."""
import ctypes

import numpy as np
import pytest

import kc_oracle as ko
import paper_1604_04997_b200 as kc  # noqa: E402
from paper_1604_04997_b200 import _capi  # noqa: E402

VARIANTS = ("matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
            "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16")


def _weights():
    a = ko.simdev_reference_alpha()
    return kc.ModelWeights(alpha=a, covered=[x != 0 for x in a])


def test_host_eval_argument_errors():
    p = kc.load_program("matmul_tiled_g16x16")
    h = (ctypes.c_void_p * 1)(p.handle.value)
    out = (ctypes.c_double * 4)()
    L = _capi.lib()
    assert L.kcg_eval_predict_host(h, 1, None, 4, None, out, None, 0) == _capi.E_INVALID_ARGUMENT  # no alpha
    assert L.kcg_eval_predict_host(h, 0, None, 4, None, out, None, 0) == _capi.E_INVALID_ARGUMENT
    w = _weights()
    assert L.kcg_eval_predict_host(h, 1, None, 4, w.alpha_array(), None, None, 0) == _capi.E_INVALID_ARGUMENT


def test_host_eval_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = kc.load_program("matmul_tiled_g16x16")
    with pytest.raises(kc.KcgError) as e:
        kc.predict_host([p], _weights(), {k: np.array([16, 32]) for k in "nml"})
    assert e.value.code == _capi.E_CUDA


def _bindings(n, seed):
    rng = np.random.default_rng(seed)
    b = {k: (rng.integers(1, 400, n) * 336).astype(np.int64) for k in "nml"}
    b["m"][::97] += 5      # inadmissible for every variant (m % 12/14/16 != 0)
    b["l"][::1013] = 0     # zero-sized
    return b


@pytest.mark.gpu
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("chunk", [65536, 1 << 22])
def test_host_eval_bitwise_equals_device_path(monkeypatch, pinned, chunk):
    import torch
    monkeypatch.setenv("KCG_HOST_CHUNK", str(chunk))
    n = 3 * 65536 + 4321  # ragged last chunk
    progs = [kc.load_program(v) for v in VARIANTS]
    w = _weights()
    b = _bindings(n, 7)
    host = {k: torch.from_numpy(v) for k, v in b.items()}
    out = None
    if pinned:
        host = {k: v.pin_memory() for k, v in host.items()}
        out = torch.empty((len(progs), n), dtype=torch.float64).pin_memory()
    pred, st = kc.predict_host(progs, w, host, status=True, out=out)
    path = _capi.lib().kcg_host_last_path()
    assert bool(path & _capi.HOST_PINNED) == pinned
    assert path & _capi.HOST_PATH_ONEPASS  # several programs: one launch per chunk
    if pinned:
        assert st.is_pinned() and path & _capi.HOST_PATH_2D
    dev = {k: v.cuda() for k, v in host.items()}
    for i, p in enumerate(progs):
        want, wst = kc.predict(w, p, dev, with_status=True)
        assert torch.equal(pred[i].view(torch.int64), want.cpu().view(torch.int64)), p.name if hasattr(p, "name") else i
        assert torch.equal(st[i], wst.cpu())
    assert int((st != 0).sum()) > 0  # the inadmissible points are there


@pytest.mark.gpu
def test_host_eval_param_order_follows_first_program():
    """Programs whose parameters are declared in another order read the
    host columns by name (progs[0]'s order)."""
    import torch
    progs = [kc.load_program("matmul_tiled_g16x16"), kc.load_program("matmul_naive_g16x16")]
    w = _weights()
    b = _bindings(5000, 3)
    pred = kc.predict_host(progs, w, b)
    dev = {k: torch.from_numpy(v).cuda() for k, v in b.items()}
    for i, p in enumerate(progs):
        want = kc.predict(w, p, dev).cpu()
        assert torch.equal(pred[i].view(torch.int64), want.view(torch.int64))


@pytest.mark.gpu
def test_host_eval_int128_and_single_param_programs(monkeypatch):
    """Skinny matmul past the int64-safe box (int128 counts, > 2^53
    conversions) and a one-parameter program through the host pipeline,
    several chunks each: bitwise the device path."""
    import torch
    monkeypatch.setenv("KCG_HOST_CHUNK", "4096")
    w = _weights()
    u = np.arange(1, 20001, dtype=np.int64) * 97
    cases = [(kc.load_program("matmul_skinny_g16x16"), {"n": 16 * u, "m": 128 * u, "l": 16 * u}),
             (kc.load_program("conv_g16x16"), {"n": 16 * u})]
    for prog, b in cases:
        pred, st = kc.predict_host([prog], w, b, status=True)
        dev = {k: torch.from_numpy(v).cuda() for k, v in b.items()}
        want, wst = kc.predict(w, prog, dev, with_status=True)
        assert torch.equal(pred[0].view(torch.int64), want.cpu().view(torch.int64))
        assert torch.equal(st[0], wst.cpu())
        assert int((wst == 0).sum()) > 0


@pytest.mark.gpu
def test_host_eval_pitch_fallback_and_growing_streams(monkeypatch):
    """Pinned callers whose n * 8 exceeds the device's max pitch take one 1D
    D2H copy per program (forced here by lowering the limit); a later call
    with more internal streams and the same chunk bytes allocates the new
    slots' staging (pageable path). Both bitwise the device path."""
    import torch
    monkeypatch.setenv("KCG_HOST_CHUNK", "8192")
    n = 5 * 8192 + 77
    progs = [kc.load_program(v) for v in VARIANTS[:3]]
    w = _weights()
    b = _bindings(n, 11)
    dev = {k: torch.from_numpy(v).cuda() for k, v in b.items()}
    want = [kc.predict(w, p, dev).cpu() for p in progs]
    host = {k: torch.from_numpy(v).pin_memory() for k, v in b.items()}
    out = torch.empty((len(progs), n), dtype=torch.float64).pin_memory()
    monkeypatch.setenv("KCG_HOST_MAX_PITCH", str(8 * (n - 1)))
    kc.predict_host(progs, w, host, out=out)
    assert _capi.lib().kcg_host_last_path() & (_capi.HOST_PINNED | _capi.HOST_PATH_2D) == _capi.HOST_PINNED
    for i in range(len(progs)):
        assert torch.equal(out[i].view(torch.int64), want[i].view(torch.int64))
    monkeypatch.delenv("KCG_HOST_MAX_PITCH")
    for streams in ("1", "4", "2", "6"):
        monkeypatch.setenv("KCG_HOST_STREAMS", streams)
        pred = kc.predict_host(progs, w, b, pinned=False)
        for i in range(len(progs)):
            assert torch.equal(pred[i].view(torch.int64), want[i].view(torch.int64)), streams


@pytest.mark.gpu
def test_host_eval_onepass_equals_per_program_launches(monkeypatch):
    """The one-pass multi-program chunk kernel and one launch per program
    (KCG_HOST_ONEPASS=0) give the same bits, with status bytes."""
    monkeypatch.setenv("KCG_HOST_CHUNK", "32768")
    n = 4 * 32768 + 5
    progs = [kc.load_program(v) for v in VARIANTS]
    w = _weights()
    b = _bindings(n, 21)
    p1, s1 = kc.predict_host(progs, w, b, status=True)
    assert _capi.lib().kcg_host_last_path() & _capi.HOST_PATH_ONEPASS
    monkeypatch.setenv("KCG_HOST_ONEPASS", "0")
    p0, s0 = kc.predict_host(progs, w, b, status=True)
    assert not _capi.lib().kcg_host_last_path() & _capi.HOST_PATH_ONEPASS
    import torch
    assert torch.equal(p1.view(torch.int64), p0.view(torch.int64))
    assert torch.equal(s1, s0)
