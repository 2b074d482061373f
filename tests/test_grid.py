"""Grid descriptors: lattices of bindings generated on the
device. kcg_grid_bindings must reproduce the lattice exactly and
kcg_eval_predict_grid must equal kcg_eval_predict over the materialised
columns bit for bit (predictions and statuses), including inadmissible
points, the int128 path, offsets into the lattice and ragged ends."""
import ctypes

import pytest

import kc_oracle as ko
from conftest import PROGRAMS

import paper_1604_04997_b200 as kc  # noqa: E402
from paper_1604_04997_b200 import _capi  # noqa: E402
from paper_1604_04997_b200.api import _KcgGrid  # noqa: E402


def _grid(np_, start, step, count):
    g = _KcgGrid()
    g.n_params = np_
    for j in range(np_):
        g.start[j], g.step[j], g.count[j] = start[j], step[j], count[j]
    return g


def test_grid_struct_layout_matches_header():
    assert ctypes.sizeof(_KcgGrid) == 8 + 3 * 8 * 8


@pytest.mark.parametrize("start,step,count,first,n", [
    ([0], [1], [0], 0, 0),                         # empty axis
    ([0], [1], [10], 5, 6),                        # beyond the end
    ([2**62], [2**62], [3], 0, 1),                 # values beyond int64
    ([0, 0], [1, 1], [2**40, 2**40], 0, 1),        # more than 2^64 points
])
def test_grid_validation_without_device(start, step, count, first, n):
    """Descriptor errors are E_INVALID_ARGUMENT, decided before any device
    work (so also on a host without a GPU)."""
    g = _grid(len(start), start, step, count)
    rc = _capi.lib().kcg_grid_bindings(ctypes.byref(g), first, n, None, None)
    assert rc == _capi.E_INVALID_ARGUMENT


def test_grid_eval_param_count_mismatch_is_rejected():
    prog = kc.load_program("matmul_tiled_g16x16")
    g = _grid(1, [16], [16], [10])
    a = (ctypes.c_double * 149)()
    rc = _capi.lib().kcg_eval_predict_grid(prog.handle, ctypes.byref(g), 0, 10, a, None, None, 0, None)
    assert rc == _capi.E_INVALID_ARGUMENT


@pytest.mark.gpu
def test_grid_bindings_match_lattice():
    torch = pytest.importorskip("torch")
    prog = kc.load_program("matmul_tiled_g16x16")
    grid = kc.Grid.for_program(prog, {"n": (336, 336, 17), "m": (16, 32, 1), "l": (-64, 16, 1001)})
    first, n = 123, grid.size - 123 - 7
    cols = kc.grid_bindings(grid, first, n)
    i = torch.arange(first, first + n, device="cuda")
    assert torch.equal(cols["l"], -64 + 16 * (i % 1001))
    assert torch.equal(cols["m"], 16 + 32 * ((i // 1001) % 1))
    assert torch.equal(cols["n"], 336 + 336 * (i // 1001))


@pytest.mark.gpu
@pytest.mark.parametrize("kid,axes", [
    ("matmul_tiled_g16x16", {"n": (336, 336, 40), "m": (336, 336, 41), "l": (8, 8, 43)}),  # half inadmissible
    ("matmul_skinny_g16x16", {"n": (16, 16 * 50_000, 30), "m": (128, 128 * 50_000, 30), "l": (16, 16, 7)}),
    ("conv_g16x16", {"n": (16, 16, 100_003)}),
    ("fd_stencil_g16x16", {"n": (-32, 16, 70_001)}),                                    # negative: inadmissible
    ("matmul_naive_g16x12", {"n": (48, 48, 31), "m": (12, 24, 33), "l": (48, 48, 35)}),
])
@pytest.mark.parametrize("first_frac,tail", [(0, 0), (0.37, 3)])
def test_eval_predict_grid_equals_materialised(kid, axes, first_frac, tail, suite_alpha):
    torch = pytest.importorskip("torch")
    prog = kc.load_program(kid)
    grid = kc.Grid.for_program(prog, axes)
    first = int(grid.size * first_frac)
    n = grid.size - first - tail
    w = kc.ModelWeights(device="t", alpha=list(suite_alpha), covered=[a != 0 for a in suite_alpha])
    pg, sg = kc.predict_grid(w, prog, grid, first, n, with_status=True)
    cols = kc.grid_bindings(grid, first, n)
    pm, sm = kc.predict(w, prog, cols, with_status=True)
    torch.cuda.synchronize()
    assert torch.equal(sg, sm)
    assert bool(((pg == pm) | (torch.isnan(pg) & torch.isnan(pm))).all())
    assert int((sg == 0).sum()) > 0
    # spot check against the oracle
    oprog = ko.Program((PROGRAMS / f"{kid}.kcp").read_text())
    for i in range(0, n, max(1, n // 23)):
        b = {p: int(cols[p][i]) for p in prog.params}
        try:
            want = ko.predict(suite_alpha, oprog.evaluate_properties(b))
            assert int(sg[i]) == 0 and float(pg[i]) == want
        except ko.AssumptionViolated:
            assert int(sg[i]) == 1


@pytest.mark.gpu
def test_noiseless_time_grid_matches_materialised():
    torch = pytest.importorskip("torch")
    prog = kc.load_program("nbody_g256")
    sim = ko.simdev_reference_alpha()
    grid = kc.Grid.for_program(prog, {"n": (256, 256, 200_000)})
    w = kc.ModelWeights(device="simdev-v1", alpha=sim, covered=[a != 0 for a in sim])
    t = kc.predict_grid(w, prog, grid, simulate=True)
    want = kc.noiseless_time(sim, prog, kc.grid_bindings(grid))
    torch.cuda.synchronize()
    assert torch.equal(t, want)


def test_columns_file_round_trip(tmp_path):
    """kcg-columns v1: write SoA columns, map them back bit-exactly; header
    layout (magic, 4096-aligned data) and error handling."""
    import numpy as np
    rng = np.random.default_rng(3)
    n = 100_003
    cols = {"n": rng.integers(-2**62, 2**62, n, dtype=np.int64),
            "time_s": rng.random(n),
            "status": rng.integers(0, 5, n, dtype=np.uint8),
            "best": rng.integers(-1, 6, n, dtype=np.int32)}
    path = tmp_path / "grid.kcgcol"
    kc.write_columns(path, cols)
    raw = path.read_bytes()
    assert raw[:8] == b"KCGCOL01"
    c = kc.read_columns(path)
    assert c.n_rows == n and c.names == list(cols)
    for k, v in cols.items():
        got = c.numpy(k)
        assert got.dtype == v.dtype and np.array_equal(got, v)
    c.close()
    bad = tmp_path / "bad.kcgcol"
    bad.write_bytes(b"KCGCOL02" + raw[8:4096])
    with pytest.raises(kc.KcgError) as e:
        kc.read_columns(bad)
    assert e.value.code == _capi.E_PARSE
    with pytest.raises(kc.KcgError):
        kc.write_columns(tmp_path / "x.kcgcol", {"x" * 40: np.zeros(3, np.int64)})


@pytest.mark.gpu
def test_columns_file_to_device_predict_and_back(tmp_path, suite_alpha):
    """Bindings grid -> columns file -> device -> predict -> columns file:
    the predictions round trip bitwise and equal the grid-descriptor path."""
    torch = pytest.importorskip("torch")
    prog = kc.load_program("matmul_tiled_g16x16")
    grid = kc.Grid.for_program(prog, {"n": (16, 16, 50), "m": (16, 48, 60), "l": (8, 8, 70)})
    cols = kc.grid_bindings(grid)
    path = tmp_path / "bindings.kcgcol"
    kc.write_columns(path, cols)
    c = kc.read_columns(path)
    dev = {p: c.to_device(p) for p in prog.params}
    part = c.to_device("l", 1000, 777)
    w = kc.ModelWeights(device="t", alpha=list(suite_alpha), covered=[a != 0 for a in suite_alpha])
    pred, st = kc.predict(w, prog, dev, with_status=True)
    pg = kc.predict_grid(w, prog, grid)
    torch.cuda.synchronize()
    assert torch.equal(part, cols["l"][1000:1777])
    assert all(torch.equal(dev[p], cols[p]) for p in prog.params)
    assert bool(((pred == pg) | (torch.isnan(pred) & torch.isnan(pg))).all())
    out = tmp_path / "pred.kcgcol"
    kc.write_columns(out, {"pred": pred, "status": st})
    r = kc.read_columns(out)
    # bitwise (NaN payloads included)
    assert torch.equal(torch.from_numpy(r.numpy("pred").copy()).view(torch.int64), pred.cpu().view(torch.int64))
    assert torch.equal(torch.from_numpy(r.numpy("status").copy()), st.cpu())
