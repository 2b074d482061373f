"""BASELINE config 2 pinned end to end: 1e6 points over the four test
kernels (skinny matmul (16u,128u,16u), conv 16u, fd_stencil 16u, nbody 256u;
u = 1..250000), every count and every prediction on the GPU against the
reference's own evaluate_properties + predict (props.cpp:259-271,
model.cpp:95-117) -- symbolic path for skinny / conv at all 250,000 points,
bound mode (enumeration, cap 2e7) for fd_stencil / nbody as far as the cap
admits (tests/golden/config2_hashes.json, tests/gen/gen_config2.py). Past
the cap, fd_stencil and nbody are checked against the GPU enumeration
oracle at log-spaced sizes up to n = 262144."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import kc_oracle as ko  # noqa: E402
import paper_1604_04997_b200 as kc  # noqa: E402

U = 250_000


def _bindings(kid, u):
    if kid == "matmul_skinny_g16x16":
        return {"n": 16 * u, "m": 128 * u, "l": 16 * u}
    if kid == "nbody_g256":
        return {"n": 256 * u}
    return {"n": 16 * u}


@pytest.mark.parametrize("kid", ["matmul_skinny_g16x16", "conv_g16x16", "fd_stencil_g16x16", "nbody_g256"])
def test_config2_every_point_equals_the_reference(kid):
    gold = load_golden("config2_hashes.json")
    g = gold["kernels"][kid]
    prog = kc.load_program(kid)
    assert list(prog.props) == g["keys"]
    u = torch.arange(1, U + 1, dtype=torch.int64, device="cuda")
    cols = {p: v.contiguous() for p, v in _bindings(kid, u).items()}
    alpha = ko.simdev_reference_alpha()
    w = kc.ModelWeights(alpha=alpha, covered=[a != 0 for a in alpha])
    bb = kc.evaluate_properties(prog, cols, wide=True)
    pred, st = kc.predict(w, prog, cols, with_status=True)
    torch.cuda.synchronize()
    assert int((st != 0).sum()) == 0 and int((bb.status != 0).sum()) == 0
    F = len(g["keys"])
    rec = torch.empty((U, 2 * F + 1), dtype=torch.int64, device="cuda")
    for j in range(F):
        rec[:, 2 * j] = bb.counts_lo[j]
        rec[:, 2 * j + 1] = bb.counts_hi[j]
    rec[:, 2 * F] = pred.view(torch.int64)
    rec = rec.cpu().numpy()
    n = g["points"]  # the reference's range: all of it (symbolic) or up to the enumeration cap (bound)
    assert n == (U if g["mode"] == "sym" else n) and n >= 10
    assert rec[0].tolist() == g["first_record"]
    B = gold["block"]
    for b, h in enumerate(g["hashes"]):
        blk = np.ascontiguousarray(rec[b * B:min(n, (b + 1) * B)])
        assert hashlib.sha256(blk.tobytes()).hexdigest() == h, (kid, b)
    if kid == "matmul_skinny_g16x16":  # counts past 2^64 (int128 path) are among them
        assert int((bb.counts_hi != 0).sum()) > 0


@pytest.mark.parametrize("kid,n", [("fd_stencil_g16x16", 16384), ("fd_stencil_g16x16", 65536),
                                   ("fd_stencil_g16x16", 262144), ("nbody_g256", 32768),
                                   ("nbody_g256", 131072), ("nbody_g256", 262144)])
def test_config2_fd_nbody_beyond_the_cap_equal_enumeration(kid, n):
    """Past the reference's cap the derived fd_stencil / nbody programs are
    compared with the GPU brute-force enumeration (enumerate_points
    semantics, bit-exact against the reference on its goldens) at
    log-spaced config-2 sizes."""
    counts, points = kc.load_enum_program(kid).enumerate_points({"n": n})
    prog = kc.load_program(kid)
    bb = kc.evaluate_properties(prog, {"n": torch.tensor([n], dtype=torch.int64, device="cuda")}, wide=True)
    torch.cuda.synchronize()
    keys = kc.schema_keys()
    sym = {keys[k]: bb.counts_int(j, 0) for j, k in enumerate(prog.props) if bb.counts_int(j, 0)}
    assert points > 0 and counts == sym
