"""The objective after a refinement step from the refinement pass itself
(api.refined_objective: |r - X d|^2 = r2 - 2 d.g + d^T G d with r2 and g
from kcg_residual_grad_obj_fused at the pre-step weights, G the fused Gram)
against the fused residual pass run at the refined weights -- the sum
model.cpp:81-92 forms. Noisy times (objective O(n sigma^2)) and noiseless
ones (objective at rounding level, where the direct pass is itself noise);
also through fit_fused / fit_sharded, which now take it."""
import numpy as np
import pytest

import paper_1604_04997_b200 as kc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _rows(kid, n, sigma, seed):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    import kc_oracle as ko
    prog = kc.load_program(kid)
    g = torch.Generator(device="cuda").manual_seed(seed)
    cols = {p: (16 * torch.randint(1, 600, (n,), device="cuda", generator=g)).contiguous() for p in prog.params}
    T = kc.noiseless_time(ko.simdev_reference_alpha(), prog, cols)
    if sigma:
        T = T * torch.exp(sigma * torch.randn(n, dtype=torch.float64, device="cuda", generator=g))
    return prog, cols, T.contiguous()


def _full(prog, a):
    out = [0.0] * kc.schema_size()
    for j, k in enumerate(prog.props):
        out[k] = a[j]
    return out


@pytest.mark.parametrize("kid", ["matmul_tiled_g16x16", "conv_g16x16", "transpose_tile_g16x16"])
@pytest.mark.parametrize("sigma", [0.05, 0.0])
def test_refined_objective_equals_the_residual_pass(kid, sigma):
    prog, cols, T = _rows(kid, 2_000_003, sigma, 3)
    st = kc.gram_fused(prog, cols, T)
    a, _ = kc.solve_gram(st)
    r2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    g = kc.residual_grad_fused(prog, cols, T, _full(prog, a), r2=r2)
    # r2 alone is the objective at the pre-step weights
    direct0 = kc.residual_fused(prog, cols, T, _full(prog, a))
    a2 = kc.refine_gram(st, a, g)
    obj = kc.refined_objective(st, a, a2, g, r2)
    direct = kc.residual_fused(prog, cols, T, _full(prog, a2))
    if sigma:
        assert float(r2.item()) == pytest.approx(direct0, rel=1e-9)
        assert obj == pytest.approx(direct, rel=1e-9)
    else:
        # rounding level: the direct pass (plain fp64 residuals) is itself
        # noise here; the refined objective stays at that level and >= 0
        tiny = 1e-28 * T.numel()
        assert -tiny <= obj <= 4.0 * max(direct, float(r2.item())) + tiny


def test_fit_fused_objective_matches_a_residual_pass():
    prog, cols, T = _rows("matmul_tiled_g16x16", 1_000_003, 0.05, 9)
    for refine in (1, 2):
        alpha, rk, obj, st = kc.fit_fused(prog, cols, T, refine=refine)
        assert obj == pytest.approx(kc.residual_fused(prog, cols, T, _full(prog, alpha)), rel=1e-9)
    alpha, rk, obj0, st = kc.fit_fused(prog, cols, T, refine=0)
    assert obj0 == pytest.approx(kc.residual_fused(prog, cols, T, _full(prog, alpha)), rel=1e-12)


def test_r2_argument_checked():
    prog, cols, T = _rows("matmul_tiled_g16x16", 1000, 0.05, 1)
    with pytest.raises(kc.KcgError):
        kc.residual_grad_fused(prog, cols, T, [0.0] * kc.schema_size(), r2=torch.zeros(1))
