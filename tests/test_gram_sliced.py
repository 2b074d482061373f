"""The integer-sliced Gram on the int8 tensor cores (gram_sliced.cu, C ABI
kcg_gram_accumulate_sliced): G within 1e-13 of sum_r |x_ri||x_rj| of torch's
fp64 product, X^T 1 within 1e-13 of sum |x|, exact column maxima -- on
tails, segment breaks (rising magnitudes), zero / signed / 1e+-140 columns,
accumulation over calls, NaN from a non-finite input, and the argument
checks (model.cpp:37-60 is the reference step either back end replaces)."""
import pytest

import paper_1604_04997_b200 as kc
from paper_1604_04997_b200._capi import KcgError

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _errors(X, st):
    A = X.abs()
    eg = float(((st.G - X.T @ X).abs() / (A.T @ A).clamp_min(1e-300)).max())
    ex = float(((st.xt1 - X.sum(0)).abs() / A.sum(0).clamp_min(1e-300)).max())
    return eg, ex, bool(torch.equal(st.colmax, A.max(0).values))


@pytest.mark.parametrize("F", [17, 24, 30, 32, 36, 40])
@pytest.mark.parametrize("n", [1, 127, 129, 128 * 148 * 2 + 77, 128 * 148 * 260 + 5])
def test_sliced_gram_uniform(F, n):
    g = torch.Generator(device="cuda").manual_seed(F * 1000 + n % 997)
    X = torch.rand((n, F), dtype=torch.float64, device="cuda", generator=g).mul_(9999.0).add_(1.0)
    eg, ex, cm = _errors(X, kc.gram_accumulate(X, sliced=True))
    assert eg < 1e-13 and ex < 1e-13 and cm


def test_sliced_gram_awkward_columns():
    g = torch.Generator(device="cuda").manual_seed(11)
    n = 128 * 148 * 300 + 33
    X = torch.randn((n, 40), dtype=torch.float64, device="cuda", generator=g)
    X[:, 3] = 0.0                                                            # zero column
    X[:, 5] *= torch.logspace(-30, 30, n, dtype=torch.float64, device="cuda")  # rising: segment breaks
    X[:, 7] *= torch.exp2(torch.randint(-40, 40, (n,), device="cuda", generator=g).double())
    X[:, 11] = -X[:, 11].abs() * 1e140
    X[:, 12] *= 1e-140
    eg, ex, cm = _errors(X, kc.gram_accumulate(X, sliced=True))
    assert eg < 1e-13 and ex < 1e-13 and cm


def test_sliced_gram_accumulates_and_propagates_nan():
    g = torch.Generator(device="cuda").manual_seed(12)
    X = torch.rand((200_000, 40), dtype=torch.float64, device="cuda", generator=g)
    st = kc.gram_accumulate(X[:100_000], sliced=True)
    kc.gram_accumulate(X[100_000:], st, sliced=True)
    eg, ex, cm = _errors(X, st)
    assert eg < 1e-13 and ex < 1e-13 and cm
    X[1234, 6] = float("inf")
    assert not torch.isfinite(kc.gram_accumulate(X, sliced=True).G).all()


def test_sliced_gram_rejects_unsupported_shapes():
    X = torch.rand((1000, 41), dtype=torch.float64, device="cuda")
    with pytest.raises(KcgError):
        kc.gram_accumulate(X, sliced=True)
    with pytest.raises(KcgError):
        kc.gram_accumulate(X[:, :40], sliced=True)  # ld != n_cols
