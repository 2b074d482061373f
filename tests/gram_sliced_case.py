"""Subprocess body of tests/test_gram_sliced.py: the integer-sliced tcgen05
Gram (gram_sliced.cu, KCG_GRAM_SLICED=1 -- read once per process) against
torch fp64 on awkward inputs. Exit status 0 = every case within bounds."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1604_04997_b200 as kc  # noqa: E402

dev = "cuda"


def compare(X):
    st = kc.gram_accumulate(X)
    A = X.abs()
    scale = (A.T @ A).clamp_min(1e-300)
    eg = float(((st.G - X.T @ X).abs() / scale).max())
    ex = float(((st.xt1 - X.sum(0)).abs() / A.sum(0).clamp_min(1e-300)).max())
    return eg, ex, bool(torch.equal(st.colmax, A.max(0).values))


g = torch.Generator(device=dev).manual_seed(11)
res = []
for F in [17, 24, 30, 32, 36, 40]:
    for n in [1, 127, 129, 128 * 148 * 2 + 77, 128 * 148 * 260 + 5]:  # tails; > one segment per CTA
        X = torch.rand((n, F), dtype=torch.float64, device=dev, generator=g).mul_(9999.0).add_(1.0)
        res.append((F, n, "uniform", *compare(X)))
n = 128 * 148 * 300 + 33
X = torch.randn((n, 40), dtype=torch.float64, device=dev, generator=g)
X[:, 3] = 0.0                                                    # zero column
X[:, 5] *= torch.logspace(-30, 30, n, dtype=torch.float64, device=dev)  # rising: segment breaks
X[:, 7] *= torch.exp2(torch.randint(-40, 40, (n,), device=dev, generator=g).double())
X[:, 11] = -X[:, 11].abs() * 1e140
X[:, 12] *= 1e-140
res.append((40, n, "signed / wide range / zero / rising", *compare(X)))
bad = [r for r in res if not (r[3] < 1e-13 and r[4] < 1e-13 and r[5])]
X = torch.rand((40_000, 40), dtype=torch.float64, device=dev, generator=g)
X[1234, 6] = float("inf")
nonfinite_ok = bool((~torch.isfinite(kc.gram_accumulate(X).G)).any())
print(json.dumps({"cases": len(res), "bad": bad, "nonfinite_propagates": nonfinite_ok,
                  "worst_G": max(r[3] for r in res), "worst_xt1": max(r[4] for r in res)}))
sys.exit(0 if not bad and nonfinite_ok else 1)
