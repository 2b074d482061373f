"""compute-sanitizer target: the row-split DMMA Gram at the 1-CTA widths, the per-width kernel, the
row-per-lane DFMA Gram (F = 2, 9, 18), the DMMA + DFMA hybrid (F = 34, 40) and the integer-sliced
tcgen05 Gram (F = 17, 33, 40, several segments per CTA), with tails."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1604_04997_b200 as kc  # noqa: E402

# row counts large enough that every CTA's TMA ring refills its stages
# (memcheck / synccheck); KCG_SANITIZE_SMALL=1: one wave of tiles, for
# racecheck, which cannot see the fence-and-counter stage hand-back
# (profiles/racecheck_mbarrier_probe.cu)
import os  # noqa: E402

SMALL = os.environ.get("KCG_SANITIZE_SMALL") == "1"
for F, N in ((2, 3_000_017), (9, 1_000_003), (18, 500_009), (34, 300_007), (40, 300_007), (41, 300_007),
             (64, 300_007), (72, 300_007), (80, 300_007)):
    N = (3001 if F > 72 else 30011) if SMALL else N
    X = torch.rand((N, F), dtype=torch.float64, device="cuda")
    st = kc.gram_accumulate(X); torch.cuda.synchronize()
    assert torch.allclose(st.G, X.T @ X, rtol=1e-12, atol=0)
# the int8 tensor-core Gram: its operand ring refills and its segments break
# (rising magnitudes) at these sizes
for F, N in ((17, 128 * 148 * 8 + 77), (33, 128 * 148 * 8 + 5), (40, 128 * 148 * 12 + 99)):
    N = 128 * 148 + 9 if SMALL else N
    X = torch.rand((N, F), dtype=torch.float64, device="cuda")
    X[:, 1] *= torch.logspace(-10, 10, N, dtype=torch.float64, device="cuda")
    st = kc.gram_accumulate(X, sliced=True); torch.cuda.synchronize()
    assert torch.allclose(st.G, X.T @ X, rtol=1e-12, atol=0)
print("gram ok")
