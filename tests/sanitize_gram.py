"""compute-sanitizer target: the row-split DMMA Gram at the 1-CTA widths and the per-width kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1604_04997_b200 as kc  # noqa: E402

for F in (41, 64, 72, 80):
    X = torch.rand((3000, F), dtype=torch.float64, device="cuda")
    st = kc.gram_accumulate(X); torch.cuda.synchronize()
    assert torch.allclose(st.G, X.T @ X, rtol=1e-12, atol=0)
print("gram ok")
