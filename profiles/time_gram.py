"""CUDA-event timing of the materialised Gram (config 3: 1e8 x 40 fp64 rows,
kcg_gram_accumulate) with a parity check against torch fp64 on a slice."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1604_04997_b200 as kc  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
out = {}
for F in [int(f) for f in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["40"])]:
    X = torch.rand((N, F), dtype=torch.float64, device="cuda").mul_(9999.0).add_(1.0)
    st = kc.GramStats.zeros(F, X.device)
    for _ in range(2):
        kc.gram_accumulate(X, st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        st = kc.GramStats.zeros(F, X.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        kc.gram_accumulate(X, st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = min(ts)
    Xs = X[:1_000_000]
    s2 = kc.gram_accumulate(Xs)
    ref = Xs.T @ Xs
    rel = float(((s2.G - ref).abs().max() / ref.abs().max()).item())
    out[F] = {"ms": t * 1e3, "GBps": 8.0 * F * N / t / 1e9, "TFLOPs": (N * F * (F + 1) + 2 * N * F) / t / 1e12,
              "rel_err": rel}
    del X
print(json.dumps(out))
