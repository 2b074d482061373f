"""CUDA-event timing of the fused config-4 argmin (6 matmul variants over
(n,m,l) = 336*(u,v,w), u,v,w <= side). Knobs: KCG_ARGMIN_CTAS,
KCG_ARGMIN_NO_TMA, KCG_TMA_RING_KB."""
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import kc_oracle as ko  # noqa: E402
import paper_1604_04997_b200 as kc  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 551
alpha = ko.simdev_reference_alpha()
w = kc.ModelWeights(alpha=alpha, covered=[a != 0 for a in alpha])
progs = [kc.load_program(v) for v in ("matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
                                      "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16")]
n = side ** 3
i = torch.arange(0, n, dtype=torch.int64, device="cuda")
cols = {"n": ((i // (side * side) + 1) * 336).contiguous(), "m": (((i // side) % side + 1) * 336).contiguous(),
        "l": ((i % side + 1) * 336).contiguous()}
del i
for _ in range(2):
    best, bt = kc.argmin(progs, w, cols)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    kc.argmin(progs, w, cols)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
knobs = {k: v for k, v in os.environ.items() if k.startswith("KCG_")}
print(json.dumps({"knobs": knobs, "ms": min(ts), "points_per_s": 6 * n / min(ts) * 1e3,
                  "hist": torch.bincount(best.to(torch.int64) + 1, minlength=7).tolist()}))
