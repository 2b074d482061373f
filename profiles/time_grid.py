"""CUDA-event timing of kcg_eval_predict_grid over the config-4 lattice
(6 matmul variants x (n,m,l) = 336*(u,v,w), u,v,w <= side)."""
import ctypes
import json
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
total = side ** 3
pred = torch.empty(total, dtype=torch.float64, device="cuda")
gs = [kc.Grid.for_program(p, {"n": (336, 336, side), "m": (336, 336, side), "l": (336, 336, side)}).c_struct()
      for p in progs]
stream = torch.cuda.current_stream().cuda_stream


def run():
    for p, g in zip(progs, gs):
        kc.api.check(kc.api.lib().kcg_eval_predict_grid(p.handle, ctypes.byref(g), 0, total, w.alpha_array(),
                                                        pred.data_ptr(), None, 0, stream))


for _ in range(2):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"ms": min(ts), "points_per_s": 6 * total / min(ts) * 1e3}))
