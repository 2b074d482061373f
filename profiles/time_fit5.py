"""CUDA-event timing of the config-5 fit passes on one GPU: fused Gram,
refinement gradient (kcg_rgrad_<k>), fused residual, over `side`^3 rows of
matmul_tiled_g16x16 at (n,m,l) = 16 (u,v,w), T = noiseless_time."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import kc_oracle as ko  # noqa: E402
import paper_1604_04997_b200 as kc  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
alpha = ko.simdev_reference_alpha()
prog = kc.load_program("matmul_tiled_g16x16")
rows = side ** 3
i = torch.arange(0, rows, dtype=torch.int64, device="cuda")
cols = {"n": ((i // (side * side) + 1) * 16).contiguous(), "m": (((i // side) % side + 1) * 16).contiguous(),
        "l": ((i % side + 1) * 16).contiguous()}
del i
T = kc.noiseless_time(alpha, prog, cols)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


st = kc.gram_fused(prog, cols, T)
a, _ = kc.solve_gram(st)
full = [0.0] * kc.schema_size()
for j, k in enumerate(prog.props):
    full[k] = a[j]
out = {"rows": rows,
       "gram_ms": timed(lambda: kc.gram_fused(prog, cols, T)),
       "rgrad_ms": timed(lambda: kc.residual_grad_fused(prog, cols, T, full)),
       "resid_ms": timed(lambda: kc.residual_fused(prog, cols, T, full))}
print(json.dumps(out))
