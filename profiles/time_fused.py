"""CUDA-event timing of the fused Gram and residual kernels over N rows of
config-5 shape (matmul_tiled_g16x16 bindings + noiseless T); prints GB/s
against the algorithmic 32 B/row. Tuning knobs come from the environment
(KCG_FUSED_RING_KB, ...)."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import kc_oracle as ko  # noqa: E402
import paper_1604_04997_b200 as kc  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
alpha = ko.simdev_reference_alpha()
g = torch.arange(0, N, dtype=torch.int64, device="cuda")
cols = {"n": (16 * (g // 1_000_000 % 1000 + 1)).contiguous(), "m": (16 * (g // 1000 % 1000 + 1)).contiguous(),
        "l": (16 * (g % 1000 + 1)).contiguous()}
del g
prog = kc.load_program("matmul_tiled_g16x16")
T = kc.noiseless_time(alpha, prog, cols)
out = {}
for name, fn in (("gram", lambda: kc.gram_fused(prog, cols, T)),
                 ("resid", lambda: kc.residual_fused(prog, cols, T, alpha))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = min(ts)
    out[name] = {"ms": t * 1e3, "GBps": 32.0 * N / t / 1e9}
print(json.dumps(out))
