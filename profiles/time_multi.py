"""CUDA-event timing of the one-pass multi-variant evaluate+predict
(kcg_eval_predict_multi) on the config-4 lattice (6 matmul variants over
(n,m,l) = 336*(u,v,w), u,v,w <= side) against six kcg_eval_predict
launches. Knobs: KCG_MULTI_CTAS, KCG_MULTI_RING_KB, KCG_MULTI_TILE_Q."""
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
# rows padded to a 16-byte multiple (as bench.py): every output row aligned
out = torch.empty((6, (n + 1) // 2 * 2), dtype=torch.float64, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


def per_program():
    for v, p in enumerate(progs):
        arr, nn, _ = kc.api._columns(p, cols)
        kc.api.check(kc.api.lib().kcg_eval_predict(p.handle, arr, nn, w.alpha_array(), out[v].data_ptr(), None,
                                                   None, None, 0, torch.cuda.current_stream().cuda_stream))


ref = out.clone()
per_program()
ref.copy_(out)
t_multi = timed(lambda: kc.predict_multi(progs, w, cols, out=out))
same = bool(torch.equal(out[:, :n].view(torch.int64), ref[:, :n].view(torch.int64)))
t_sep = timed(per_program) if "--sep" in sys.argv else None
knobs = {k: v for k, v in os.environ.items() if k.startswith("KCG_")}
uniq = n * (24 + 48)
print(json.dumps({"knobs": knobs, "ms_multi": t_multi, "points_per_s": 6 * n / t_multi * 1e3,
                  "unique_GBps": uniq / t_multi / 1e6, "bitwise_equal_to_per_program": same,
                  "ms_per_program_x6": t_sep}))
if "--stream" in sys.argv:
    print(json.dumps({"stream_GBps": {f"{r}r{w}w": kc.measure_stream(r, w, 1 << 27) / 1e9
                                      for r, w in ((3, 6), (3, 1), (1, 6), (1, 1))}}))
