"""compute-sanitizer target (memcheck / racecheck / synccheck) for the round-2
kernels: the one-pass multi-variant evaluate+predict in its three launch
shapes (bulk-store TMA kernel with per-warp shared staging, 16-byte-store
TMA kernel, grid-stride kernel) with slow-path points, the argmin epilogue,
the fused refinement gradient and the floordiv-over-domain enumeration.
  python tests/sanitize_multi.py"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import kc_oracle as ko  # noqa: E402
import paper_1604_04997_b200 as kc  # noqa: E402

alpha = ko.simdev_reference_alpha()
w = kc.ModelWeights(alpha=alpha, covered=[a != 0 for a in alpha])
V = ("matmul_tiled_g12x12", "matmul_tiled_g14x14", "matmul_tiled_g16x16",
     "matmul_naive_g16x12", "matmul_naive_g16x14", "matmul_naive_g16x16")
progs = [kc.load_program(v) for v in V]
import os  # noqa: E402

# even: bulk-store kernel (2 CTAs/SM); 6 tiles per CTA, so the TMA ring
# refills (memcheck / synccheck). KCG_SANITIZE_SMALL=1: one wave of tiles,
# for racecheck, which cannot see the fence-and-counter stage hand-back
# (profiles/racecheck_mbarrier_probe.cu)
n = 148 * 1024 * 2 * (1 if os.environ.get("KCG_SANITIZE_SMALL") == "1" else 6) + 2
u = torch.randint(1, 400, (3, n), device="cuda")
cols = {p: (u[j] * 336).contiguous() for j, p in enumerate(("n", "m", "l"))}
cols["m"][::97] += 5
cols["n"][7::5003] = 336 * 10 ** 5
cols["n"][::4099] = -336
for extra in (0, 1):  # even n -> _tmab, odd n -> _tma
    m = n - extra
    sub = {k: v[:m] for k, v in cols.items()}
    pred, st = kc.predict_multi(progs, w, sub, status=True)
    pred2 = kc.predict_multi(progs, w, sub)
    ref = kc.predict(w, progs[2], sub)
    torch.cuda.synchronize()
    assert torch.equal(pred[2].view(torch.int64), ref.view(torch.int64))
    assert torch.equal(pred2.view(torch.int64), pred.view(torch.int64))
small = {k: v[:5000] for k, v in cols.items()}
kc.predict_multi(progs, w, small)
best, bt, preds = kc.argmin(progs, w, cols, return_preds=True)
prog = progs[2]
T = kc.noiseless_time(alpha, prog, {k: (u[j] * 16)[:2000000].contiguous() for j, k in enumerate(("n", "m", "l"))})
c16 = {k: (u[j] * 16)[:2000000].contiguous() for j, k in enumerate(("n", "m", "l"))}
a, rank, obj, stt = kc.fit_fused(prog, c16, T, refine=1)
ep = kc.EnumProgram("""kernelcost-enum v1
kernel x_fd
param n
assume n >= 1
array a global 32 1 0
group (n)//2
stmt assign
var g0 0 | (n)//2
var i 0 | n
var j (i)//3 | (i + 1)//2 + 1
access a load 1 | i + j
op flop.f32.addsub 1
endstmt
end
""")
ep.enumerate_points({"n": 64})
torch.cuda.synchronize()
print("multi ok")
