"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): python tests/sanitize_smoke.py"""
import ctypes
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
n = 148 * 1024 + 129
u = torch.randint(1, 3000, (3, n), device="cuda")
prog = kc.load_program("matmul_tiled_g16x16")
cols = {p: (u[j] * 16).contiguous() for j, p in enumerate(prog.params)}
cols["n"][::7] += 1
for eng in ("jit", "interp"):
    prog.set_engine(eng)
    kc.predict(w, prog, cols, with_status=True)
    kc.evaluate_properties(prog, cols)
prog.set_engine("jit")
T = kc.noiseless_time(alpha, prog, cols)
T[::7] = 1.0
st = kc.gram_fused(prog, cols, T)
obj = torch.zeros(1, dtype=torch.float64, device="cuda")
arr = (ctypes.c_void_p * 3)(*[cols[p].data_ptr() for p in prog.params])
kc.api.check(kc.api.lib().kcg_residual_fused(prog.handle, arr, T.data_ptr(), n, (ctypes.c_double * 149)(*alpha),
                                             obj.data_ptr(), None))
progs = [kc.load_program(v) for v in ("matmul_tiled_g12x12", "matmul_naive_g16x16")]
kc.argmin(progs, w, {p: (u[j] * 336).contiguous() for j, p in enumerate(progs[0].params)})
for F in (3, 40, 64):
    X = torch.rand((20000 + F, F), dtype=torch.float64, device="cuda")
    kc.fit_weights(X, refine=1)
# per-key (direct) fused Gram path too
prog.set_gram_basis(False)
kc.gram_fused(prog, cols, T)
prog.set_gram_basis(True)
# grid descriptors: fused evaluate + predict and the binding generator
grid = kc.Grid.for_program(prog, {"n": (8, 8, 61), "m": (16, 16, 59), "l": (16, 48, 47)})
kc.predict_grid(w, prog, grid, 17, grid.size - 20, with_status=True)
kc.grid_bindings(grid, 5, 1000)
# fused rows wider than 48 columns: the chunked path (counts -> rows -> wide DMMA Gram)
keys = kc.schema_keys()
wl = ["kernelcost-program v1", "kernel wide52", "param n", "param m", "assume n >= 1", "assume m >= 1"]
wl += [f"prop {keys[k]} (* (^ n {1 + k // 8}) (^ m {k % 8}))" for k in range(52)] + ["end"]
wp = kc.Program("\n".join(wl) + "\n")
wc = {q: torch.randint(1, 9, (5000,), device="cuda") for q in wp.params}
kc.gram_fused(wp, wc, torch.rand(5000, dtype=torch.float64, device="cuda") + 0.5)
# GPU enumeration oracle: box-flattened and triangular domains
kc.load_enum_program("fd_stencil_g16x16").enumerate_points({"n": 256})
kc.load_enum_program("x_triangle").enumerate_points({"n": 300})
kc.load_enum_program("x_guarded").enumerate_points({"n": 200, "m": 150})
torch.cuda.synchronize()
print("sanitize smoke ok")
