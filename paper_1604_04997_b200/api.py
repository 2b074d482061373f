"""Python host mirror of the reference API for the batched hot path.

Names and meaning follow kernelcost's C++ API (proj/core/include/kernelcost):
``evaluate_properties`` (props.hpp:49-50), ``predict`` (model.hpp:61),
``noiseless_time`` (simdevice.hpp:33), ``build_design_matrix`` /
``fit_weights`` (model.hpp:43-49), ``read_weights_json`` /
``write_weights_json`` (jsonio.hpp:27-29) -- batched over SoA bindings that
live in HBM. Every call goes through the C ABI of libkcg.so (include/kcg.h);
PyTorch only provides device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Mapping, Optional, Sequence

from . import _capi
from ._capi import check, lib

PROGRAM_DIR = Path(__file__).resolve().parent / "programs"


# ---------------------------------------------------------------------------
# schema v1 (schema.cpp:16-38)

def schema_keys() -> list[str]:
    L = lib()
    return [L.kcg_schema_key(i).decode() for i in range(L.kcg_schema_size())]


def schema_size() -> int:
    return lib().kcg_schema_size()


def schema_index(key: str) -> int:
    i = lib().kcg_schema_index(key.encode())
    if i < 0:
        raise _capi.KcgError(_capi.E_SCHEMA_MISMATCH, f"unknown property key '{key}'")
    return i


# ---------------------------------------------------------------------------
# programs

class Program:
    """A kernel's symbolic PropertyVector + assumptions, lowered for the GPU.

    ``text`` is the front end's program text (kernelcost-program v1), i.e.
    what ``program_text(k, extract_properties(k))`` prints on the reference
    side.
    """

    def __init__(self, text: str):
        self.text = text
        h = _capi.P()
        raw = text.encode()
        check(lib().kcg_program_create(raw, len(raw), ctypes.byref(h)))
        self._h = h
        L = lib()
        self.name = L.kcg_program_kernel_name(h).decode()
        self.params = [L.kcg_program_param_name(h, i).decode()
                       for i in range(L.kcg_program_num_params(h))]
        self.props = [L.kcg_program_prop_schema_index(h, j)
                      for j in range(L.kcg_program_num_props(h))]
        keys = schema_keys()
        self.keys = [keys[i] for i in self.props]

    @classmethod
    def from_file(cls, path) -> "Program":
        return cls(Path(path).read_text())

    @property
    def handle(self):
        return self._h

    def safe_bounds(self) -> tuple[int, int]:
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(lib().kcg_program_safe_bounds(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def set_engine(self, engine: str) -> None:
        code = {"jit": _capi.ENGINE_JIT, "interp": _capi.ENGINE_INTERP}[engine]
        check(lib().kcg_program_set_engine(self._h, code))

    def set_gram_basis(self, enable: bool) -> None:
        """Fused Gram / residual rows over the keys' monomial basis (default)
        or one correctly rounded column per key (include/kcg.h)."""
        check(lib().kcg_program_set_gram_basis(self._h, 1 if enable else 0))

    def jit_source(self) -> str:
        return lib().kcg_program_jit_source(self._h).decode()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _capi._lib is not None:
            _capi._lib.kcg_program_destroy(h)
            self._h = None

    def __repr__(self):
        return f"Program({self.name!r}, params={self.params}, props={len(self.props)})"


def suite_index() -> list[dict]:
    import json
    return json.loads((PROGRAM_DIR / "index.json").read_text())["kernels"]


def load_program(kernel_id: str) -> Program:
    """Front-end output for one bundled suite kernel (programs/<id>.kcp)."""
    path = PROGRAM_DIR / f"{kernel_id}.kcp"
    if not path.exists():
        raise FileNotFoundError(f"no symbolic program for '{kernel_id}' (extraction needs a binding)")
    return Program.from_file(path)


# ---------------------------------------------------------------------------
# weights (jsonio.cpp:96-143)

@dataclass
class ModelWeights:
    device: str = ""
    schema_version: str = "v1"
    alpha: list = field(default_factory=lambda: [0.0] * 149)
    covered: list = field(default_factory=lambda: [False] * 149)
    objective: float = 0.0
    n_cases: int = 0

    def alpha_array(self):
        n = schema_size()
        if self.schema_version != "v1" or len(self.alpha) != n:
            raise _capi.KcgError(_capi.E_SCHEMA_MISMATCH,
                                 f"model weights use schema '{self.schema_version}', expected 'v1'")
        return (ctypes.c_double * n)(*self.alpha)


def read_weights_json(path) -> ModelWeights:
    n = schema_size()
    a = (ctypes.c_double * n)()
    c = (ctypes.c_uint8 * n)()
    obj = ctypes.c_double()
    nc = ctypes.c_uint64()
    check(lib().kcg_weights_read_json(str(path).encode(), a, c, ctypes.byref(obj), ctypes.byref(nc)))
    import json
    dev = json.loads(Path(path).read_text()).get("device", "")
    return ModelWeights(dev, "v1", list(a), [bool(x) for x in c], obj.value, nc.value)


def write_weights_json(path, w: ModelWeights) -> None:
    n = schema_size()
    a = w.alpha_array()
    c = (ctypes.c_uint8 * n)(*[1 if x else 0 for x in w.covered])
    check(lib().kcg_weights_write_json(str(path).encode(), w.device.encode(), a, c,
                                        float(w.objective), int(w.n_cases)))


# ---------------------------------------------------------------------------
# launches

def _torch():
    import torch
    return torch


def _stream(stream=None) -> int:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _np():
    import numpy
    return numpy


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _columns(prog: Program, bindings):
    """SoA int64 device columns in ``prog.params`` order."""
    torch = _torch()
    if isinstance(bindings, Mapping):
        cols = [bindings[p] for p in prog.params]
    elif isinstance(bindings, torch.Tensor) and bindings.dim() == 2:
        cols = [bindings[j] for j in range(bindings.shape[0])]
    else:
        cols = list(bindings)
    if len(cols) != len(prog.params):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT,
                             f"binding has {len(cols)} columns, kernel has params {prog.params}")
    n = None
    out = []
    for c in cols:
        if not (c.is_cuda and c.dtype == torch.int64 and c.is_contiguous()):
            raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "binding columns must be contiguous int64 CUDA tensors")
        if n is None:
            n = c.numel()
        elif c.numel() != n:
            raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "ragged binding columns")
        out.append(c)
    arr = (ctypes.c_void_p * max(1, len(out)))(*[c.data_ptr() for c in out])
    return arr, (n or 0), out


@dataclass
class BoundBatch:
    """Batched evaluate_properties result: exact counts + per-point status."""
    program: Program
    counts_lo: object          # [F_nz, N] int64
    counts_hi: object | None   # [F_nz, N] int64 (high words) or None
    status: object             # [N] uint8

    def counts_int(self, j: int, i: int) -> int:
        lo = int(self.counts_lo[j, i]) & ((1 << 64) - 1)
        hi = int(self.counts_hi[j, i]) if self.counts_hi is not None else (-1 if lo >> 63 else 0)
        return (hi << 64) | lo


def evaluate_properties(prog: Program, bindings, wide: bool = True, stream=None) -> BoundBatch:
    """Batched ``evaluate_properties`` (props.cpp:259-271): exact counts of
    the program's nonzero keys at every binding, plus a status per point
    (E_ASSUMPTION_VIOLATED etc. instead of an exception)."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    dev = cols[0].device if cols else torch.device("cuda")
    F = len(prog.props)
    lo = torch.empty((max(F, 1), n), dtype=torch.int64, device=dev)
    hi = torch.empty((max(F, 1), n), dtype=torch.int64, device=dev) if wide else None
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    check(lib().kcg_eval_predict(prog.handle, arr, n, None, None, st.data_ptr(), lo.data_ptr(),
                                 _ptr(hi), 0, _stream(stream)))
    return BoundBatch(prog, lo[:F], hi[:F] if hi is not None else None, st)


def predict(w: ModelWeights, prog: Program, bindings, with_status: bool = False, stream=None):
    """Batched ``predict`` (model.cpp:95-117) fused with the evaluation:
    seconds per binding; NaN where the binding is not admissible."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    dev = cols[0].device if cols else torch.device("cuda")
    pred = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev) if with_status else None
    check(lib().kcg_eval_predict(prog.handle, arr, n, w.alpha_array(), pred.data_ptr(), _ptr(st),
                                 None, None, 0, _stream(stream)))
    return (pred, st) if with_status else pred


def noiseless_time(alpha149: Sequence[float], prog: Program, bindings, stream=None):
    """Batched ``noiseless_time`` (simdevice.cpp:76-90): the stored-timing
    inner product, summed in schema order skipping zero weights."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    pred = torch.empty(n, dtype=torch.float64, device=cols[0].device)
    a = (ctypes.c_double * len(alpha149))(*alpha149)
    check(lib().kcg_eval_predict(prog.handle, arr, n, a, pred.data_ptr(), None, None, None, 1,
                                 _stream(stream)))
    return pred


def simulate_time(alpha149: Sequence[float], prog: Program, bindings, sigma: float = 0.0, seed: int = 0,
                  run: int = 0, with_status: bool = False, stream=None):
    """Batched ``simulate_time`` / ``simulate_runs`` (simdevice.cpp:96-127):
    the synthetic device's stored timings, noise keyed by
    "<kernel>|<binding_str>" exactly as the reference keys it."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    out = torch.empty(n, dtype=torch.float64, device=cols[0].device)
    st = torch.empty(n, dtype=torch.uint8, device=cols[0].device) if with_status else None
    a = (ctypes.c_double * len(alpha149))(*alpha149)
    check(lib().kcg_simulate_time(prog.handle, arr, n, a, float(sigma), int(seed), int(run), out.data_ptr(),
                                  _ptr(st), _stream(stream)))
    return (out, st) if with_status else out


def geometric_mean_error(pred, actual, stream=None) -> float:
    """``geometric_mean_error`` (model.cpp:119-133) over device tensors."""
    torch = _torch()
    if pred.numel() == 0:
        raise _capi.KcgError(_capi.E_EMPTY, "no error pairs")
    ls = torch.zeros(1, dtype=torch.float64, device=pred.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=pred.device)
    bad = torch.zeros(1, dtype=torch.int64, device=pred.device)
    check(lib().kcg_geomean_accumulate(pred.data_ptr(), actual.data_ptr(), pred.numel(), ls.data_ptr(),
                                       cnt.data_ptr(), bad.data_ptr(), _stream(stream)))
    if int(bad.item()):
        raise _capi.KcgError(_capi.E_NONPOSITIVE_TIME, "actual time must be positive")
    return math.exp(float(ls.item()) / int(cnt.item()))


def argmin(progs: Sequence[Program], w: ModelWeights, bindings, return_preds: bool = False, stream=None):
    """Autotuning sweep: fused evaluate + predict over kernel variants with
    an argmin per problem size (lowest variant index wins ties)."""
    torch = _torch()
    arr, n, cols = _columns(progs[0], bindings)
    dev = cols[0].device
    best = torch.empty(n, dtype=torch.int32, device=dev)
    best_t = torch.empty(n, dtype=torch.float64, device=dev)
    preds = torch.empty((len(progs), n), dtype=torch.float64, device=dev) if return_preds else None
    handles = (ctypes.c_void_p * len(progs))(*[p.handle.value for p in progs])
    check(lib().kcg_argmin(handles, len(progs), arr, n, w.alpha_array(), best.data_ptr(),
                           best_t.data_ptr(), _ptr(preds), _stream(stream)))
    return (best, best_t, preds) if return_preds else (best, best_t)


def predict_multi(progs: Sequence[Program], w: ModelWeights, bindings, status: bool = False, out=None,
                  stream=None):
    """``predict`` of every program over one set of device bindings in one
    pass (kcg_eval_predict_multi): each size's bindings are read once.
    bindings follow progs[0]'s parameters; returns a [len(progs), n] float64
    CUDA tensor (and the [len(progs), n] uint8 status). `out` may be a
    preallocated [len(progs), >= n] float64 CUDA tensor with unit column
    stride (its row stride is the leading dimension)."""
    torch = _torch()
    progs = list(progs)
    arr, n, cols = _columns(progs[0], bindings)
    dev = cols[0].device if cols else torch.device("cuda")
    V = len(progs)
    pred = out if out is not None else torch.empty((V, n), dtype=torch.float64, device=dev)
    if (pred.dim() != 2 or pred.shape[0] != V or pred.shape[1] < n or pred.dtype != torch.float64
            or not pred.is_cuda or (pred.stride(1) != 1 and n > 1)):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "out must be a [n_progs, >= n] float64 CUDA tensor")
    st = torch.empty((V, n), dtype=torch.uint8, device=dev) if status else None
    handles = (ctypes.c_void_p * V)(*[p.handle.value for p in progs])
    check(lib().kcg_eval_predict_multi(handles, V, arr, n, w.alpha_array(), pred.data_ptr(), max(pred.stride(0), n),
                                       _ptr(st), n, _stream(stream)))
    return (pred, st) if status else pred


def multi_jit_source(progs: Sequence[Program], argmin: bool = False) -> str:
    """Generated CUDA of the one-pass multi-program kernels (diagnostics):
    predict_multi's, or (argmin=True) argmin's."""
    progs = list(progs)
    handles = (ctypes.c_void_p * len(progs))(*[p.handle.value for p in progs])
    src = lib().kcg_multi_jit_source(handles, len(progs), int(argmin))
    if src is None:
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, lib().kcg_last_error().decode())
    return src.decode()


def predict_host(progs: Sequence[Program], w: ModelWeights, bindings, status: bool = False,
                 out=None, pinned: Optional[bool] = None):
    """The reference's calling convention: HOST bindings in, HOST
    predictions out (predict over every program, model.cpp:95-117), through
    kcg_eval_predict_host -- chunked H2D / kernels / D2H on internal
    streams, each binding copied to the device once for all programs.
    bindings: {param: int64 numpy array or CPU tensor}; returns a
    [len(progs), n] float64 CPU tensor (and [len(progs), n] uint8 status).
    `out` may be a preallocated (pinned) CPU tensor of that shape. pinned:
    the buffers are page-locked (default: detected from the tensors)."""
    torch = _torch()
    progs = list(progs)
    cols = []
    for name in progs[0].params:
        c = bindings[name]
        c = c if isinstance(c, torch.Tensor) else torch.from_numpy(_np().ascontiguousarray(c, dtype=_np().int64))
        if c.dtype != torch.int64 or c.device.type != "cpu":
            raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "predict_host takes int64 CPU columns")
        cols.append(c.contiguous())
    n = int(cols[0].numel()) if cols else 0
    if any(int(c.numel()) != n for c in cols):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "binding columns differ in length")
    V = len(progs)
    pred = out if out is not None else torch.empty((V, n), dtype=torch.float64)
    if tuple(pred.shape) != (V, n) or pred.dtype != torch.float64 or not pred.is_contiguous():
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "out must be a contiguous [n_progs, n] float64 CPU tensor")
    if pinned is None:
        pinned = all(t.is_pinned() for t in cols + [pred]) if n else False
    st = None
    if status:  # the status buffer follows the caller's buffers (pinned or not)
        st = torch.empty((V, n), dtype=torch.uint8, pin_memory=bool(pinned and n))
    handles = (ctypes.c_void_p * V)(*[p.handle.value for p in progs])
    arr = (ctypes.c_void_p * max(1, len(cols)))(*[c.data_ptr() for c in cols])
    check(lib().kcg_eval_predict_host(handles, V, arr, n, w.alpha_array(), pred.data_ptr(),
                                      _ptr(st), _capi.HOST_PINNED if pinned else 0))
    return (pred, st) if status else pred


# ---------------------------------------------------------------------------
# fit (model.cpp:11-93) via Gram statistics

@dataclass
class GramStats:
    G: object       # [F, F] fp64
    xt1: object     # [F]
    colmax: object  # [F]
    n_rows: int = 0
    bad_rows: int = 0

    @classmethod
    def zeros(cls, F: int, device="cuda"):
        torch = _torch()
        z = lambda *s: torch.zeros(*s, dtype=torch.float64, device=device)
        return cls(z(F, F), z(F), z(F))


def _check_design(X) -> None:
    """X: a CUDA float64 [N, F] matrix with unit column stride (rows may be
    padded: stride(0) >= F). Anything else would be read out of bounds or
    silently mis-strided by the kernels."""
    torch = _torch()
    if not (isinstance(X, torch.Tensor) and X.dim() == 2 and X.is_cuda and X.dtype == torch.float64
            and (X.stride(1) == 1 or X.shape[1] <= 1) and X.stride(0) >= X.shape[1]):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT,
                             "X must be a CUDA float64 [N, F] tensor with stride(1) == 1")


def _check_times(T, n: int, device) -> None:
    """T: n contiguous CUDA float64 measured times on the bindings' device."""
    torch = _torch()
    if not (isinstance(T, torch.Tensor) and T.is_cuda and T.dtype == torch.float64 and T.is_contiguous()
            and T.numel() == n and T.device == device):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT,
                             f"T must be {n} contiguous CUDA float64 times on {device}")


def gram_accumulate(X, stats: GramStats | None = None, stream=None, sliced: bool = False) -> GramStats:
    """G += XᵀX, Xᵀ1, colmax over a materialised design X [N, F] fp64.
    sliced=True takes the int8 tensor-core back end (kcg_gram_accumulate_sliced,
    17 <= F <= 40, contiguous X)."""
    _check_design(X)
    N, F = X.shape
    stats = stats or GramStats.zeros(F, X.device)
    fn = lib().kcg_gram_accumulate_sliced if sliced else lib().kcg_gram_accumulate
    check(fn(X.data_ptr(), N, F, X.stride(0), stats.G.data_ptr(),
             stats.xt1.data_ptr(), stats.colmax.data_ptr(), _stream(stream)))
    stats.n_rows += N
    return stats


def gram_fused(prog: Program, bindings, T, stats: GramStats | None = None, stream=None) -> GramStats:
    """Fused evaluate -> design row (count/T, model.cpp:29) -> Gram."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    _check_times(T, n, cols[0].device if cols else T.device)
    F = len(prog.props)
    stats = stats or GramStats.zeros(F, cols[0].device)
    bad = torch.zeros(1, dtype=torch.int64, device=cols[0].device)
    check(lib().kcg_gram_fused(prog.handle, arr, T.data_ptr(), n, stats.G.data_ptr(),
                               stats.xt1.data_ptr(), stats.colmax.data_ptr(), bad.data_ptr(),
                               _stream(stream)))
    stats.n_rows += n
    stats.bad_rows += int(bad.item())
    return stats


def residual_fused(prog: Program, bindings, T, alpha149: Sequence[float], stream=None) -> float:
    """Objective sum_r (1 - x_r . alpha)^2 of the fit (model.cpp:81-92) with
    rows x_r = count/T formed from the bindings on the fly."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    _check_times(T, n, cols[0].device if cols else T.device)
    obj = torch.zeros(1, dtype=torch.float64, device=cols[0].device)
    a = (ctypes.c_double * len(alpha149))(*alpha149)
    check(lib().kcg_residual_fused(prog.handle, arr, T.data_ptr(), n, a, obj.data_ptr(), _stream(stream)))
    return float(obj.item())


def residual_grad_fused(prog: Program, bindings, T, alpha149: Sequence[float], g=None, stream=None, r2=None):
    """g += X^T (1 - X alpha) over the rows x_j = RN(count_j)/T formed on the
    fly (model.cpp:29), residual in twice the working precision: the
    refinement gradient after a fused Gram. Returns the [F] device tensor
    (program key order). r2 (a [1] fp64 device tensor, optional) += the sum
    of the squared residuals, for refined_objective."""
    torch = _torch()
    arr, n, cols = _columns(prog, bindings)
    _check_times(T, n, cols[0].device if cols else T.device)
    if g is None:
        g = torch.zeros(len(prog.props), dtype=torch.float64, device=T.device)
    a = (ctypes.c_double * len(alpha149))(*alpha149)
    if r2 is None:
        check(lib().kcg_residual_grad_fused(prog.handle, arr, T.data_ptr(), n, a, g.data_ptr(), _stream(stream)))
    else:
        if not (r2.is_cuda and r2.dtype == torch.float64 and r2.numel() >= 1):
            raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "r2 must be a CUDA float64 tensor")
        check(lib().kcg_residual_grad_obj_fused(prog.handle, arr, T.data_ptr(), n, a, g.data_ptr(), r2.data_ptr(),
                                                _stream(stream)))
    return g


def refined_objective(stats: GramStats, alpha_old: Sequence[float], alpha_new: Sequence[float], g, r2) -> float:
    """sum (1 - x.alpha_new)^2 (model.cpp:81-92) from the refinement pass at
    alpha_old -- r2 = sum r^2, g = X^T r with r = 1 - X alpha_old -- and the
    Gram: |r - X d|^2 = r2 - 2 d.g + d^T G d, d = alpha_new - alpha_old.
    The two correction terms are second order in a refinement step, so the
    result carries r2's relative accuracy; no further pass over the rows."""
    import numpy as np
    G = stats.G.double().cpu().numpy()
    gh = g.double().cpu().numpy()
    d = np.asarray(alpha_new, dtype=np.float64) - np.asarray(alpha_old, dtype=np.float64)
    return float(float(r2.double().sum().item()) - 2.0 * float(d @ gh) + float(d @ (G @ d)))


def refine_gram(stats: GramStats, alpha: Sequence[float], g) -> list[float]:
    """One refinement step of the equilibrated solve: alpha += G^+ g
    (kcg_refine_gram); g = X^T (1 - X alpha) from an accurate residual."""
    G = stats.G.double().cpu().contiguous()
    F = G.shape[0]
    dp = lambda t: ctypes.cast(t.data_ptr(), _capi.DP)
    cm = stats.colmax.double().cpu().contiguous()
    gh = g.double().cpu().contiguous()
    arr = (ctypes.c_double * F)(*alpha)
    check(lib().kcg_refine_gram(F, dp(G), dp(cm), dp(gh), arr))
    return list(arr)


def fit_fused(prog: Program, bindings, T, refine: int = 2, stream=None):
    """fit_weights (model.cpp:37-93) over rows formed from bindings and
    measured times on the fly: fused Gram, host equilibrated min-norm
    solve, `refine` refinement steps with the fused residual gradient, the
    objective at the refined weights from the last of them
    (refined_objective; the fused residual pass when refine = 0). Returns
    (alpha over the program's keys, rank, objective, GramStats)."""
    torch = _torch()
    st = gram_fused(prog, bindings, T, stream=stream)
    alpha, rank = solve_gram(st)
    K = schema_size()

    def full(a):
        out = [0.0] * K
        for j, k in enumerate(prog.props):
            out[k] = a[j]
        return out
    if refine == 0:
        return alpha, rank, residual_fused(prog, bindings, T, full(alpha), stream=stream), st
    for step in range(refine):
        last = step == refine - 1
        r2 = torch.zeros(1, dtype=torch.float64, device=T.device) if last else None
        g = residual_grad_fused(prog, bindings, T, full(alpha), stream=stream, r2=r2)
        new = refine_gram(st, alpha, g)
        if last:  # the objective at the refined weights from this pass (no residual pass)
            obj = refined_objective(st, alpha, new, g, r2)
        alpha = new
    return alpha, rank, obj, st


def solve_gram(stats: GramStats) -> tuple[list[float], int]:
    """Host minimum-norm solve of the equilibrated normal equations."""
    G = stats.G.double().cpu().contiguous()
    F = G.shape[0]
    dp = lambda t: ctypes.cast(t.data_ptr(), _capi.DP)
    xt1 = stats.xt1.double().cpu().contiguous()
    cm = stats.colmax.double().cpu().contiguous()
    out = (ctypes.c_double * F)()
    rank = ctypes.c_int()
    check(lib().kcg_solve_gram(F, dp(G), dp(xt1), dp(cm), out, ctypes.byref(rank)))
    return list(out), rank.value


@dataclass
class FitResult:
    alpha: list
    covered: list
    objective: float
    rank: int
    n_cases: int


def fit_weights(X, refine: int = 2, stream=None) -> FitResult:
    """``fit_weights`` (model.cpp:37-93) over a materialised design X whose
    rows are p/T (``build_design_matrix``): Gram reduction on the GPU, host
    min-norm solve, `refine` semi-normal refinement passes (the residual in
    double-double, so each pass moves the weights toward the exact
    least-squares solution of X: two reach it to ~1e-13 on the reference's
    fit fixtures), objective from a residual pass (never from the Gram
    identity)."""
    torch = _torch()
    _check_design(X)
    N, F = X.shape
    if N == 0:
        raise _capi.KcgError(_capi.E_EMPTY, "empty design matrix")
    st = gram_accumulate(X, stream=stream)
    alpha, rank = solve_gram(st)
    G = st.G.cpu().contiguous()
    cm = st.colmax.cpu().contiguous()
    dp = lambda t: ctypes.cast(t.data_ptr(), _capi.DP)
    for _ in range(refine):
        a_dev = torch.tensor(alpha, dtype=torch.float64, device=X.device)
        g = torch.zeros(F, dtype=torch.float64, device=X.device)
        check(lib().kcg_gram_residual_grad(X.data_ptr(), N, F, X.stride(0), a_dev.data_ptr(),
                                           g.data_ptr(), _stream(stream)))
        gh = g.cpu().contiguous()
        arr = (ctypes.c_double * F)(*alpha)
        check(lib().kcg_refine_gram(F, dp(G), dp(cm), dp(gh), arr))
        alpha = list(arr)
    a_dev = torch.tensor(alpha, dtype=torch.float64, device=X.device)
    obj = torch.zeros(1, dtype=torch.float64, device=X.device)
    check(lib().kcg_residual_accumulate(X.data_ptr(), N, F, X.stride(0), a_dev.data_ptr(),
                                        obj.data_ptr(), _stream(stream)))
    covered = [bool(c > 0) for c in cm.tolist()]
    return FitResult(alpha, covered, float(obj.item()), rank, N)


def launch_count() -> int:
    return int(lib().kcg_launch_count())


PIPE_KINDS = {"imad": 0, "lop3": 1, "dfma": 2, "issue": 3}


def measure_stream(n_read: int, n_write: int, n_points: int = 1 << 27) -> float:
    """HBM bytes/s of a stream reading n_read int64 and writing n_write fp64
    columns (kcg_measure_stream): the same-mix bandwidth roofline."""
    out = ctypes.c_double()
    check(lib().kcg_measure_stream(n_read, n_write, n_points, ctypes.byref(out)))
    return out.value


def measure_pipe_peak(kind: str, iters: int = 4096) -> float:
    """Measured lane operations per second of one pipe of the current device
    (csrc/peaks.cu): "imad", "lop3", "dfma", or "issue" (IMAD and LOP3
    alternating, i.e. the scheduler's issue rate for an integer mix)."""
    import ctypes
    out = ctypes.c_double()
    check(lib().kcg_measure_pipe_peak(PIPE_KINDS[kind], iters, ctypes.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# measurement CSVs -> GPU fit / eval (the CLI's `fit` and `eval`,
# kernelcost.cpp:236-272 and 366-400)

@dataclass
class KernelMeasurements:
    kernel: str
    params: list          # binding parameter names (sorted)
    columns: dict         # name -> numpy int64 array
    times: object         # numpy float64 array


def read_measurements(path, discard: int = 4) -> list[KernelMeasurements]:
    """Measurement or raw-runs CSV (csvio.cpp:104-225), grouped per kernel."""
    import numpy as np
    h = _capi.P()
    check(lib().kcg_measurements_read_csv(str(path).encode(), int(discard), ctypes.byref(h)))
    L = lib()
    try:
        out = []
        for i in range(L.kcg_measurements_num_kernels(h)):
            n = L.kcg_measurements_num_rows(h, i)
            params = [L.kcg_measurements_param_name(h, i, j).decode()
                      for j in range(L.kcg_measurements_num_params(h, i))]
            cols = {p: np.ctypeslib.as_array(L.kcg_measurements_column(h, i, j), shape=(n,)).copy()
                    for j, p in enumerate(params)}
            t = np.ctypeslib.as_array(L.kcg_measurements_times(h, i), shape=(n,)).copy()
            out.append(KernelMeasurements(L.kcg_measurements_kernel(h, i).decode(), params, cols, t))
        return out
    finally:
        L.kcg_measurements_destroy(h)


@dataclass
class CampaignRecord:
    """One simulated observation (MeasurementRecord / RawRun, csvio.hpp)."""
    kernel: str
    binding: dict
    group_config: str
    run_index: int
    time_s: float


def binding_str(b: Mapping) -> str:
    """csvio.cpp:77-84: "k=v;..." in key order (std::map)."""
    return ";".join(f"{k}={int(b[k])}" for k in sorted(b))


def run_campaign(cases, alpha149: Sequence[float], sigma: float = 0.0, seed: int = 0, runs: int = 1,
                 programs=None, stream=None):
    """``kernelcost simulate`` on the GPU: run_campaign (campaign.cpp:11-45)
    with simulate_time / simulate_runs (simdevice.cpp:96-128) for every case
    (kernel, binding, group_config), all cases of one kernel in one batched
    launch per run. Returns (records in case order, runs innermost, and
    the diagnostics of failed cases "<kernel> [<binding>]: <error>", as the
    reference reports instead of aborting)."""
    torch = _torch()
    if runs <= 0:
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "run count must be positive")
    cases = [(k, {p: int(v) for p, v in b.items()}, g) for k, b, g in cases]
    by_kernel = {}
    for i, (k, _, _) in enumerate(cases):
        by_kernel.setdefault(k, []).append(i)
    times = [[0.0] * runs for _ in cases]
    fails = {}
    for k, idx in by_kernel.items():
        prog = _program_for(k, programs)
        cols = {}
        for p in prog.params:
            if any(p not in cases[i][1] for i in idx):
                for i in idx:
                    if p not in cases[i][1]:
                        fails[i] = f"E_INVALID_ARGUMENT: binding missing parameter '{p}'"
            cols[p] = torch.tensor([cases[i][1].get(p, 0) for i in idx], dtype=torch.int64, device="cuda")
        for r in range(runs):
            t, st = simulate_time(alpha149, prog, cols, sigma=sigma, seed=seed, run=r, with_status=True,
                                  stream=stream)
            t, st = t.cpu().tolist(), st.cpu().tolist()
            for j, i in enumerate(idx):
                if st[j] != _capi.PT_OK and i not in fails:
                    fails[i] = ("E_ASSUMPTION_VIOLATED: binding violates the kernel's assumptions"
                                if st[j] == _capi.PT_ASSUMPTION_VIOLATED
                                else lib().kcg_point_status_str(st[j]).decode())
                times[i][r] = t[j]
    records, diags = [], []
    for i, (k, b, g) in enumerate(cases):
        if i in fails:
            diags.append(f"{k} [{binding_str(b)}]: {fails[i]}")
            continue
        records.extend(CampaignRecord(k, b, g, r, times[i][r]) for r in range(runs))
    return records, diags


def write_measurements_csv(path, records) -> None:
    """csvio.cpp:104-114 (kernel,binding,group_config,time_s; %.17g),
    byte-identical to the reference's file for the same records."""
    lines = ["kernel,binding,group_config,time_s"]
    lines += [f"{r.kernel},{binding_str(r.binding)},{r.group_config},{r.time_s:.17g}" for r in records]
    Path(path).write_text("\n".join(lines) + "\n")


def write_raw_runs_csv(path, records) -> None:
    """csvio.cpp:144-155 (... ,run_index,time_s)."""
    lines = ["kernel,binding,group_config,run_index,time_s"]
    lines += [f"{r.kernel},{binding_str(r.binding)},{r.group_config},{r.run_index},{r.time_s:.17g}" for r in records]
    Path(path).write_text("\n".join(lines) + "\n")


def write_campaign_columns(path, records) -> None:
    """The same records as a kcg-columns v1 file (bulk campaigns): one int64
    column per parameter, run_index and time_s (records of one kernel)."""
    import numpy as np
    if not records:
        raise _capi.KcgError(_capi.E_EMPTY, "no records")
    params = sorted(records[0].binding)
    if any(r.kernel != records[0].kernel or sorted(r.binding) != params for r in records):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "a columns campaign file holds one kernel")
    cols = {p: np.array([r.binding[p] for r in records], dtype=np.int64) for p in params}
    cols["run_index"] = np.array([r.run_index for r in records], dtype=np.int64)
    cols["time_s"] = np.array([r.time_s for r in records], dtype=np.float64)
    write_columns(path, cols)


_SUITE_PROGRAMS: dict = {}  # bundled programs used by the CSV fit / eval (parsed and lowered once)


def _program_for(kernel: str, programs) -> Program:
    if programs is None:
        prog = _SUITE_PROGRAMS.get(kernel)
        if prog is None:
            prog = _SUITE_PROGRAMS[kernel] = load_program(kernel)
        return prog
    if isinstance(programs, Mapping):
        return programs[kernel]
    return Program.from_file(Path(programs) / f"{kernel}.kcp")


def _device_rows(km: KernelMeasurements, prog: Program, device="cuda"):
    torch = _torch()
    if sorted(prog.params) != sorted(km.params):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT,
                             f"binding missing parameter for kernel '{km.kernel}': {km.params} vs {prog.params}")
    cols = {p: torch.from_numpy(km.columns[p]).to(device) for p in prog.params}
    T = torch.from_numpy(km.times).to(device)
    return cols, T


def fit_from_csv(path, programs=None, device: str = "", discard: int = 4, stream=None, refine: int = 2):
    """``kernelcost fit <csv>`` on the GPU: per kernel the fused
    evaluate -> row -> Gram kernel, scattered into the schema-wide Gram
    (rows of different kernels are disjoint), one equilibrated min-norm
    solve, `refine` refinement steps (residual gradient over the reference's
    own rows in twice the working precision), the objective at the refined
    weights from the last of them (refined_objective; the fused residual
    pass when refine = 0). Returns
    (ModelWeights, report) with report = {objective, n_cases, rank, bad_rows}."""
    torch = _torch()
    K = schema_size()
    G = torch.zeros((K, K), dtype=torch.float64, device="cuda")
    x1 = torch.zeros(K, dtype=torch.float64, device="cuda")
    cm = torch.zeros(K, dtype=torch.float64, device="cuda")
    meas = read_measurements(path, discard)
    if not meas:
        raise _capi.KcgError(_capi.E_EMPTY, "no fit cases")
    rows = 0
    staged = []
    bad_dev = torch.zeros(1, dtype=torch.int64, device="cuda")  # read once, after every kernel
    for km in meas:
        if (km.times <= 0).any():
            raise _capi.KcgError(_capi.E_NONPOSITIVE_TIME, f"observed time must be positive ({km.kernel})")
        prog = _program_for(km.kernel, programs)
        cols, T = _device_rows(km, prog)
        arr, n, _ = _columns(prog, cols)
        st = GramStats.zeros(len(prog.props), "cuda")
        check(lib().kcg_gram_fused(prog.handle, arr, T.data_ptr(), n, st.G.data_ptr(), st.xt1.data_ptr(),
                                   st.colmax.data_ptr(), bad_dev.data_ptr(), _stream(stream)))
        idx = torch.tensor(prog.props, dtype=torch.int64, device="cuda")
        G[idx.unsqueeze(1), idx.unsqueeze(0)] += st.G
        x1[idx] += st.xt1
        cm[idx] = torch.maximum(cm[idx], st.colmax)
        rows += n
        staged.append((prog, cols, T, idx, arr, n))
    bad = int(bad_dev.item())
    if bad:
        raise _capi.KcgError(_capi.E_ASSUMPTION_VIOLATED, f"{bad} measurement rows are not admissible")
    stats = GramStats(G, x1, cm, rows)
    alpha, rank = solve_gram(stats)
    if refine == 0:
        obj = sum(residual_fused(prog, cols, T, alpha, stream=stream) for prog, cols, T, *_ in staged)
    for step in range(refine):  # schema-wide gradient: the kernels' rows are disjoint
        last = step == refine - 1
        g = torch.zeros(K, dtype=torch.float64, device="cuda")
        r2 = torch.zeros(1, dtype=torch.float64, device="cuda") if last else None
        a = (ctypes.c_double * len(alpha))(*alpha)  # one host weight array for every kernel of the step
        for prog, cols, T, idx, arr, n in staged:
            gk = torch.zeros(len(prog.props), dtype=torch.float64, device="cuda")
            if r2 is None:
                check(lib().kcg_residual_grad_fused(prog.handle, arr, T.data_ptr(), n, a, gk.data_ptr(),
                                                    _stream(stream)))
            else:
                check(lib().kcg_residual_grad_obj_fused(prog.handle, arr, T.data_ptr(), n, a, gk.data_ptr(),
                                                        r2.data_ptr(), _stream(stream)))
            g[idx] += gk
        new = refine_gram(stats, alpha, g)
        if last:  # objective at the refined weights from this pass (no residual pass per kernel)
            obj = refined_objective(stats, alpha, new, g, r2)
        alpha = new
    covered = [bool(c > 0) for c in cm.cpu().tolist()]
    w = ModelWeights(device, "v1", list(alpha), covered, obj, rows)
    return w, {"objective": obj, "n_cases": rows, "rank": rank, "bad_rows": bad}


def eval_from_csv(w: ModelWeights, path, programs=None, discard: int = 4, stream=None) -> dict:
    """``kernelcost eval <csv> --weights w.json`` on the GPU: batched
    predict per kernel and geometric mean relative error per kernel and
    overall (model.cpp:119-133)."""
    torch = _torch()
    per, preds, acts = {}, [], []
    for km in read_measurements(path, discard):
        prog = _program_for(km.kernel, programs)
        cols, T = _device_rows(km, prog)
        p = predict(w, prog, cols, stream=stream)
        per[km.kernel] = geometric_mean_error(p, T, stream=stream)
        preds.append(p)
        acts.append(T)
    overall = geometric_mean_error(torch.cat(preds), torch.cat(acts), stream=stream)
    return {"per_kernel": per, "overall": overall, "n_cases": sum(int(a.numel()) for a in acts)}


# ---- GPU enumeration oracle (enumerate.cpp:371-456) -------------------------

ENUM_DIR = PROGRAM_DIR / "enum"


class EnumProgram:
    """A kernel's enumeration program ("kernelcost-enum v1", printed by the
    reference front end with oracle/kcref_program.hpp enum_text): every
    statement domain, guard, access and per-point op count that
    ``enumerate_points`` walks."""

    def __init__(self, text: str):
        h = ctypes.c_void_p()
        b = text.encode()
        check(lib().kcg_enum_program_create(b, len(b), ctypes.byref(h)))
        self._h = h
        L = lib()
        self.params = [L.kcg_enum_program_param_name(h, i).decode()
                       for i in range(L.kcg_enum_program_num_params(h))]

    @classmethod
    def from_file(cls, path) -> "EnumProgram":
        return cls(Path(path).read_text())

    def enumerate_points(self, binding: dict, cap: int = 0, stream=None) -> tuple[dict, int]:
        """Brute-force bound property vector at one binding, walked on the
        GPU: ({schema key: exact int} for the nonzero keys, visited points).
        Raises KcgError E_ASSUMPTION_VIOLATED / E_CAP_EXCEEDED like the
        reference."""
        b = (ctypes.c_int64 * max(1, len(self.params)))(*[int(binding[p]) for p in self.params])
        n = schema_size()
        lo, hi = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
        pts = ctypes.c_uint64()
        check(lib().kcg_enumerate_points(self._h, b, cap, lo, hi, ctypes.byref(pts), _stream(stream)))
        keys = schema_keys()
        out = {}
        for i in range(n):
            v = (hi[i] << 64) | (lo[i] & ((1 << 64) - 1))
            if v:
                out[keys[i]] = v
        return out, pts.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _capi._lib is not None:
            _capi._lib.kcg_enum_program_destroy(h)
            self._h = None


def load_enum_program(kernel_id: str) -> EnumProgram:
    """Enumeration program of one bundled suite kernel (programs/enum/<id>.kce)."""
    return EnumProgram.from_file(ENUM_DIR / f"{kernel_id}.kce")


# ---- grid descriptors --------------------------------------


class _KcgGrid(ctypes.Structure):
    _fields_ = [("n_params", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("start", ctypes.c_int64 * 8), ("step", ctypes.c_int64 * 8), ("count", ctypes.c_uint64 * 8)]


@dataclass
class Grid:
    """Lattice of bindings (include/kcg.h kcg_grid): parameter j takes
    start[j] + step[j] * d_j, d_j in [0, count[j]), the last parameter
    varying fastest. ``axes`` maps parameter name -> (start, step, count)
    and is ordered by the program's declaration order when built with
    :meth:`for_program`."""
    params: list
    start: list
    step: list
    count: list

    @classmethod
    def for_program(cls, prog, axes: Mapping) -> "Grid":
        ps = list(prog.params)
        return cls(ps, [int(axes[p][0]) for p in ps], [int(axes[p][1]) for p in ps], [int(axes[p][2]) for p in ps])

    @property
    def size(self) -> int:
        n = 1
        for c in self.count:
            n *= c
        return n

    def c_struct(self) -> _KcgGrid:
        g = _KcgGrid()
        g.n_params = len(self.params)
        for j in range(len(self.params)):
            g.start[j], g.step[j], g.count[j] = self.start[j], self.step[j], self.count[j]
        return g


def grid_bindings(grid: Grid, first: int = 0, n: int | None = None, device="cuda", stream=None) -> dict:
    """Materialise lattice points [first, first + n) as SoA int64 columns."""
    torch = _torch()
    n = grid.size - first if n is None else n
    cols = {p: torch.empty(n, dtype=torch.int64, device=device) for p in grid.params}
    arr = (ctypes.c_void_p * max(1, len(cols)))(*[c.data_ptr() for c in cols.values()])
    g = grid.c_struct()
    check(lib().kcg_grid_bindings(ctypes.byref(g), first, n, arr, _stream(stream)))
    return cols


def predict_grid(w: ModelWeights, prog: Program, grid: Grid, first: int = 0, n: int | None = None,
                 with_status: bool = False, simulate: bool = False, device="cuda", stream=None):
    """``predict`` (or ``noiseless_time`` with simulate=True) over lattice
    points [first, first + n) without materialising the bindings."""
    torch = _torch()
    if list(grid.params) != list(prog.params):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, f"grid params {grid.params} != kernel params {prog.params}")
    n = grid.size - first if n is None else n
    pred = torch.empty(n, dtype=torch.float64, device=device)
    st = torch.empty(n, dtype=torch.uint8, device=device) if with_status else None
    g = grid.c_struct()
    check(lib().kcg_eval_predict_grid(prog.handle, ctypes.byref(g), first, n, w.alpha_array(), pred.data_ptr(),
                                      _ptr(st), 1 if simulate else 0, _stream(stream)))
    return (pred, st) if with_status else pred


# ---- kcg-columns v1 binary side format -----------------------

_COL_DTYPES = {"int64": 1, "float64": 2, "uint8": 3, "int32": 4}
_COL_NAMES = {v: k for k, v in _COL_DTYPES.items()}


def write_columns(path, columns: Mapping) -> None:
    """Write SoA columns (numpy arrays or CPU/CUDA tensors of int64, float64,
    uint8 or int32, equal lengths) as a kcg-columns v1 file."""
    import numpy as np
    arrs = []
    for name, c in columns.items():
        if hasattr(c, "detach"):
            c = c.detach().cpu().numpy()
        a = np.ascontiguousarray(c)
        if a.dtype.name not in _COL_DTYPES:
            raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, f"column '{name}': unsupported dtype {a.dtype}")
        arrs.append((name, a))
    n = len(arrs[0][1]) if arrs else 0
    if any(len(a) != n for _, a in arrs):
        raise _capi.KcgError(_capi.E_INVALID_ARGUMENT, "ragged columns")
    k = len(arrs)
    names = (ctypes.c_char_p * max(1, k))(*[nm.encode() for nm, _ in arrs])
    dts = (ctypes.c_int * max(1, k))(*[_COL_DTYPES[a.dtype.name] for _, a in arrs])
    ptrs = (ctypes.c_void_p * max(1, k))(*[a.ctypes.data for _, a in arrs])
    check(lib().kcg_columns_write(str(path).encode(), k, names, dts, ptrs, n))


class Columns:
    """A mapped kcg-columns v1 file: ``numpy(name)`` is a zero-copy view of
    the mapping, ``to_device(name)`` copies (a slice of) a column into a new
    CUDA tensor through kcg_columns_load."""

    def __init__(self, path):
        h = ctypes.c_void_p()
        check(lib().kcg_columns_open(str(path).encode(), ctypes.byref(h)))
        self._h = h
        L = lib()
        self.n_rows = int(L.kcg_columns_num_rows(h))
        self.names = [L.kcg_columns_name(h, j).decode() for j in range(L.kcg_columns_num_cols(h))]
        self.dtypes = {nm: _COL_NAMES[L.kcg_columns_dtype(h, j)] for j, nm in enumerate(self.names)}

    def _index(self, name: str) -> int:
        j = lib().kcg_columns_find(self._h, name.encode())
        if j < 0:
            raise KeyError(name)
        return j

    def numpy(self, name: str):
        import numpy as np
        j = self._index(name)
        dt = np.dtype(self.dtypes[name])
        ptr = lib().kcg_columns_data(self._h, j)
        buf = (ctypes.c_char * (self.n_rows * dt.itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dt)

    def to_device(self, name: str, row0: int = 0, n: int | None = None, device="cuda", stream=None):
        torch = _torch()
        j = self._index(name)
        n = self.n_rows - row0 if n is None else n
        out = torch.empty(n, dtype=getattr(torch, self.dtypes[name]), device=device)
        check(lib().kcg_columns_load(self._h, j, row0, n, out.data_ptr(), _stream(stream)))
        return out

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and _capi._lib is not None:
            _capi._lib.kcg_columns_close(h)
            self._h = None

    def __del__(self):
        self.close()


def read_columns(path) -> Columns:
    return Columns(path)


# ---- Prediction detail (model.cpp:95-117) -------------------------------------


@dataclass
class Prediction:
    """``kernelcost::Prediction``: seconds, the per-key (key, part)
    breakdown in schema order and the uncovered keys that contributed."""
    seconds: float
    breakdown: list
    warnings: list


def predict_detail(w: ModelWeights, prog: Program, bindings, indices=None, stream=None) -> list:
    """``predict`` with its breakdown and warnings for selected points
    (model.cpp:95-117): the exact counts come from the GPU
    (evaluate_properties), the per-key parts are formed on the host in
    schema order exactly as the reference does (double(count) round to
    nearest even, part = alpha * count, seconds += part). Inadmissible
    points give None (the reference raises E_ASSUMPTION_VIOLATED)."""
    w.alpha_array()  # schema check (model.cpp:96-100)
    bb = evaluate_properties(prog, bindings, wide=True, stream=stream)
    torch = _torch()
    torch.cuda.synchronize()
    st = bb.status.cpu().tolist()
    n = len(st)
    keys = schema_keys()
    out = []
    for i in (range(n) if indices is None else indices):
        if st[i] != _capi.PT_OK:
            out.append(None)
            continue
        seconds, br, warn = 0.0, [], []
        for j, k in enumerate(prog.props):
            c = bb.counts_int(j, i)
            if c == 0:
                continue
            part = w.alpha[k] * float(c)
            seconds += part
            br.append((keys[k], part))
            if not w.covered[k]:
                warn.append(keys[k])
        out.append(Prediction(seconds, br, warn))
    return out
