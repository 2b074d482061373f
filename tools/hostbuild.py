"""Tooling, not product (lives outside the package on purpose). The exact evaluator of a lowered program compiled for the host CPU
(kcg_program_jit_source_kind(prog, 4) + g++ -ffp-contract=off): the
optimised-CPU baseline bench.py times beside the GPU, and a CPU-side
cross-check of the code generator in the tests. It is never a fallback:
the package's launch paths only run on the GPU."""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import tempfile
from pathlib import Path

from paper_1604_04997_b200 import _capi

_CACHE = Path(os.environ.get("KCG_HOST_BUILD_DIR", Path(tempfile.gettempdir()) / "kcg_host_build"))


class HostEvaluator:
    """evaluate_properties + predict of one program on host cores."""

    def __init__(self, prog, march: str = "native"):
        self.prog = prog
        src = _capi.lib().kcg_program_jit_source_kind(prog.handle, 4).decode()
        h = hashlib.sha1((src + march).encode()).hexdigest()[:16]
        _CACHE.mkdir(parents=True, exist_ok=True)
        so = _CACHE / f"kcg_host_{h}.so"
        if not so.exists():
            cpp = _CACHE / f"kcg_host_{h}.cpp"
            cpp.write_text(src)
            tmp = so.with_suffix(f".{os.getpid()}.tmp")
            subprocess.run(["g++", "-std=c++17", "-O3", f"-march={march}", "-ffp-contract=off", "-w", "-shared",
                            "-fPIC", str(cpp), "-o", str(tmp)], check=True)
            os.replace(tmp, so)
        self._lib = ctypes.CDLL(str(so))
        self._fn = self._lib.kcg_host_eval
        self._fn.restype = None
        self._fn.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong]
        np_ = max(1, len(prog.params))
        fa = max(1, len(prog.props))

        class Args(ctypes.Structure):
            _fields_ = [("p", ctypes.c_void_p * np_), ("pred", ctypes.c_void_p), ("status", ctypes.c_void_p),
                        ("clo", ctypes.c_void_p), ("chi", ctypes.c_void_p), ("n", ctypes.c_int64),
                        ("sim", ctypes.c_int), ("vec", ctypes.c_int), ("vout", ctypes.c_int),
                        ("alpha", ctypes.c_double * fa), ("alpha_f", ctypes.c_double * fa)]
        self._Args = Args

    def predict(self, alpha149, cols: dict, threads: int = 1, simulate: bool = False):
        """cols: numpy int64 arrays by parameter name -> (pred float64, status uint8)."""
        import concurrent.futures as cf

        import numpy as np
        cs = [np.ascontiguousarray(cols[p], dtype=np.int64) for p in self.prog.params]
        n = len(cs[0]) if cs else 0
        pred = np.empty(n, dtype=np.float64)
        st = np.empty(n, dtype=np.uint8)
        a = self._Args()
        for j, c in enumerate(cs):
            a.p[j] = c.ctypes.data
        a.pred, a.status, a.n, a.sim = pred.ctypes.data, st.ctypes.data, n, 1 if simulate else 0
        for j, k in enumerate(self.prog.props):
            a.alpha[j] = alpha149[k]
        bounds = [n * t // threads for t in range(threads + 1)]
        if threads == 1:
            self._fn(ctypes.byref(a), 0, n)
        else:
            with cf.ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
                list(ex.map(lambda t: self._fn(ctypes.byref(a), bounds[t], bounds[t + 1]), range(threads)))
        return pred, st
