"""ctypes binding of libkcg.so (include/kcg.h).

This is the reference-side binding a Python caller would add; the C++ side
uses the header directly. Loading fails loudly when the library has not been
built -- there is no CPU fallback for any launch entry point.
"""
from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# KCG_LIB: another build of the same library (e.g. the ASan/UBSan build of
# `make -C paper_1604_04997_b200/csrc asan`, run under LD_PRELOAD=libasan)
LIB_PATH = Path(os.environ["KCG_LIB"]) if os.environ.get("KCG_LIB") else _PKG / "_lib" / "libkcg.so"
HEADER_PATH = _PKG.parent / "include" / "kcg.h"

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded libkcg.so (built by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the kcg back end has no CPU fallback)")
        # torch (if imported first) already holds libcudart.so.12; libkcg
        # links it dynamically so both share one CUDA runtime.
        _lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        _declare(_lib)
    return _lib


P = ctypes.c_void_p
I64P = ctypes.POINTER(ctypes.c_int64)
DP = ctypes.POINTER(ctypes.c_double)
U8P = ctypes.POINTER(ctypes.c_uint8)


def _declare(L: ctypes.CDLL) -> None:
    sig = {
        "kcg_schema_size": (ctypes.c_int, []),
        "kcg_schema_key": (ctypes.c_char_p, [ctypes.c_int]),
        "kcg_schema_index": (ctypes.c_int, [ctypes.c_char_p]),
        "kcg_schema_version": (ctypes.c_char_p, []),
        "kcg_program_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(P)]),
        "kcg_program_destroy": (None, [P]),
        "kcg_program_num_params": (ctypes.c_int, [P]),
        "kcg_program_param_name": (ctypes.c_char_p, [P, ctypes.c_int]),
        "kcg_program_num_props": (ctypes.c_int, [P]),
        "kcg_program_prop_schema_index": (ctypes.c_int, [P, ctypes.c_int]),
        "kcg_program_kernel_name": (ctypes.c_char_p, [P]),
        "kcg_program_safe_bounds": (ctypes.c_int, [P, I64P, I64P]),
        "kcg_program_set_engine": (ctypes.c_int, [P, ctypes.c_int]),
        "kcg_program_set_gram_basis": (ctypes.c_int, [P, ctypes.c_int]),
        "kcg_program_jit_source": (ctypes.c_char_p, [P]),
        "kcg_program_jit_source_kind": (ctypes.c_char_p, [P, ctypes.c_int]),
        "kcg_jit_compile_check": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p]),
        "kcg_eval_predict": (ctypes.c_int, [P, P, ctypes.c_size_t, DP, P, P, P, P, ctypes.c_int, P]),
        "kcg_argmin": (ctypes.c_int, [P, ctypes.c_int, P, ctypes.c_size_t, DP, P, P, P, P]),
        "kcg_gram_accumulate": (ctypes.c_int, [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, P, P, P, P]),
        "kcg_gram_accumulate_sliced": (ctypes.c_int, [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, P, P, P, P]),
        "kcg_gram_fused": (ctypes.c_int, [P, P, P, ctypes.c_size_t, P, P, P, P, P]),
        "kcg_residual_accumulate": (ctypes.c_int, [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, P, P, P]),
        "kcg_residual_fused": (ctypes.c_int, [P, P, P, ctypes.c_size_t, DP, P, P]),
        "kcg_residual_grad_fused": (ctypes.c_int, [P, P, P, ctypes.c_size_t, DP, P, P]),
        "kcg_residual_grad_obj_fused": (ctypes.c_int, [P, P, P, ctypes.c_size_t, DP, P, P, P]),
        "kcg_gram_residual_grad": (ctypes.c_int, [P, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, P, P, P]),
        "kcg_simulate_time": (ctypes.c_int, [P, P, ctypes.c_size_t, DP, ctypes.c_double, ctypes.c_uint64,
                                             ctypes.c_uint64, P, P, P]),
        "kcg_geomean_accumulate": (ctypes.c_int, [P, P, ctypes.c_size_t, P, P, P, P]),
        "kcg_measurements_read_csv": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(P)]),
        "kcg_measurements_destroy": (None, [P]),
        "kcg_measurements_num_kernels": (ctypes.c_int, [P]),
        "kcg_measurements_kernel": (ctypes.c_char_p, [P, ctypes.c_int]),
        "kcg_measurements_num_rows": (ctypes.c_size_t, [P, ctypes.c_int]),
        "kcg_measurements_num_params": (ctypes.c_int, [P, ctypes.c_int]),
        "kcg_measurements_param_name": (ctypes.c_char_p, [P, ctypes.c_int, ctypes.c_int]),
        "kcg_measurements_column": (I64P, [P, ctypes.c_int, ctypes.c_int]),
        "kcg_measurements_times": (DP, [P, ctypes.c_int]),
        "kcg_solve_gram": (ctypes.c_int, [ctypes.c_int, DP, DP, DP, DP, ctypes.POINTER(ctypes.c_int)]),
        "kcg_refine_gram": (ctypes.c_int, [ctypes.c_int, DP, DP, DP, DP]),
        "kcg_weights_read_json": (ctypes.c_int, [ctypes.c_char_p, DP, U8P, DP, ctypes.POINTER(ctypes.c_uint64)]),
        "kcg_weights_write_json": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, DP, U8P, ctypes.c_double, ctypes.c_uint64]),
        "kcg_enum_program_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(P)]),
        "kcg_enum_program_destroy": (None, [P]),
        "kcg_enum_program_num_params": (ctypes.c_int, [P]),
        "kcg_enum_program_param_name": (ctypes.c_char_p, [P, ctypes.c_int]),
        "kcg_enumerate_points": (ctypes.c_int, [P, I64P, ctypes.c_uint64, I64P, I64P,
                                                ctypes.POINTER(ctypes.c_uint64), P]),
        "kcg_grid_bindings": (ctypes.c_int, [P, ctypes.c_uint64, ctypes.c_size_t, P, P]),
        "kcg_eval_predict_grid": (ctypes.c_int, [P, P, ctypes.c_uint64, ctypes.c_size_t, DP, P, P, ctypes.c_int, P]),
        "kcg_columns_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, P, P, P, ctypes.c_uint64]),
        "kcg_columns_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(P)]),
        "kcg_columns_close": (None, [P]),
        "kcg_columns_num_rows": (ctypes.c_uint64, [P]),
        "kcg_columns_num_cols": (ctypes.c_int, [P]),
        "kcg_columns_name": (ctypes.c_char_p, [P, ctypes.c_int]),
        "kcg_columns_dtype": (ctypes.c_int, [P, ctypes.c_int]),
        "kcg_columns_find": (ctypes.c_int, [P, ctypes.c_char_p]),
        "kcg_columns_data": (P, [P, ctypes.c_int]),
        "kcg_columns_load": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t, P, P]),
        "kcg_status_str": (ctypes.c_char_p, [ctypes.c_int]),
        "kcg_point_status_str": (ctypes.c_char_p, [ctypes.c_int]),
        "kcg_last_error": (ctypes.c_char_p, []),
        "kcg_launch_count": (ctypes.c_uint64, []),
        "kcg_eval_predict_host": (ctypes.c_int, [P, ctypes.c_int, P, ctypes.c_size_t, P, P, P, ctypes.c_uint]),
        "kcg_host_last_path": (ctypes.c_uint, []),
        "kcg_multi_jit_source": (ctypes.c_char_p, [P, ctypes.c_int, ctypes.c_int]),
        "kcg_eval_predict_multi": (ctypes.c_int, [P, ctypes.c_int, P, ctypes.c_size_t, P, P, ctypes.c_size_t, P,
                                                  ctypes.c_size_t, P]),
        "kcg_measure_stream": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]),
        "kcg_measure_pipe_peak": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def header_functions() -> list[str]:
    """Function names declared in include/kcg.h (for the export check)."""
    text = HEADER_PATH.read_text()
    return sorted(set(re.findall(r"\b(kcg_[a-z0-9_]+)\s*\(", text)))


class KcgError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        name = lib().kcg_status_str(code).decode()
        super().__init__(f"{name}: {message}")
        self.name = name


def check(rc: int) -> None:
    if rc != 0:
        raise KcgError(rc, lib().kcg_last_error().decode())


# status codes (kcg.h)
OK = 0
E_PARSE = 1
E_CAP_EXCEEDED = 4
E_ASSUMPTION_VIOLATED = 6
E_SCHEMA_MISMATCH = 7
E_NONPOSITIVE_TIME = 8
E_EMPTY = 9
E_IO = 10
E_INVALID_ARGUMENT = 11
E_CUDA = 100
HOST_PINNED = 1  # kcg_eval_predict_host flags (KCG_HOST_PINNED)
HOST_PATH_2D = 2  # kcg_host_last_path bits
HOST_PATH_ONEPASS = 4
E_JIT = 101
E_UNSUPPORTED = 102

PT_OK = 0
PT_ASSUMPTION_VIOLATED = 1
PT_NONINTEGRAL = 2
PT_OVERFLOW = 3
PT_COUNT_WIDE = 4

ENGINE_JIT = 0
ENGINE_INTERP = 1
