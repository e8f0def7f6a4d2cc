"""ctypes binding of include/figaro_cuda.h (libfigaro_cuda.so, built in-tree).

The library is the only compute path: if it is missing or no sm_100 GPU is
present, every call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FG_LIB") or os.path.join(_HERE, "lib", "libfigaro_cuda.so")

FG_OK = 0
FG_E_ARG, FG_E_SCHEMA, FG_E_TREE, FG_E_INTEGRITY, FG_E_SIZE = 1, 2, 3, 4, 5
FG_E_EMPTY_JOIN, FG_E_UNSUPPORTED, FG_E_CUDA, FG_E_RANK, FG_E_NCCL = 6, 7, 8, 9, 10
FG_MEM_DEVICE, FG_MEM_HOST = 0, 1
FG_ENGINE_THIN, FG_ENGINE_HOUSEHOLDER = 0, 1
(FG_ROWS_PER_KEY, FG_THETA_DOWN, FG_FULL_JOIN_SIZE, FG_PHI_CIRC,
 FG_PHI_DOWN, FG_PHI_UP) = range(6)

EXPORTED = [
    "fg_ctx_create", "fg_ctx_destroy", "fg_ctx_set_stream", "fg_ctx_stream",
    "fg_last_error", "fg_version", "fg_kernel_launches", "fg_options_default",
    "fg_run_pipeline", "fg_get_sizes", "fg_get_segments", "fg_get_keys",
    "fg_get_counts", "fg_get_permutation", "fg_get_r0_span_count",
    "fg_get_r0_span", "fg_group_keys", "fg_heads_tails", "fg_tsqr",
    "fg_join_size", "fg_materialize_join", "fg_recover_q", "fg_ctx_set_nccl",
    "fg_gather_r",
]


class fg_relation(C.Structure):
    _fields_ = [("name", C.c_char_p), ("n_key", C.c_int32),
                ("key_attrs", C.POINTER(C.c_char_p)), ("n_data", C.c_int32),
                ("data_attrs", C.POINTER(C.c_char_p)), ("rows", C.c_int64),
                ("keys", C.c_void_p), ("data", C.c_void_p)]


class fg_options(C.Structure):
    _fields_ = [("assume_reduced", C.c_int32), ("engine", C.c_int32),
                ("memory", C.c_int32), ("keep_r0", C.c_int32),
                ("fuse", C.c_int32), ("reserved", C.c_int32 * 3)]


class fg_result(C.Structure):
    _fields_ = [("data_columns", C.c_int64), ("input_rows", C.c_int64),
                ("r0_rows", C.c_int64), ("seconds_group", C.c_double),
                ("seconds_counts", C.c_double), ("seconds_figaro", C.c_double),
                ("seconds_postprocess", C.c_double),
                ("seconds_total", C.c_double), ("kernels", C.c_int64),
                ("seconds_headtail_kernels", C.c_double),
                ("seconds_tsqr_kernels", C.c_double), ("headtail_launches", C.c_int64),
                ("headtail_bytes", C.c_double), ("headtail_fused_flops", C.c_double),
                ("tsqr_stage_flops", C.c_double), ("fused_launches", C.c_int64),
                ("host_syncs", C.c_int64), ("device_mallocs", C.c_int64),
                ("reserved", C.c_int64 * 2)]


class fg_block(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("ld", C.c_int64),
                ("cols", C.c_int32), ("col_begin", C.c_int32)]


_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> C.CDLL:
    """Loads the CUDA library; raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libfigaro_cuda.so not found at {path}; run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
        lib = C.CDLL(path)
        P, I32, I64, V = C.c_void_p, C.c_int32, C.c_int64, None
        sig = {
            "fg_ctx_create": (I32, [I32, C.POINTER(P)]),
            "fg_ctx_destroy": (I32, [P]),
            "fg_ctx_set_stream": (I32, [P, P]),
            "fg_ctx_stream": (P, [P]),
            "fg_last_error": (C.c_char_p, [P]),
            "fg_version": (I32, []),
            "fg_kernel_launches": (I64, [P]),
            "fg_options_default": (V, [C.POINTER(fg_options)]),
            "fg_run_pipeline": (I32, [P, I32, C.POINTER(fg_relation), I32,
                                      C.POINTER(I32), C.POINTER(fg_options), P,
                                      C.POINTER(fg_result)]),
            "fg_get_sizes": (I32, [P, I32, C.POINTER(I64), C.POINTER(I64)]),
            "fg_get_segments": (I32, [P, I32, P]),
            "fg_get_keys": (I32, [P, I32, I32, P]),
            "fg_get_counts": (I32, [P, I32, I32, P]),
            "fg_get_permutation": (I32, [P, I32, P]),
            "fg_get_r0_span_count": (I32, [P, C.POINTER(I32)]),
            "fg_get_r0_span": (I32, [P, I32, C.POINTER(I32), C.POINTER(I64),
                                     C.POINTER(I64), C.POINTER(I64), P]),
            "fg_group_keys": (I32, [P, P, I64, I32, P, P, P, C.POINTER(I64)]),
            "fg_heads_tails": (I32, [P, P, I64, I32, P, P, I64, P, P, P, I64,
                                     P, I64, P]),
            "fg_tsqr": (I32, [P, I32, C.POINTER(fg_block), I32, P]),
            "fg_join_size": (I32, [P, I32, C.POINTER(fg_relation), I32, C.POINTER(I32),
                                   I32, C.c_uint64, C.POINTER(I64)]),
            "fg_materialize_join": (I32, [P, I32, C.POINTER(fg_relation), I32,
                                          C.POINTER(I32), I32, C.c_uint64, P,
                                          C.POINTER(I64)]),
            "fg_ctx_set_nccl": (I32, [P, P]),
            "fg_gather_r": (I32, [P, P, I32, I32, P]),
            "fg_recover_q": (I32, [P, I32, C.POINTER(fg_relation), I32, C.POINTER(I32),
                                   I32, C.c_uint64, P, P, P, C.POINTER(I64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols(path: str = LIB_PATH):
    """Names from EXPORTED that the shared object really exports (no GPU)."""
    lib = C.CDLL(path)
    return [n for n in EXPORTED if hasattr(lib, n)]
