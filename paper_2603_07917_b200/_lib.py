"""ctypes binding of libsagesched.so (include/sagesched.h).

This is the only place the package touches the native library.  There is no
CPU fallback: if the library is missing or no CUDA device is present every
entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from ._build import LIB_PATH

SS_OK, SS_ERR_ARG, SS_ERR_RANGE, SS_ERR_EMPTY, SS_ERR_CUDA, SS_ERR_ZERODIV, SS_ERR_UNSUPPORTED = range(7)
ALGO = {"auto": 0, "scan": 1, "tcgen05": 2}
COST_KIND = {"resource-bound": 0, "output-only": 1, "weighted-sum": 2}

P, I64, I32, F32, F64, U64 = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_double, C.c_uint64

# name -> (restype, argtypes); kept in the order of include/sagesched.h
SIGNATURES = {
    "ss_last_error": (C.c_char_p, []),
    "ss_version": (C.c_int, []),
    "ss_launch_count": (I64, []),
    "ss_match_pmfs": (C.c_int, [P, I64, I64, P, F64, I64, P, P, P, I64, P]),
    "ss_gittins_min_batch": (C.c_int, [P, P, P, I64, I64, P, P]),
    "ss_gittins_dist_batch": (C.c_int, [P, P, P, P, P, I64, I64, P, P]),
    "ss_embed_accumulate_batch": (C.c_int, [P, P, I64, U64, I32, P, P]),
    "ss_embed_quantize_batch": (C.c_int, [P, P, I64, U64, I32, P, P, C.POINTER(I64), P]),
    "ss_cost_distribution_batch": (C.c_int, [I32, F64, F64, P, P, P, I64, I64, P, P]),
    "ss_gittins_min_host": (C.c_int, [P, P, I64, C.POINTER(F64), P]),
    "ss_cost_distribution_host": (C.c_int, [I32, F64, F64, F64, P, I64, P, P]),
    "ss_bank_create": (C.c_int, [C.POINTER(P), I32, I64, I32, I64, I64]),
    "ss_bank_destroy": (C.c_int, [P]),
    "ss_bank_push": (C.c_int, [P, P, P, P, I64, P]),
    "ss_bank_push16": (C.c_int, [P, P, P, P, I64, P]),
    "ss_bank_write16": (C.c_int, [P, P, P, P, P, P, I64, P]),
    "ss_bank_write": (C.c_int, [P, P, P, P, P, P, I64, P]),
    "ss_bank_set_head": (C.c_int, [P, I64]),
    "ss_bank_info": (C.c_int, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(I32)]),
    "ss_bank_device_ptrs": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
    "ss_bank_sync_check": (C.c_int, [P, P]),
    "ss_bank_fallback_hist": (C.c_int, [P, I32, I32, P, P, P, P]),
    "ss_topk": (C.c_int, [P, P, P, I64, I32, F32, I32, P, P, P]),
    "ss_topk_wide": (C.c_int, [P, P, P, I64, I64, P, P, P, I32, F32, I32, P, P, P]),
    "ss_query_similar": (C.c_int, [P, P, F32, F32, P, P, P, C.POINTER(I64), P]),
    "ss_topk_partials": (C.c_int, [P, P, P, I64, I32, F32, I32, P, I32, C.POINTER(I32), P]),
    "ss_merge_topk": (C.c_int, [P, P, I32, I64, I32, P, P, P]),
    "ss_topk_scatter": (C.c_int, [P, P, P, I64, I32, F32, I32, I32, I32, P, P, P]),
    "ss_topk_gather": (C.c_int, [P, P, P, I64, I32, F32, I32, I32, I32, P, P, P]),
    "ss_ipc_malloc": (C.c_int, [I32, I64, C.POINTER(P)]),
    "ss_ipc_free": (C.c_int, [P]),
    "ss_ipc_handle": (C.c_int, [P, P]),
    "ss_ipc_open": (C.c_int, [P, C.POINTER(P)]),
    "ss_ipc_close": (C.c_int, [P]),
    "ss_decode_topk": (C.c_int, [P, I64, I64, I64, P, P, P, P]),
    "ss_finish": (C.c_int, [P, P, I64, I32, I32, I32, I32, P, P, P, P, I32, P, P, P, P, P, P, P, P]),
    "ss_refresh": (C.c_int, [I64, P, P, P, I32, P, P, P, I32, P, P, I32, P]),
    "ss_rank_workspace_bytes": (I64, [I64]),
    "ss_rank": (C.c_int, [P, P, I64, P, P, I64, P]),
    "ss_pack_batch": (C.c_int, [P, P, P, I64, I64, I32, I32, P, P, P, P]),
    "ss_table_create": (C.c_int, [C.POINTER(P), I32, I64, I32, I32]),
    "ss_table_destroy": (C.c_int, [P]),
    "ss_table_view": (C.c_int, [P, C.POINTER(I64), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                C.POINTER(P)]),
    "ss_engine_round": (C.c_int, [P, P, P, P, P, P, I64, C.POINTER(I64), I64, I32, I32, I64, I32,
                                  I32, F32, I32, I32, I32, I32, C.POINTER(I64), C.POINTER(I64), P]),
    "ss_schedule_round": (C.c_int, [P, P, P, P, P, I64, I32, F32, I32, I32, I32, I32, I32,
                                    P, P, P, P, P, P, P, P]),
    "ss_schedule_round_wide": (C.c_int, [P, P, P, P, P, I64, I64, P, P, P, I32, F32, I32, I32, I32,
                                         I32, I32, P, P, P, P, P, P, P, P]),
    "ss_schedule_round_host": (C.c_int, [P, P, P, P, P, I64, I32, F32, I32, I32, I32, I32,
                                         P, P, P]),
}

_lib = None


class CudaExtensionMissing(RuntimeError):
    """The sm_100a library is not built / not loadable: there is no fallback."""


def load(path: str | None = None):
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise CudaExtensionMissing(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _lib if _lib is not None else load()


def require_cuda():
    if not torch.cuda.is_available():
        raise CudaExtensionMissing("libsagesched requires a CUDA (sm_100a) device; none is visible")


def last_error() -> str:
    return lib().ss_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == SS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == SS_ERR_ZERODIV:
        raise ZeroDivisionError(msg)
    if rc in (SS_ERR_ARG, SS_ERR_RANGE):
        raise ValueError(msg)
    if rc == SS_ERR_EMPTY:
        raise ColdStartError(msg)
    if rc == SS_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


class ColdStartError(ValueError):
    """Empty window and no fallback."""


def call(name: str, *args) -> int:
    """Call an int-status entry point and raise on failure."""
    rc = getattr(lib(), name)(*args)
    check(rc, name)
    return rc


def ptr(t) -> int | None:
    """Device/host pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def launch_count() -> int:
    return int(lib().ss_launch_count())
