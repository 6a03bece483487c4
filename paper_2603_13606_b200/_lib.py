"""ctypes binding of libepb200.so (the C ABI in include/epb200.h).

There is no Python fallback for anything this library computes: if the
shared object is missing or cannot be loaded, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libepb200.so")

# status codes (include/epb200.h, epsim ErrorCode order core.py:21-28)
OK, INVALID_ARGUMENT, SHAPE_MISMATCH, TAG_MISMATCH, CONFIG_MISMATCH, \
    CAPACITY_EXCEEDED, HANDLE_STATE_ERROR, TRANSPORT_CLOSED, CUDA_ERROR = range(9)

F32, BF16, F16, FP8 = range(4)
LL, HT = 0, 1


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "algorithm", "num_ranks", "ranks_per_node", "num_experts", "top_k", "hidden",
        "max_tokens_per_rank", "token_dtype", "with_scales", "layout",
        "ht_chunk_tokens", "ht_fifo_depth", "combine_dtype", "expert_out_window")]


class WindowInfo(ctypes.Structure):
    _fields_ = [("physical_bytes", ctypes.c_uint64), ("logical_bytes", ctypes.c_uint64),
                ("expert_out_offset", ctypes.c_uint64), ("expert_out_rows", ctypes.c_uint64),
                ("token_in_offset", ctypes.c_uint64), ("token_in_rows", ctypes.c_uint64)]


class Layout(ctypes.Structure):
    _fields_ = [("expert_count", ctypes.c_void_p), ("rank_count", ctypes.c_void_p),
                ("tok_rank", ctypes.c_void_p), ("tok_slot", ctypes.c_void_p),
                ("num_tokens", ctypes.c_int32)]


class LLDispatchArgs(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("x_dtype", ctypes.c_int32), ("x_scales", ctypes.c_void_p),
                ("topk_idx", ctypes.c_void_p), ("num_tokens", ctypes.c_int32),
                ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32), ("out_scales", ctypes.c_void_p),
                ("counts_f32", ctypes.c_void_p), ("counts_i32", ctypes.c_void_p),
                ("src_info", ctypes.c_void_p), ("self_row", ctypes.c_void_p), ("owner_row", ctypes.c_void_p)]


class LLCombineArgs(ctypes.Structure):
    _fields_ = [("expert_out", ctypes.c_void_p), ("in_dtype", ctypes.c_int32),
                ("counts_i32", ctypes.c_void_p), ("src_info", ctypes.c_void_p),
                ("weights", ctypes.c_void_p), ("num_tokens", ctypes.c_int32),
                ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32), ("self_row", ctypes.c_void_p),
                ("topk", ctypes.c_void_p), ("owner_row", ctypes.c_void_p),
                ("expert_out_in_window", ctypes.c_int32)]


class HTDispatchArgs(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("x_dtype", ctypes.c_int32), ("weights", ctypes.c_void_p),
                ("topk_idx", ctypes.c_void_p), ("num_tokens", ctypes.c_int32),
                ("rank_count", ctypes.c_void_p), ("tok_rank", ctypes.c_void_p), ("tok_slot", ctypes.c_void_p),
                ("offsets", ctypes.c_void_p), ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32),
                ("origin", ctypes.c_void_p), ("origin_w", ctypes.c_void_p)]


class HTCombineArgs(ctypes.Structure):
    _fields_ = [("expert_rows", ctypes.c_void_p), ("in_dtype", ctypes.c_int32), ("origin", ctypes.c_void_p),
                ("recv_total", ctypes.c_int32), ("topk_idx", ctypes.c_void_p), ("weights", ctypes.c_void_p),
                ("num_tokens", ctypes.c_int32), ("tok_rank", ctypes.c_void_p), ("offsets", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32),
                ("dispatch_weights", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p),
                ("expert_rows_in_window", ctypes.c_int32)]


PHASE_SEND, PHASE_RECV, PHASE_BOTH = 1, 2, 3


class IpcDesc(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_uint8 * 64), ("offset", ctypes.c_uint64),
                ("bytes", ctypes.c_uint64), ("device", ctypes.c_int32), ("pid", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_U = ctypes.c_uint32
_L = ctypes.c_int64
_Q = ctypes.c_uint64

SIGNATURES = {
    "epb_version": [],
    "epb_last_error": [],
    "epb_window_geometry": [ctypes.POINTER(Config), ctypes.POINTER(WindowInfo)],
    "epb_group_create": [ctypes.POINTER(Config), ctypes.c_int, _P, _Q, _P, ctypes.POINTER(_P)],
    "epb_group_window": [_P, ctypes.POINTER(_P), ctypes.POINTER(_Q)],
    "epb_group_ipc_desc": [_P, ctypes.POINTER(IpcDesc)],
    "epb_group_open_peers": [_P, ctypes.POINTER(IpcDesc)],
    "epb_group_set_peers": [_P, ctypes.POINTER(_Q)],
    "epb_group_set_timeout": [_P, _Q],
    "epb_group_set_trace": [_P, _P],
    "epb_group_barrier": [_P, _P],
    "epb_group_poll_error": [_P, ctypes.c_int, ctypes.POINTER(_I)],
    "epb_group_error_word": [_P, ctypes.POINTER(ctypes.c_void_p)],
    "epb_group_set_op_trace": [_P, _P, _U],
    "epb_group_destroy": [_P],
    "epb_routing_layout": [_P, _P, _I, ctypes.POINTER(Layout), _P],
    "epb_ll_dispatch": [_P, _P, _I, ctypes.c_void_p, _P],
    "epb_ll_combine": [_P, _P, _I, ctypes.c_void_p, _P],
    "epb_ht_meta_send": [_P, _U, ctypes.POINTER(Layout), _P],
    "epb_ht_meta_recv": [_P, _U, _P, _P, _P, _P],
    "epb_ht_open": [_P, _U, _P, _I, ctypes.POINTER(Layout), _P, _P, _P],
    "epb_ht_dispatch": [_P, _U, _I, ctypes.c_void_p, _P],
    "epb_ht_combine": [_P, _U, _I, ctypes.c_void_p, _P],
    "epb_weights_equal": [_P, _P, _P, _L, _P],
    "epb_fp8_quantize": [_P, _I, _L, _I, _P, _P, _P],
    "epb_fp8_dequantize": [_P, _P, _L, _I, _P, _P],
    "epb_e4m3_encode": [_P, _L, _P, _P],
    "epb_convert": [_P, _I, _P, _I, _L, _P],
    "epb_check_finite": [_P, _L, _P, _P],
}

_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load (once) and return the CDLL; raises LibraryMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = ctypes.c_char_p if name == "epb_last_error" else ctypes.c_int
            _lib = lib
    return _lib


def last_error() -> str:
    return load().epb_last_error().decode(errors="replace")


def call(name: str, *args) -> None:
    """Invoke an entry point; non-zero status raises EpError."""
    rc = getattr(load(), name)(*args)
    if rc != OK:
        from .core import raise_status
        raise_status(rc, f"{name}: {last_error()}")
