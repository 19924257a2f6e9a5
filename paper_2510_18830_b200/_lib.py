"""ctypes loader for libmtsa.so (the C ABI in include/mtsa.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no fallback — a missing or unloadable library raises.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libmtsa.so"

MT_STATUS = {
    0: "MT_OK", 1: "MT_ESHAPE", 2: "MT_EWINDOW", 3: "MT_ECONFIG", 4: "MT_ELAYOUT",
    5: "MT_ECAPACITY", 6: "MT_EWORKSPACE", 7: "MT_EUNSUPPORTED", 8: "MT_ECUDA", 9: "MT_ENCCL",
}


class MTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{MT_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = MT_STATUS.get(status, str(status))


class Shape(ctypes.Structure):
    _fields_ = [("seq_len", ctypes.c_int64), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("block", ctypes.c_int32), ("last_q", ctypes.c_int32), ("layout", ctypes.c_int32)]


class VSParams(ctypes.Structure):
    _fields_ = [("p_v", ctypes.c_float), ("p_s", ctypes.c_float)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA path has no fallback)")
        _lib = ctypes.CDLL(str(LIB_PATH))
        _lib.mt_last_error.restype = ctypes.c_char_p
        for name, argtypes in _SIGS.items():
            fn = getattr(_lib, name)
            fn.restype = _RESTYPE.get(
                name, ctypes.c_size_t if name.endswith("_workspace_bytes") else ctypes.c_int)
            fn.argtypes = argtypes
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise MTError(status, lib().mt_last_error().decode(errors="replace"))


P = ctypes.c_void_p
I = ctypes.c_int
I64 = ctypes.c_int64
SZ = ctypes.c_size_t

_SIGS: dict[str, list] = {
    "mt_selftest_mma": [I, P, P, P, P],
    "mt_debug_bwd_timeline": [P],
    "mt_debug_fwd_timeline": [P],
    "mt_sparse_attn_fwd_workspace_bytes": [P, I],
    "mt_sparse_attn_fwd": [P, P, P, P, P, P, P, P, SZ, P],
    "mt_attn_fwd_step": [P, I, I, I, I, I, P, P, P, P, P, P, P, P, SZ, P],
    "mt_build_vs_index_workspace_bytes": [P, I],
    "mt_build_vs_index": [P, P, P, P, P, P, P, SZ, P],
    "mt_rope_vs_index": [P, P, P, P, ctypes.c_float, P, P, P, P, P, P, SZ, P],
    "mt_vs_column_scores": [P, P, P, P, P, P, SZ, P],
    "mt_comm_unique_id": [P],
    "mt_comm_create": [P, I, I, I, P],
    "mt_comm_destroy": [P],
    "mt_comm_check": [P],
    "mt_comm_profile": [P, I],
    "mt_comm_step_times": [P, I, I, P, P],
    "mt_sparse_attn_bwd_workspace_bytes": [P],
    "mt_sparse_attn_bwd": [P, P, P, P, P, P, P, P, P, P, P, P, SZ, P],
    "mt_attn_step_workspace_bytes": [P, I],
    "mt_attn_bwd_preprocess": [P, I, P, P, P, P],
    "mt_attn_bwd_step": [P, I, I, I, P, P, P, P, P, P, P, P, P, P, P, SZ, P],
    "mt_ring_attn_workspace_bytes": [P, I, I],
    "mt_ring_attn_fwd": [P, P, P, P, P, P, P, P, P, SZ, P],
    "mt_ring_attn_bwd": [P, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P],
    "mt_ring_schedule": [I, I, P],
    "mt_stripe": [I64, I64, I, I, P, P, P],
    "mt_block_sparse_attn_fwd_workspace_bytes": [P],
    "mt_block_sparse_attn_fwd": [P, P, P, P, P, P, I64, P, P, P, SZ, P],
    "mt_block_sparse_attn_bwd_workspace_bytes": [P, I64],
    "mt_block_sparse_attn_bwd": [P, P, P, P, P, P, P, P, P, I64, P, P, P, P, SZ, P],
    "mt_xattn_index_workspace_bytes": [P],
    "mt_xattn_index_count": [P, P, P, P, P, P, P, P, SZ, P],
    "mt_xattn_index_fill": [P, P, P, P, I64, I64, P, SZ, P],
    "mt_rope_inv_freq": [I, ctypes.c_double, ctypes.c_double, I64, P, P],
    "mt_rope": [I64, I, I, I, P, ctypes.c_float, I, P, P],
    "mt_vs_format_workspace_bytes": [P],
    "mt_vs_format_count": [P, P, P, P, P, P, P, SZ, P],
    "mt_vs_format_fill": [P, P, P, P, P, I64, P, I64, I64, I64, P, SZ, P],
    "mt_unstripe": [I64, I64, I, I, P, P, P],
    "mt_layout_to_local": [I, I64, I64, I, I, P, P, P],
    "mt_layout_to_global": [I, I64, I64, I, I, P, P, P],
    "mt_launch_count": [],
    "mt_ring_flags_bytes": [],
    "mt_comm_register_workspace": [P, P, SZ, P],
    "mt_comm_copy_engine": [P],
    "mt_library_call_count": [],
}
_RESTYPE = {"mt_sparse_attn_fwd_workspace_bytes": ctypes.c_size_t,
            "mt_build_vs_index_workspace_bytes": ctypes.c_size_t,
            "mt_sparse_attn_bwd_workspace_bytes": ctypes.c_size_t,
            "mt_attn_step_workspace_bytes": ctypes.c_size_t,
            "mt_ring_attn_workspace_bytes": ctypes.c_size_t,
            "mt_vs_format_workspace_bytes": ctypes.c_size_t,
            "mt_launch_count": ctypes.c_ulonglong,
            "mt_ring_flags_bytes": ctypes.c_size_t,
            "mt_library_call_count": ctypes.c_ulonglong}


def declared_symbols() -> list[str]:
    return ["mt_last_error", *_SIGS.keys()]
