"""ctypes binding of the C-ABI in include/ulysses_b200.h.

The native library is mandatory: if ``libulysses_b200.so`` is missing or
fails to load, importing any compute entry point raises immediately --
there is no CPU or eager-PyTorch fallback for the hot path.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

LIB_NAME = "libulysses_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# profiling A/B only (tools/): load a variant build of the same library
LIB_PATH = os.environ.get("UL_LIB", LIB_PATH)

UL_OK = 0
DTYPE_F32 = 0
DTYPE_BF16 = 1
MASK_NONE = 0
MASK_CAUSAL = 1
MASK_BLOCKED = 2   # Python-side tag; the blocked forward has its own entry point
MAX_RANKS = 16
MAX_FUSED = 4
IPC_HANDLE_BYTES = 128
ABI_VERSION = 2
ATTN_SCHED_BYTES = 8
ATTN_DETERMINISTIC = 1

# every symbol include/ulysses_b200.h declares (tests check the exports)
EXPORTS = (
    "ul_abi_version", "ul_last_error", "ul_preload_kernels", "ul_comm_create", "ul_comm_export_handle",
    "ul_comm_open_peers", "ul_comm_validate_handles", "ul_comm_link_local", "ul_comm_destroy", "ul_comm_rank",
    "ul_comm_world", "ul_comm_slot_bytes", "ul_comm_set_timeout_ms", "ul_comm_status",
    "ul_comm_ledger", "ul_comm_ledger_device", "ul_all_to_all", "ul_all_to_all_head_group", "ul_all_to_all_slot_bytes", "ul_attn_fwd", "ul_attn_fwd_blocked", "ul_qkv_proj_exchange", "ul_proj_exchange", "ul_ring_shift", "ul_lse_merge",
    "ul_attn_bwd_workspace_bytes", "ul_attn_bwd", "ul_attn_bwd_stages", "ul_attn_fwd_exchange",
    "ul_attn_bwd_exchange", "ul_last_launch_count",
    "ul_total_launch_count", "ul_ulysses_volume", "ul_add_layernorm", "ul_layernorm_bwd_workspace_bytes",
    "ul_layernorm_bwd", "ul_gelu",
)

_lib = None

c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p


def _declare(lib):
    P = ctypes.POINTER
    sig = {
        "ul_abi_version": (ctypes.c_int, []),
        "ul_last_error": (ctypes.c_char_p, []),
        "ul_preload_kernels": (ctypes.c_int, []),
        "ul_comm_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_size_t,
                                          P(c_vp)]),
        "ul_comm_export_handle": (ctypes.c_int, [c_vp, c_vp]),
        "ul_comm_open_peers": (ctypes.c_int, [c_vp, c_vp]),
        "ul_comm_validate_handles": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_size_t]),
        "ul_comm_link_local": (ctypes.c_int, [P(c_vp), ctypes.c_int]),
        "ul_comm_destroy": (ctypes.c_int, [c_vp]),
        "ul_comm_rank": (ctypes.c_int, [c_vp]),
        "ul_comm_world": (ctypes.c_int, [c_vp]),
        "ul_comm_slot_bytes": (ctypes.c_size_t, [c_vp]),
        "ul_comm_set_timeout_ms": (ctypes.c_int, [c_vp, c_i64]),
        "ul_comm_status": (ctypes.c_int, [c_vp, ctypes.c_char_p, ctypes.c_size_t]),
        "ul_comm_ledger": (ctypes.c_int, [c_vp, P(ctypes.c_uint64), P(ctypes.c_uint64),
                                          P(ctypes.c_uint64)]),
        "ul_comm_ledger_device": (ctypes.c_int, [c_vp, P(ctypes.c_uint64), P(ctypes.c_uint64), P(ctypes.c_uint64)]),
        "ul_all_to_all": (ctypes.c_int, [c_vp, ctypes.c_int, P(c_vp), P(c_vp), P(c_i64), ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, c_vp]),
        "ul_all_to_all_head_group": (ctypes.c_int, [c_vp, ctypes.c_int, P(c_vp), P(c_vp), P(c_i64), ctypes.c_int,
                                                    ctypes.c_int, ctypes.c_int, ctypes.c_uint64, c_vp]),
        "ul_all_to_all_slot_bytes": (ctypes.c_size_t, [ctypes.c_int, P(c_i64), ctypes.c_int, ctypes.c_int,
                                                       ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "ul_lse_merge": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, ctypes.c_int,
                                        ctypes.c_int, c_vp]),
        "ul_ring_shift": (ctypes.c_int, [c_vp, ctypes.c_int, P(c_vp), P(c_vp), P(c_i64), ctypes.c_int,
                                         ctypes.c_uint64, c_vp]),
        "ul_qkv_proj_exchange": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64,
                                                 c_i64, ctypes.c_uint64, c_vp]),
        "ul_proj_exchange": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, P(c_vp), P(c_i64), c_i64,
                                            c_i64, c_i64, c_i64, ctypes.c_uint64, c_vp]),
        "ul_attn_fwd_blocked": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64,
                                                ctypes.c_int, c_i64, c_vp, c_i64, ctypes.c_float, c_vp]),
        "ul_attn_fwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_float, c_vp, c_vp]),
        "ul_attn_bwd_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i64, c_i64, c_i64, c_i64, ctypes.c_int]),
        "ul_attn_bwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       ctypes.c_size_t, c_i64, c_i64, c_i64, c_i64, c_i64, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_float, ctypes.c_int, c_vp]),
        "ul_attn_bwd_stages": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                              ctypes.c_size_t, c_i64, c_i64, c_i64, c_i64, c_i64, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_float, ctypes.c_int, ctypes.c_int, c_vp]),
        "ul_attn_fwd_exchange": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                                                c_i64, c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                                ctypes.c_uint64, c_vp, c_vp]),
        "ul_attn_bwd_exchange": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                                ctypes.c_size_t, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64,
                                                c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_uint64,
                                                ctypes.c_int, c_vp]),
        "ul_add_layernorm": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, ctypes.c_float,
                                            ctypes.c_int, c_vp]),
        "ul_layernorm_bwd_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i64]),
        "ul_layernorm_bwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, c_i64,
                                            c_i64, ctypes.c_int, c_vp]),
        "ul_gelu": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, ctypes.c_int, c_vp]),
        "ul_last_launch_count": (ctypes.c_int, []),
        "ul_total_launch_count": (ctypes.c_uint64, []),
        "ul_ulysses_volume": (ctypes.c_int, [c_i64, c_i64, c_i64, c_i64, ctypes.c_int, P(c_i64), P(c_i64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded native library (raises if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_NAME} is not built ({LIB_PATH}); run `make` or __graft_entry__.build(). "
                "There is no fallback path.")
        _lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        _declare(_lib)
        if _lib.ul_abi_version() != ABI_VERSION:
            raise RuntimeError("libulysses_b200 ABI version mismatch")
    return _lib


def check(status: int, exc_override=None):
    """Raise the reference-named exception for a non-zero C-ABI status."""
    if status == UL_OK:
        return
    msg = lib().ul_last_error().decode(errors="replace")
    cls = errors.STATUS.get(status, errors.NativeError)
    if exc_override is not None and status in exc_override:
        cls = exc_override[status]
    raise cls(msg)


def last_launch_count() -> int:
    return int(lib().ul_last_launch_count())


def total_launch_count() -> int:
    """Cumulative number of kernels this library launched in the process."""
    return int(lib().ul_total_launch_count())
