"""ctypes binding of the C ABI in include/terngemm_b200.h.

This is the whole boundary between the Python host mirror and the sm_100a
library: plain pointers, sizes and a stream handle, no torch types.  The
library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2510_06957_b200``) as ``libterngemm_b200.so``.  There is deliberately no
fallback: if the library is missing or the device is not an sm_100 GPU every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CorruptionError, ParameterError

LIB_NAME = "libterngemm_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# developer override (e.g. the clock64-instrumented libterngemm_b200_trace.so); never set in production
LIB_PATH = os.environ.get("TG_LIB_PATH") or LIB_PATH

TG_OK = 0
TG_ERR_PARAM = 1
TG_ERR_CORRUPT = 2
TG_ERR_CUDA = 3
TG_ERR_UNSUPPORTED = 4
TG_ERR_OVERFLOW = 5

TG_FMT_TCSC = 0
TG_FMT_BLOCKED = 1
TG_FMT_INTERLEAVED_BLOCKED = 2
TG_FMT_SYMMETRIC = 3

TG_ORDER_INTERLEAVED_BLOCKED = 0
TG_ORDER_VECTORIZED_OPTIMAL = 1
TG_ORDER_VERTICAL = 0
TG_ORDER_HORIZONTAL = 1


class NativeError(RuntimeError):
    """The CUDA library failed (launch error, missing device, unsupported GPU)."""


class TgSizes(ctypes.Structure):
    _fields_ = [
        ("nnz_pos", ctypes.c_int64),
        ("nnz_neg", ctypes.c_int64),
        ("n_indices", ctypes.c_int64),
        ("num_blocks", ctypes.c_int64),
        ("offsets_len", ctypes.c_int64),
    ]


TG_VARIANT_BASE = 0
TG_VARIANT_BLOCKED = 1
TG_VARIANT_INTERLEAVED_BLOCKED = 2
TG_VARIANT_VECTORIZED_OPTIMAL = 3
TG_VARIANT_UNROLLED = 4
TG_VARIANT_VERTICAL = 5
TG_VARIANT_HORIZONTAL = 6
TG_VARIANT_COMPRESSED = 7

TG_PEER_HEADER_BYTES = 256
TG_PEER_MAX_WORLD = 32
TG_PEER_DONE_WORD = 32
TG_PEER_EPOCH_WORD = 33
TG_PEER_TIMEOUT_WORD = 34
TG_PEER_HANDLE_BYTES = 64


class TgPeerScatter(ctypes.Structure):
    """tg_peer_scatter: peer tables of a fused column-shard scatter (device arrays)."""

    _fields_ = [
        ("y_peers", ctypes.c_void_p),
        ("sig_peers", ctypes.c_void_p),
        ("sig_local", ctypes.c_void_p),
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("col_off", ctypes.c_int64),
    ]


class TgFormatRef(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("g", ctypes.c_int32),
        ("uf", ctypes.c_int32),
        ("mr", ctypes.c_int32),
        ("B", ctypes.c_int64),
        ("a0", ctypes.c_void_p),
        ("a1", ctypes.c_void_p),
        ("a2", ctypes.c_void_p),
        ("a3", ctypes.c_void_p),
        ("codes", ctypes.c_void_p),
    ]


# tg_device_flags: int32 bad_input, int32 nonfinite_output, uint64 nonpositive_outputs,
# int32 corrupt, int32 pad  -> 24 bytes; Python reads it back as 6 int32 words.
FLAGS_BYTES = 24

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_F = ctypes.c_float
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); kept in the order of include/terngemm_b200.h
SIGNATURES: dict[str, tuple] = {
    "tg_abi_version": (_I, []),
    "tg_last_error": (ctypes.c_char_p, []),
    "tg_device_supported": (_I, [_I]),
    "tg_build_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "tg_build_count": (_I, [_P, _I64, _I64, _I64, _I, _I64, _I, _I, _P, _SZ, ctypes.POINTER(TgSizes), _P]),
    "tg_build_fill_tcsc": (_I, [_P, _I64, _I64, _P, _P, _P, _P, _P]),
    "tg_build_fill_blocked": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P]),
    "tg_build_fill_interleaved_blocked": (_I, [_P, _I64, _I64, _I64, _I, _I, _P, _P, _P]),
    "tg_build_fill_symmetric": (_I, [_P, _I64, _I64, _I, _P, _P, _I64, _P]),
    "tg_build_compressed": (_I, [_P, _I64, _I64, _I64, _P, _P]),
    "tg_codes_check": (_I, [_P, _I64, _P, _P]),
    "tg_tiles_bytes": (_SZ, [_I64, _I64]),
    "tg_tiles_from_dense": (_I, [_P, _I64, _I64, _I64, _P, _P, _P]),
    "tg_tiles_from_tcsc": (_I, [_P, _P, _P, _P, _I64, _I64, _P, _P, _P]),
    "tg_tiles_from_blocked": (_I, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P]),
    "tg_tiles_from_interleaved_blocked": (_I, [_P, _P, _I64, _I64, _I64, _I, _P, _P, _P]),
    "tg_tiles_from_symmetric": (_I, [_P, _P, _I64, _I64, _I, _P, _P, _P]),
    "tg_tiles_from_compressed": (_I, [_P, _I64, _I64, _P, _P]),
    "tg_tiles_to_dense": (_I, [_P, _I64, _I64, _P, _P]),
    "tg_gemm_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "tg_gemm_tcsc": (_I, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _P, _P, _I64, _I, _I, _F, _P, _SZ, _P, _P]),
    "tg_gemm_blocked": (
        _I,
        [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _P, _P, _I64, _I, _I, _I, _F, _P, _SZ, _P, _P],
    ),
    "tg_gemm_interleaved_blocked": (
        _I,
        [_P, _I64, _I64, _I64, _I64, _I, _P, _P, _I64, _P, _P, _I64, _I, _I, _F, _P, _SZ, _P, _P],
    ),
    "tg_gemm_symmetric": (
        _I,
        [_P, _I64, _I64, _I64, _I, _P, _P, _I64, _P, _P, _I64, _I, _I, _F, _P, _SZ, _P, _P],
    ),
    "tg_gemm_compressed": (_I, [_P, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _SZ, _P, _P]),
    "tg_gemm_tiles_prepare": (_I, [_P, _I64, _I64, _I64, _P, _SZ, _P, _P]),
    "tg_gemm_tiles_row_stats": (_I, [_P, _SZ, _I64, _I64, _P, _P]),
    "tg_gemm_tiles_run": (_I, [_P, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _I, _F, _P, _P, _SZ, _P, _P]),
    "tg_gemm_tiles": (_I, [_P, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _I, _F, _P, _P, _SZ, _P, _P]),
    "tg_gemm_host_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "tg_gemm_tiles_host": (
        _I,
        [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _I, _F, _P, _P, _SZ, _P, _P, _P],
    ),
    "tg_peer_alloc": (_I, [_SZ, ctypes.POINTER(_P)]),
    "tg_peer_free": (_I, [_P]),
    "tg_peer_export": (_I, [_P, _P]),
    "tg_peer_import": (_I, [_P, ctypes.POINTER(_P)]),
    "tg_peer_release": (_I, [_P]),
    "tg_peer_wait": (_I, [_P, _I, _P]),
    "tg_gemm_tiles_run_scatter": (
        _I,
        [_P, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _I, _F, _P, ctypes.POINTER(TgPeerScatter), _P, _SZ, _P, _P],
    ),
    "tg_probe_i8_mma_rate": (_I, [_I, _I, _I, _I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library (once) and declare every signature."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = LIB_PATH
        if not os.path.exists(path):
            raise NativeError(
                f"{LIB_NAME} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                f"or `make -C {os.path.dirname(LIB_PATH)}` (there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    """Map a tg_status to the reference's exception types (errors.py:4-29)."""
    if rc == TG_OK:
        return
    msg = load().tg_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == TG_ERR_PARAM or rc == TG_ERR_OVERFLOW:
        raise ParameterError(text)
    if rc == TG_ERR_CORRUPT:
        raise CorruptionError(text)
    raise NativeError(f"{text} (status {rc})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
