"""ctypes binding of the C-ABI in ``include/kvx.h`` (the drop-in boundary).

There is no CPU fallback: if ``_kvx.so`` is missing or fails to load, every
data-path call raises.  Error codes map to the reference's conventions
(``costs.py:25-26,98-99`` ValueError; ``costs.py:63-64`` NoPath).
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import NoPath

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "_kvx.so")

KVX_OK = 0
KVX_ERR_INVALID_ARG = 10001
KVX_ERR_NO_PATH = 10002
KVX_ERR_UNSUPPORTED = 10003
KVX_ERR_NCCL = 10004

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_SZ = ctypes.c_size_t
_U64 = ctypes.c_uint64

# name -> argtypes (restype is int for every entry point except kvx_strerror)
SIGNATURES = {
    "kvx_version": [],
    "kvx_strerror": [_I],
    "kvx_device_count": [ctypes.POINTER(_I)],
    "kvx_quant_pack": [_P, _P, _I64, _P, _I64, _I64, _I, _I, _I, _I, _P, _P, _P, _I64, _I, _I, _P],
    "kvx_quant_pack_signal": [_P, _P, _I64, _P, _I64, _I64, _I, _I, _I, _I, _P, _P, _P, _I64,
                              _I, _I, _P, _P, _I, _U32, _P, _U32, _P, _P],
    "kvx_dequant_scatter_paged": [_P, _P, _P, _I64, _P, _I64, _I64, _I, _I, _I, _I, _P, _P, _I64,
                                  _I, _I, _P],
    "kvx_pull_dequant_scatter_paged": [_P, _P, _P, _I64, _P, _I64, _I64, _I, _I, _I, _I, _P, _P,
                                       _I64, _I, _I, _P, _U32, _I, _P, _P, _P, _I, _P],
    "kvx_pull_supported": [_I64, _I, _I, _I, _I],
    "kvx_quant_pack_kivi": [_P, _P, _I64, _I64, _I64, _I, _I, _I, _I, _P, _I64, _P, _I64, _P,
                            _I64, _P, _P],
    "kvx_quant_pack_kivi_signal": [_P, _P, _I64, _I64, _I64, _I, _I, _I, _I, _P, _I64, _P, _I64,
                                   _P, _I64, _P, _P, _P, _I, _U32, _P, _U32, _P, _P],
    "kvx_dequant_scatter_paged_kivi": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I64, _I64, _I, _I,
                                       _I, _I, _P, _P, _I64, _P],
    "kvx_pull_dequant_scatter_paged_kivi": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I64, _I64, _I,
                                            _I, _I, _I, _P, _P, _I64, _P, _U32, _I, _P, _P, _P,
                                            _I, _P],
    "kvx_packed_sizes": [_I64, _I, _I, _I, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                         ctypes.POINTER(_I64)],
    "kvx_enable_peer": [_I, _I],
    "kvx_copy_peer": [_P, _I, _P, _I, _SZ, _P],
    "kvx_malloc": [ctypes.POINTER(_P), _SZ],
    "kvx_free": [_P],
    "kvx_memset_async": [_P, _I, _SZ, _P],
    "kvx_ipc_handle_size": [],
    "kvx_ipc_get_handle": [_P, _P],
    "kvx_ipc_open": [_P, ctypes.POINTER(_P)],
    "kvx_ipc_close": [_P],
    "kvx_stream_signal": [_P, _U32, _P],
    "kvx_stream_wait": [_P, _U32, _P],
    "kvx_memcpy_async": [_P, _P, _SZ, _P],
    "kvx_stream_wait_eq": [_P, _U32, _P],
    "kvx_stream_memops_supported": [ctypes.POINTER(_I)],
    "kvx_ctl_alloc": [ctypes.POINTER(_P)],
    "kvx_ctl_free": [_P],
    "kvx_handoff_chunk_plan": [_I64, _I64, _I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)],
    "kvx_pair_create": [_I, _I64, _I64, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I64, _P,
                        ctypes.POINTER(_P)],
    "kvx_pair_send": [_P, _U64, _P, _P, _I64, _P, _I64, _I, _I, _I, _P],
    "kvx_pair_recv": [_P, _U64, _P, _P, _I64, _P, _I64, _I, _I, _I, _P],
    "kvx_pair_recv_many": [_P, _U64, _I, _P, _P, _I64, _P, _P, _I, _I, _I, _P],
    "kvx_nccl_unique_id_size": [],
    "kvx_nccl_get_unique_id": [_P],
    "kvx_nccl_pair_init": [_P, _I, _I, ctypes.POINTER(_P)],
    "kvx_nccl_sendrecv": [_P, _P, _SZ, _I, _P, _SZ, _I, _P],
    "kvx_nccl_pair_destroy": [_P],
    "kvx_pair_destroy": [_P],
}

# constants of include/kvx.h
KVX_KIVI_V_FLAGS = 32
KVX_PULL_PDL, KVX_PULL_CHAINED = 1, 2
KVX_ROLE_PREFILL, KVX_ROLE_DECODE = 0, 1
KVX_PAIR_GATE, KVX_PAIR_PDL, KVX_PAIR_CHAINED = 1, 2, 4
KVX_STATUS_OK, KVX_STATUS_ABORTED, KVX_STATUS_TIMEOUT = 0, 1, 2

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load ``_kvx.so`` (raises if absent: the product has no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or os.environ.get("KVX_LIB") or SO_PATH
        if not os.path.exists(p):
            raise ImportError(
                f"{p} not built: run `python -m paper_2502_09334_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(p)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_char_p if name == "kvx_strerror" else _I
        _lib = L
    return _lib


def strerror(code: int) -> str:
    return load().kvx_strerror(code).decode()


def check(rc: int, what: str = "kvx") -> None:
    if rc == KVX_OK:
        return
    msg = f"{what}: {strerror(rc)} (rc={rc})"
    if rc == KVX_ERR_INVALID_ARG:
        raise ValueError(msg)
    if rc == KVX_ERR_NO_PATH:
        raise NoPath(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
