"""ctypes binding of oracle/kvq_oracle.c (TEST INFRASTRUCTURE ONLY).

Second restatement of the oracle (C, OpenMP).  Used by the tests to cross-check
the numpy oracle and by bench.py as the CPU baseline (``kind: "port"``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libkvq_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "kvq_oracle.c"))
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.kvq_quant_pack.argtypes = [P, I64, I, I, I, P, P, P]
        L.kvq_dequant.argtypes = [P, P, P, I64, I, I, I, P]
        L.kvq_dequant_scatter_paged.argtypes = [P, P, P, P, I64, I64, I, I, I, I, P, P, I64]
        L.kvq_quant_pack_scalar.argtypes = [P, I64, I, I, I, P, P, P]
        L.kvq_dequant_scalar.argtypes = [P, P, P, I64, I, I, I, P]
        L.kvq_threads.argtypes = []
        L.kvq_set_threads.argtypes = [ctypes.c_int]
        # all host threads this process may use (torchrun exports OMP_NUM_THREADS=1)
        L.kvq_set_threads(len(os.sched_getaffinity(0)))
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def threads() -> int:
    return lib().kvq_threads()


def simd() -> bool:
    """True when the library was built with its AVX2/F16C/FMA path."""
    return bool(lib().kvq_simd())


def quant_pack_scalar(x: np.ndarray, bits: int = 4, group: int = 128):
    """The scalar statement of quant_pack (single thread), for SIMD == scalar checks."""
    x = np.ascontiguousarray(x, dtype=np.float16)
    rows, d = x.shape
    ng = d // group
    codes = np.empty((rows, d * bits // 8), np.uint8)
    scale = np.empty((rows, ng), np.float16)
    zero = np.empty((rows, ng), np.float16)
    rc = lib().kvq_quant_pack_scalar(_p(x), rows, d, group, bits, _p(codes), _p(scale), _p(zero))
    if rc:
        raise ValueError(f"kvq_quant_pack_scalar rc={rc}")
    return codes, scale, zero


def unpack_dequant_scalar(codes, scale, zero, bits: int, group: int, head_dim: int):
    out = np.empty((codes.shape[0], head_dim), np.float16)
    rc = lib().kvq_dequant_scalar(_p(np.ascontiguousarray(codes)), _p(np.ascontiguousarray(scale)),
                                  _p(np.ascontiguousarray(zero)), codes.shape[0], head_dim, group,
                                  bits, _p(out))
    if rc:
        raise ValueError(f"kvq_dequant_scalar rc={rc}")
    return out


def quant_pack(x: np.ndarray, bits: int = 4, group: int = 128, out=None):
    """``out=(codes, scale, zero)``: preallocated outputs (bench.py reuses them,
    so the timed loop does not fault fresh pages in on every layer)."""
    x = np.ascontiguousarray(x, dtype=np.float16)
    rows, d = x.shape
    if bits == 16:
        return x.view(np.uint8).reshape(rows, -1).copy(), None, None
    ng = d // group
    if out is not None:
        codes, scale, zero = out
        assert codes.shape == (rows, d * bits // 8) and scale.shape == zero.shape == (rows, ng)
    else:
        codes = np.empty((rows, d * bits // 8), np.uint8)
        scale = np.empty((rows, ng), np.float16)
        zero = np.empty((rows, ng), np.float16)
    rc = lib().kvq_quant_pack(_p(x), rows, d, group, bits, _p(codes), _p(scale), _p(zero))
    if rc:
        raise ValueError(f"kvq_quant_pack rc={rc}")
    return codes, scale, zero


def unpack_dequant(codes, scale, zero, bits: int, group: int, head_dim: int):
    rows = codes.shape[0]
    if bits == 16:
        return np.ascontiguousarray(codes).view(np.float16).reshape(rows, head_dim).copy()
    out = np.empty((rows, head_dim), np.float16)
    rc = lib().kvq_dequant(_p(np.ascontiguousarray(codes)), _p(np.ascontiguousarray(scale)),
                           _p(np.ascontiguousarray(zero)), rows, head_dim, group, bits, _p(out))
    if rc:
        raise ValueError(f"kvq_dequant rc={rc}")
    return out


def dequant_scatter_paged(codes, scale, zero, slots, n_layers, tokens, heads, head_dim, group,
                          bits, k_cache, v_cache):
    assert k_cache.flags.c_contiguous and v_cache.flags.c_contiguous
    layer_stride = k_cache[0].size
    slots = np.ascontiguousarray(slots, dtype=np.int64)
    rc = lib().kvq_dequant_scatter_paged(
        _p(np.ascontiguousarray(codes)), _p(scale) if scale is not None else None,
        _p(zero) if zero is not None else None, _p(slots), n_layers, tokens, heads, head_dim,
        group, bits, _p(k_cache), _p(v_cache), layer_stride)
    if rc:
        raise ValueError(f"kvq_dequant_scatter_paged rc={rc}")
