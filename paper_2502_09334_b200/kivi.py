"""The "kivi" payload format: KIVI-style per-channel key
quantisation with a full-precision residual window.

The paper borrows KIVI's quantisation (``PAPER.md:490-492``); KIVI quantises
keys per channel (outlier channels stay in their own scale) over groups of G
tokens and keeps the tokens that do not fill a group in fp16, values per
token.  This is the accuracy variant of the hand-off: same arithmetic, same
HBM/NVLink layout rules (one segment per layer), kernels in
``csrc/kvx_kivi.cuh``.  Groups never straddle requests: ``seqlens`` gives the
lengths of the requests packed back to back in the batch.
"""
from __future__ import annotations

import os

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .costs import KvPrecision
from .datapath import KVPlanes, _round_up, _stream_ptr

KIVI_GROUPS = (32, 64)


def kivi_groups(seqlens, group: int):
    """(group_starts, residual_tokens) int64 arrays in batch token order."""
    gs, rt, off = [], [], 0
    for n in seqlens:
        n = int(n)
        full = n // group
        gs.extend(off + g * group for g in range(full))
        rt.extend(range(off + full * group, off + n))
        off += n
    return np.asarray(gs, np.int64), np.asarray(rt, np.int64)


@dataclass(frozen=True)
class KiviLayout:
    n_layers: int
    n_heads: int
    head_dim: int
    bits: int
    group: int
    seqlens: tuple

    def __post_init__(self):
        if self.bits not in (4, 8):
            raise ValueError("kivi format supports bits 4 or 8")
        if self.group not in KIVI_GROUPS or self.head_dim % self.group or self.head_dim % 32:
            raise ValueError("kivi group must be 32 or 64 and divide head_dim (multiple of 32)")

    @property
    def n_tokens(self) -> int:
        return int(sum(self.seqlens))

    @property
    def n_groups(self) -> int:
        return sum(int(n) // self.group for n in self.seqlens)

    @property
    def n_residual(self) -> int:
        return self.n_tokens - self.n_groups * self.group

    @property
    def sizes(self):
        """Bytes per layer of Kc, Ks, Kz, Kr, Vc, Vs, Vz."""
        hd = self.n_heads * self.head_dim
        q = self.n_groups * self.group
        return (q * hd * self.bits // 8, self.n_groups * hd * 2, self.n_groups * hd * 2,
                self.n_residual * hd * 2, self.n_tokens * hd * self.bits // 8,
                self.n_tokens * hd // self.group * 2, self.n_tokens * hd // self.group * 2)

    @property
    def offsets(self):
        off, out = 0, []
        for sz in self.sizes:
            out.append(off)
            off += _round_up(sz)
        return tuple(out)

    @property
    def layer_stride(self) -> int:
        return self.offsets[-1] + _round_up(self.sizes[-1])

    @property
    def nbytes(self) -> int:
        return self.layer_stride * self.n_layers

    @property
    def wire_bytes(self) -> int:
        return self.n_layers * sum(self.sizes)

    @property
    def fp16_bytes(self) -> int:
        return self.n_layers * 2 * self.n_tokens * self.n_heads * self.head_dim * 2


@dataclass
class PackedKiviKV:
    layout: KiviLayout
    buffer: torch.Tensor
    base: int
    group_starts: torch.Tensor      # device int64 [n_groups]
    residual_tokens: torch.Tensor   # device int64 [n_residual]

    def part(self, i: int, dtype=torch.uint8) -> torch.Tensor:
        """Sub-array i (0..6 = Kc, Ks, Kz, Kr, Vc, Vs, Vz) of every layer, stacked."""
        lay = self.layout
        off0 = self.base - self.buffer.data_ptr()
        segs = [self.buffer[off0 + l * lay.layer_stride + lay.offsets[i]:
                            off0 + l * lay.layer_stride + lay.offsets[i] + lay.sizes[i]]
                for l in range(lay.n_layers)]
        return torch.stack(segs).view(dtype)


def _offsets_arg(lay: KiviLayout):
    arr = (ctypes.c_int64 * 7)(*lay.offsets)
    return arr


def compress_kivi(kv: torch.Tensor, prec=KvPrecision(4), group_size: int = 32, seqlens=None,
                  stream=None) -> PackedKiviKV:
    """Quantise + pack a dense fp16 [L, 2, T, H, D] KV batch in the kivi format."""
    if not kv.is_cuda:
        raise ValueError("kv must be a CUDA tensor (no CPU path)")
    src = KVPlanes.dense(kv)
    T = kv.shape[2]
    seqlens = tuple(int(n) for n in (seqlens if seqlens is not None else (T,)))
    if sum(seqlens) != T or any(n < 0 for n in seqlens):
        raise ValueError("seqlens must sum to the token count")
    lay = KiviLayout(src.n_layers, src.n_heads, src.head_dim, KvPrecision(
        getattr(prec, "bits", prec)).bits, group_size, seqlens)
    gs, rt = kivi_groups(seqlens, group_size)
    gs_d = torch.from_numpy(gs).to(kv.device)
    rt_d = torch.from_numpy(rt).to(kv.device)
    buf = torch.empty(lay.nbytes + 256, dtype=torch.uint8, device=kv.device)
    base = _round_up(buf.data_ptr())
    k, v = src.ptrs(0)
    _lib.call("kvx_quant_pack_kivi", k, v, src.layer_stride, lay.n_layers, T, lay.n_heads,
              lay.head_dim, group_size, lay.bits, gs_d.data_ptr() if len(gs) else None, len(gs),
              rt_d.data_ptr() if len(rt) else None, len(rt), base, lay.layer_stride,
              _offsets_arg(lay), _stream_ptr(stream))
    return PackedKiviKV(lay, buf, base, gs_d, rt_d)


def decompress_kivi_into_paged(packed: PackedKiviKV, k_cache: torch.Tensor, v_cache: torch.Tensor,
                               slot_mapping: torch.Tensor, stream=None, bulk: bool = False) -> None:
    """Dequantise a kivi payload and scatter it into the paged cache.
    ``bulk``: stage the payload through shared memory with TMA bulk copies
    (the variant for a payload read over NVLink)."""
    dst = KVPlanes.paged(k_cache, v_cache, slot_mapping)
    lay = packed.layout
    if slot_mapping.numel() != lay.n_tokens:
        raise ValueError("slot_mapping length must equal the payload's token count")
    if (dst.n_layers, dst.n_heads, dst.head_dim) != (lay.n_layers, lay.n_heads, lay.head_dim):
        raise ValueError("cache geometry does not match the payload")
    gs = packed.group_starts.to(k_cache.device)
    rdst = dst.slots[packed.residual_tokens.to(k_cache.device)].contiguous()
    k, v = dst.ptrs(0)
    args = (packed.base, lay.layer_stride, _offsets_arg(lay),
            dst.slots_ptr, gs.data_ptr() if gs.numel() else None, gs.numel(),
            rdst.data_ptr() if rdst.numel() else None, rdst.numel(), lay.n_layers,
            lay.n_tokens, lay.n_heads, lay.head_dim, lay.group, lay.bits, k, v,
            dst.layer_stride)
    if bulk:
        _lib.call("kvx_pull_dequant_scatter_paged_kivi", *args, None, 0, 1, None, None, None,
                  0, _stream_ptr(stream))
    else:
        _lib.call("kvx_dequant_scatter_paged_kivi", *args, _stream_ptr(stream))
    if stream is not None:  # temporaries were allocated on the current stream
        gs.record_stream(stream)
        rdst.record_stream(stream)


class KiviHandoff:
    """Reusable single-GPU kivi-format hand-off (K1-kivi then K3-kivi), all
    buffers and index arrays allocated once (bench.py --format kivi)."""

    def __init__(self, kv: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                 slot_mapping: torch.Tensor, prec=KvPrecision(4), group_size: int = 32,
                 seqlens=None):
        self.src = KVPlanes.dense(kv)
        self.dst = KVPlanes.paged(k_cache, v_cache, slot_mapping)
        T = kv.shape[2]
        seqlens = tuple(int(n) for n in (seqlens if seqlens is not None else (T,)))
        self.layout = lay = KiviLayout(self.src.n_layers, self.src.n_heads, self.src.head_dim,
                                       KvPrecision(getattr(prec, "bits", prec)).bits, group_size,
                                       seqlens)
        gs, rt = kivi_groups(seqlens, group_size)
        self.gs = torch.from_numpy(gs).to(kv.device)
        self.rt = torch.from_numpy(rt).to(kv.device)
        self.rdst = self.dst.slots[self.rt].contiguous()
        self.buf = torch.empty(lay.nbytes + 256, dtype=torch.uint8, device=kv.device)
        self.base = _round_up(self.buf.data_ptr())
        self.offs = _offsets_arg(lay)
        self.packed = PackedKiviKV(lay, self.buf, self.base, self.gs, self.rt)
        # decode side: the per-lane kernels, or (A/B, KVX_KIVI_LOCAL_PULL=1)
        # the single bulk-staged kivi pull kernel on the local payload
        self.bulk = os.environ.get("KVX_KIVI_LOCAL_PULL") == "1"

    def run(self, timing: list | None = None) -> None:
        lay, s = self.layout, torch.cuda.current_stream()
        ev = None
        if timing is not None:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(s)
        k, v = self.src.ptrs(0)
        _lib.call("kvx_quant_pack_kivi", k, v, self.src.layer_stride, lay.n_layers, lay.n_tokens,
                  lay.n_heads, lay.head_dim, lay.group, lay.bits,
                  self.gs.data_ptr() if self.gs.numel() else None, self.gs.numel(),
                  self.rt.data_ptr() if self.rt.numel() else None, self.rt.numel(), self.base,
                  lay.layer_stride, self.offs, _stream_ptr(s))
        if ev is not None:
            ev[1].record(s)
        kc, vc = self.dst.ptrs(0)
        args = (self.base, lay.layer_stride, self.offs,
                self.dst.slots_ptr, self.gs.data_ptr() if self.gs.numel() else None,
                self.gs.numel(), self.rdst.data_ptr() if self.rdst.numel() else None,
                self.rdst.numel(), lay.n_layers, lay.n_tokens, lay.n_heads, lay.head_dim,
                lay.group, lay.bits, kc, vc, self.dst.layer_stride)
        if self.bulk:  # the single TMA-staged kivi pull kernel, reading local HBM
            _lib.call("kvx_pull_dequant_scatter_paged_kivi", *args, None, 0, 1, None, None,
                      None, 0, _stream_ptr(s))
        else:
            _lib.call("kvx_dequant_scatter_paged_kivi", *args, _stream_ptr(s))
        if ev is not None:
            ev[2].record(s)
            timing.append({"k1": (ev[0], ev[1]), "k3": (ev[1], ev[2])})
