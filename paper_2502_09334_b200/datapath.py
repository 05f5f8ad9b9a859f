"""Data-path API of the prefill->decode KV hand-off (the layer the reference models).

The reference charges the hand-off as a pure delay
(``/root/reference/pkg/src/hetplan/simulate.py:221-235``, ``costs.py:83-103``);
the paper describes the real path (``PAPER.md:490-493``: quantise + pack on
the prefill replica, transfer, "immediately unpacked and dequantized" on the
decode replica).  This module is that path on B200s:

    compress / compress_paged    K1 quant+pack        (kvx_quant_pack)
    transfer                     NVLink copy-engine   (kvx_copy_peer)
    decompress_into_paged        K3 dequant+scatter   (kvx_dequant_scatter_paged)
    handoff                      all three, layer-chunk pipelined on streams,
                                 with fused push (K1 stores over NVLink) and
                                 fused pull (K3 loads over NVLink) variants

Everything runs through ``_kvx.so``; there is no CPU path.  Errors follow the
reference: ValueError for bad bits/b/s (costs.py:25-26, 98-99), NoPath when two
GPUs cannot reach each other (costs.py:63-64), RuntimeError for CUDA errors.

Packed payload layout (one buffer, one segment per layer, see include/kvx.h):
``[codes(l) | scale(l) | zero(l)]`` for l = 0..L-1, each sub-array 256-B
aligned, so any layer range is one contiguous byte range.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

from . import _lib
from .costs import DEFAULT_GROUP, KvPrecision

_ALIGN = 256

# NVTX ranges around every hand-off stage when KVX_NVTX=1 (for nsys/ncu
# timelines; off by default so the hot path pays nothing).
_NVTX = os.environ.get("KVX_NVTX", "0") == "1"


class nvtx_range:
    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if _NVTX:
            torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *a):
        if _NVTX:
            torch.cuda.nvtx.range_pop()


def _round_up(x: int, a: int = _ALIGN) -> int:
    return (x + a - 1) // a * a


def _bits_of(prec) -> int:
    if isinstance(prec, int):
        return KvPrecision(prec).bits
    return KvPrecision(getattr(prec, "bits")).bits


def _check_group(bits: int, group: int, head_dim: int):
    if head_dim <= 0 or head_dim % 8:
        raise ValueError("head_dim must be a positive multiple of 8")
    if bits == 16:
        return
    if group not in (32, 64, 128) or head_dim % group:
        raise ValueError("group_size must be 32, 64 or 128 and divide head_dim")


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


@dataclass(frozen=True)
class PackedLayout:
    """Byte geometry of a packed payload (per-layer segments)."""

    n_layers: int
    n_tokens: int
    n_heads: int
    head_dim: int
    bits: int
    group: int

    @property
    def rows_per_layer(self) -> int:
        return 2 * self.n_tokens * self.n_heads

    @property
    def codes_bytes(self) -> int:  # per layer
        return self.rows_per_layer * self.head_dim * self.bits // 8

    @property
    def meta_bytes(self) -> int:  # per layer, each of scale / zero
        if self.bits == 16:
            return 0
        return self.rows_per_layer * (self.head_dim // self.group) * 2

    @property
    def scale_offset(self) -> int:
        return _round_up(self.codes_bytes)

    @property
    def zero_offset(self) -> int:
        return self.scale_offset + _round_up(self.meta_bytes)

    @property
    def layer_stride(self) -> int:
        return self.zero_offset + _round_up(self.meta_bytes) if self.bits != 16 else _round_up(
            self.codes_bytes)

    @property
    def nbytes(self) -> int:
        return self.layer_stride * self.n_layers

    @property
    def wire_bytes(self) -> int:
        """Bytes of real payload (codes + scale + zero), excluding alignment pad."""
        return self.n_layers * (self.codes_bytes + 2 * self.meta_bytes)

    @property
    def fp16_bytes(self) -> int:
        """The reference's 16-bit volume 2*b*s*h*2*L (costs.py:102)."""
        return self.n_layers * self.rows_per_layer * self.head_dim * 2


@dataclass
class PackedKV:
    """A packed KV payload living in one device buffer (possibly a peer mapping).

    ``base`` is the device address of layer 0's segment; ``owner`` keeps the
    backing tensor alive when the buffer is torch-allocated."""

    layout: PackedLayout
    base: int
    device: torch.device
    owner: object = field(default=None, repr=False)

    @property
    def bits(self) -> int:
        return self.layout.bits

    @property
    def group(self) -> int:
        return self.layout.group

    def ptrs(self, layer: int = 0):
        """(codes, scale, zero) device addresses of layer ``layer``'s segment."""
        b = self.base + layer * self.layout.layer_stride
        if self.layout.bits == 16:
            return b, None, None
        return b, b + self.layout.scale_offset, b + self.layout.zero_offset

    def byte_range(self, l0: int, l1: int):
        """(address, nbytes) of layers [l0, l1) -- one contiguous range."""
        ls = self.layout.layer_stride
        return self.base + l0 * ls, (l1 - l0) * ls

    # -- host-side views (tests / debugging) --------------------------------
    def _segment(self, layer: int) -> torch.Tensor:
        if not isinstance(self.owner, torch.Tensor):
            raise RuntimeError("views need a torch-owned buffer")
        ls = self.layout.layer_stride
        off = self.base - self.owner.data_ptr()
        return self.owner[off + layer * ls: off + (layer + 1) * ls]

    def codes(self) -> torch.Tensor:
        """uint8 [L, 2, T, H, D*bits/8]"""
        L, lay = self.layout.n_layers, self.layout
        segs = [self._segment(l)[: lay.codes_bytes] for l in range(L)]
        return torch.stack(segs).view(L, 2, lay.n_tokens, lay.n_heads, -1)

    def scale(self) -> torch.Tensor:
        """fp16 [L, 2, T, H, D/G]"""
        lay = self.layout
        segs = [self._segment(l)[lay.scale_offset: lay.scale_offset + lay.meta_bytes]
                for l in range(lay.n_layers)]
        return torch.stack(segs).view(torch.float16).view(lay.n_layers, 2, lay.n_tokens,
                                                          lay.n_heads, -1)

    def zero(self) -> torch.Tensor:
        lay = self.layout
        segs = [self._segment(l)[lay.zero_offset: lay.zero_offset + lay.meta_bytes]
                for l in range(lay.n_layers)]
        return torch.stack(segs).view(torch.float16).view(lay.n_layers, 2, lay.n_tokens,
                                                          lay.n_heads, -1)


def alloc_packed(layout: PackedLayout, device) -> PackedKV:
    buf = torch.empty(layout.nbytes + _ALIGN, dtype=torch.uint8, device=device)
    base = _round_up(buf.data_ptr())
    return PackedKV(layout, base, buf.device, buf)


# ---------------------------------------------------------------------------
# KV sources / destinations: planes + optional slot mapping
# ---------------------------------------------------------------------------

@dataclass
class KVPlanes:
    """K and V planes of every layer: plane(l) = base + l*layer_stride elements;
    token t at pos(t)*H*D with pos = slots[t] (paged) or t (dense)."""

    k: torch.Tensor
    v: torch.Tensor
    layer_stride: int
    n_layers: int
    n_heads: int
    head_dim: int
    slots: torch.Tensor | None = None
    plane_heads: int = 0    # heads per token row of the planes (0 = n_heads)
    head_offset: int = 0    # first head of this window

    def window(self, head_offset: int, n_heads: int) -> "KVPlanes":
        """The same planes restricted to heads [head_offset, head_offset + n_heads)
        (a TP head shard: packed by a prefill rank or filled by a decode rank)."""
        full = self.plane_heads or self.n_heads
        h0 = self.head_offset + head_offset
        if head_offset < 0 or n_heads < 1 or h0 + n_heads > full:
            raise ValueError("head window outside the planes")
        return KVPlanes(self.k, self.v, self.layer_stride, self.n_layers, n_heads,
                        self.head_dim, self.slots, full, h0)

    @property
    def window_args(self):
        return (self.plane_heads or self.n_heads, self.head_offset)

    @staticmethod
    def dense(kv: torch.Tensor) -> "KVPlanes":
        """kv: fp16 [L, 2, T, H, D] contiguous."""
        if kv.dtype != torch.float16 or kv.dim() != 5 or kv.shape[1] != 2:
            raise ValueError("kv must be fp16 [L, 2, T, H, D]")
        if not kv.is_contiguous():
            raise ValueError("kv must be contiguous")
        L, _, T, H, D = kv.shape
        return KVPlanes(kv[:, 0], kv[:, 1], kv.stride(0), L, H, D)

    @staticmethod
    def paged(k_cache: torch.Tensor, v_cache: torch.Tensor, slots: torch.Tensor) -> "KVPlanes":
        """k_cache/v_cache: fp16 [L, num_blocks, block_size, H, D] (vLLM flash
        layout per layer, stacked), same strides; slots: int64 [T]."""
        for c in (k_cache, v_cache):
            if c.dtype != torch.float16 or c.dim() != 5:
                raise ValueError("caches must be fp16 [L, num_blocks, block_size, H, D]")
            if not c[0].is_contiguous():
                raise ValueError("each layer of the cache must be contiguous")
        if k_cache.shape != v_cache.shape or k_cache.stride() != v_cache.stride():
            raise ValueError("k_cache and v_cache must have identical shape and strides")
        if slots.dtype != torch.int64 or slots.dim() != 1:
            raise ValueError("slot_mapping must be int64 [T]")
        if slots.device != k_cache.device:
            raise ValueError("slot_mapping must live on the cache's device")
        L, _, _, H, D = k_cache.shape
        return KVPlanes(k_cache, v_cache, k_cache.stride(0), L, H, D, slots.contiguous())

    def ptrs(self, l0: int = 0):
        off = l0 * self.layer_stride * 2
        return self.k.data_ptr() + off, self.v.data_ptr() + off

    @property
    def slots_ptr(self):
        return self.slots.data_ptr() if self.slots is not None else None

    @property
    def device(self):
        return self.k.device


# ---------------------------------------------------------------------------
# K1 / K3 launches on a layer range (the chunk unit of the pipeline)
# ---------------------------------------------------------------------------

def quant_pack_layers(src: KVPlanes, packed: PackedKV, l0: int, l1: int, stream=None) -> None:
    with nvtx_range(f"kvx.K1 layers[{l0},{l1})"):
        _quant_pack_layers(src, packed, l0, l1, stream)


def _quant_pack_layers(src: KVPlanes, packed: PackedKV, l0: int, l1: int, stream=None) -> None:
    lay = packed.layout
    k, v = src.ptrs(l0)
    c, s, z = packed.ptrs(l0)
    _lib.call("kvx_quant_pack", k, v, src.layer_stride, src.slots_ptr, l1 - l0, lay.n_tokens,
              lay.n_heads, lay.head_dim, lay.group, lay.bits, c, s, z, lay.layer_stride,
              *src.window_args, _stream_ptr(stream))


def dequant_scatter_layers(packed: PackedKV, dst: KVPlanes, l0: int, l1: int,
                           stream=None, bulk: bool = False, ready: tuple | None = None,
                           done: tuple | None = None, ctl: int | None = None,
                           pdl: bool = False, chained: bool = False) -> None:
    """K3 on layers [l0, l1).  ``bulk``: TMA bulk-staged variant (for payloads
    read over NVLink).  ``ready=(flags_addr, value, layers_per_chunk)``: the
    bulk kernel waits in-kernel until each chunk's doorbell reaches ``value``
    (one launch per hand-off).  ``done=(counter_addr, peer_free_addr)``:
    in-kernel completion (the last CTA sets the prefill side's free flag to
    ``value``; see kvx.h for the sequence protocol).  ``ctl``: control block
    (abort / timeout of the waits).  ``pdl``: programmatic dependent launch;
    ``chained`` (with ``pdl``): kvx.h KVX_PULL_CHAINED."""
    with nvtx_range(f"kvx.K3 layers[{l0},{l1})"):
        _dequant_scatter_layers(packed, dst, l0, l1, stream, bulk, ready, done, ctl, pdl,
                                chained)


def _dequant_scatter_layers(packed, dst, l0, l1, stream, bulk, ready, done, ctl, pdl,
                            chained=False) -> None:
    lay = packed.layout
    k, v = dst.ptrs(l0)
    c, s, z = packed.ptrs(l0)
    args = (c, s, z, lay.layer_stride, dst.slots_ptr, l1 - l0, lay.n_tokens, lay.n_heads,
            lay.head_dim, lay.group, lay.bits, k, v, dst.layer_stride, *dst.window_args)
    if bulk or ready is not None:
        rf, rv, lpc = ready if ready is not None else (None, 0, 1)
        dc, pf = done if done is not None else (None, None)
        flags = (_lib.KVX_PULL_PDL | (_lib.KVX_PULL_CHAINED if chained else 0)) if pdl else 0
        _lib.call("kvx_pull_dequant_scatter_paged", *args, rf, rv, lpc, dc, pf, ctl, flags,
                  _stream_ptr(stream))
    else:
        _lib.call("kvx_dequant_scatter_paged", *args, _stream_ptr(stream))


def local_bulk_preferred(lay: PackedLayout) -> bool:
    """Which K3 a LOCAL payload (N=1, the host-buffer path) runs: K3-bulk when
    a token row has at least 64 chunks of 32 elements (the consumer warps then
    amortise each staged span over several chunks per lane), the per-lane K3
    for short rows (a 70B-GQA row of 8 KV heads is 32 chunks: K3-bulk there is
    7-43 % slower).  N=1 sweep, K3 ms, per-lane -> bulk (32 KB stages, spans of
    whole consumer passes): config 2 1.807 -> 1.749, 13B 2.781 -> 2.731, 8-bit
    2.136 -> 1.992, 2-bit 1.740 -> 1.545, 70B-GQA 0.535 -> 0.768
    (profiles/r02_bench/k3_local_geo_n1.log)."""
    return lay.bits != 16 and (lay.n_heads * lay.head_dim) // 32 >= 64 and pull_supported(lay)


def pull_supported(lay: PackedLayout) -> bool:
    return bool(_lib.load().kvx_pull_supported(lay.n_tokens, lay.n_heads, lay.head_dim,
                                                  lay.group, lay.bits))


def _layout_for(src: KVPlanes, n_tokens: int, bits: int, group: int) -> PackedLayout:
    _check_group(bits, group, src.head_dim)
    return PackedLayout(src.n_layers, n_tokens, src.n_heads, src.head_dim, bits,
                        group if bits != 16 else DEFAULT_GROUP)


# ---------------------------------------------------------------------------
# Public API
# ---------------------------------------------------------------------------

def compress(kv: torch.Tensor, prec=KvPrecision(4), group_size: int = DEFAULT_GROUP, *,
             out: PackedKV | None = None, stream=None) -> PackedKV:
    """Quantise + pack a dense fp16 [L, 2, T, H, D] KV tensor on its GPU."""
    if not kv.is_cuda:
        raise ValueError("kv must be a CUDA tensor (no CPU path)")
    src = KVPlanes.dense(kv)
    bits = _bits_of(prec)
    lay = _layout_for(src, kv.shape[2], bits, group_size)
    packed = out if out is not None else alloc_packed(lay, kv.device)
    if packed.layout != lay:
        raise ValueError("out has a different layout")
    quant_pack_layers(src, packed, 0, lay.n_layers, stream)
    return packed


def compress_paged(k_cache: torch.Tensor, v_cache: torch.Tensor, slot_mapping: torch.Tensor,
                   prec=KvPrecision(4), group_size: int = DEFAULT_GROUP, *,
                   out: PackedKV | None = None, stream=None) -> PackedKV:
    """Quantise + pack the tokens ``slot_mapping`` selects from a paged cache
    (the prefill replica's own KV cache, gathered in token order)."""
    src = KVPlanes.paged(k_cache, v_cache, slot_mapping)
    if not k_cache.is_cuda:
        raise ValueError("caches must be CUDA tensors (no CPU path)")
    bits = _bits_of(prec)
    lay = _layout_for(src, slot_mapping.numel(), bits, group_size)
    packed = out if out is not None else alloc_packed(lay, k_cache.device)
    if packed.layout != lay:
        raise ValueError("out has a different layout")
    quant_pack_layers(src, packed, 0, lay.n_layers, stream)
    return packed


def decompress_into_paged(packed: PackedKV, k_cache: torch.Tensor, v_cache: torch.Tensor,
                          slot_mapping: torch.Tensor, *, stream=None, bulk: bool = False) -> None:
    """Unpack + dequantise + scatter into the decode side's paged cache.
    ``packed`` may live on a peer GPU (fused NVLink pull) if peer access is on;
    ``bulk`` selects the TMA bulk-staged kernel (best for peer payloads)."""
    dst = KVPlanes.paged(k_cache, v_cache, slot_mapping)
    lay = packed.layout
    if (dst.n_layers, dst.n_heads, dst.head_dim) != (lay.n_layers, lay.n_heads, lay.head_dim):
        raise ValueError("cache geometry does not match the packed payload")
    if slot_mapping.numel() != lay.n_tokens:
        raise ValueError("slot_mapping length must equal the payload's token count")
    dequant_scatter_layers(packed, dst, 0, lay.n_layers, stream, bulk=bulk)


def enable_peer(dev_a: int, dev_b: int) -> None:
    """Enable NVLink peer access both ways (NoPath if impossible, costs.py:63-64)."""
    _lib.call("kvx_enable_peer", int(dev_a), int(dev_b))


def transfer(packed: PackedKV, dst_device, dst_gpu_ids=None, *, out: PackedKV | None = None,
             stream=None, layers: tuple[int, int] | None = None) -> PackedKV:
    """Copy-engine NVLink transfer of the packed payload (cudaMemcpyPeerAsync;
    the non-fused baseline).

    Two call forms: ``transfer(packed, dst_device)``, or SURVEY 8(b)'s
    ``transfer(packed, src_gpu_ids, dst_gpu_ids)`` with the reference's
    stage GPU lists (``kv_comm_cost``'s ``prefill_gpu_ids`` /
    ``decode_gpu_ids``, costs.py:83): the payload must live on one of the
    source GPUs and goes to the first destination GPU; ``NoPath`` when the two
    cannot reach each other (costs.py:63-64)."""
    if dst_gpu_ids is not None:
        src_ids = [int(i) for i in dst_device]
        dst_ids = [int(i) for i in dst_gpu_ids]
        if not dst_ids:
            raise ValueError("dst_gpu_ids is empty")
        if packed.device.index not in src_ids:
            raise ValueError(f"payload on cuda:{packed.device.index}, not on the source GPUs "
                             f"{src_ids}")
        dst_device = torch.device("cuda", dst_ids[0])
        if dst_device.index != packed.device.index:
            enable_peer(packed.device.index, dst_device.index)  # NoPath if unreachable
    dst_device = torch.device(dst_device)
    if out is None:
        out = alloc_packed(packed.layout, dst_device)
    if out.layout != packed.layout:
        raise ValueError("out has a different layout")
    l0, l1 = layers if layers is not None else (0, packed.layout.n_layers)
    src_addr, n = packed.byte_range(l0, l1)
    dst_addr, _ = out.byte_range(l0, l1)
    _lib.call("kvx_copy_peer", dst_addr, out.device.index, src_addr, packed.device.index, n,
              _stream_ptr(stream))
    return out


def layers_per_chunk(n_layers: int, n_chunks: int) -> int:
    n_chunks = max(1, min(n_chunks, max(n_layers, 1)))
    return max(1, -(-n_layers // n_chunks))


def layer_chunks(n_layers: int, n_chunks: int):
    """Uniform chunks of ceil(L / n_chunks) layers (chunk of layer l = l // lpc,
    the rule the in-kernel doorbell wait uses)."""
    lpc = layers_per_chunk(n_layers, n_chunks)
    return [(l0, min(n_layers, l0 + lpc)) for l0 in range(0, n_layers, lpc)]


class HandoffPlan:
    """Reusable single-process hand-off between two GPUs (or within one GPU).

    mode:
      "copy" - K1 on P -> cudaMemcpyPeerAsync -> K3 on D   (3 streams)
      "push" - K1 on P writes the payload into D's buffer over NVLink -> K3 on D
      "pull" - K1 on P -> K3 on D reads the payload over NVLink
      "local"- P == D: K1 -> K3 on one stream (1-GPU round trip)
    Layers are processed in ``n_chunks`` chunks so K1 of chunk i+1, the link
    and K3 of chunk i overlap; chunk ordering uses CUDA events across devices.
    """

    def __init__(self, src: KVPlanes, dst: KVPlanes, n_tokens: int, prec=KvPrecision(4),
                 group_size: int = DEFAULT_GROUP, mode: str = "pull", n_chunks: int = 8,
                 bulk: bool | None = None, min_chunk_bytes: int = 0):
        self.src, self.dst = src, dst
        self.bits = _bits_of(prec)
        self.layout = _layout_for(src, n_tokens, self.bits, group_size)
        # TMA bulk-staged K3 by default when the payload is read over NVLink;
        # on a local payload (N=1) by row length (local_bulk_preferred); push /
        # copy land the payload on D and keep the per-lane K3
        if bulk is None:
            local = mode == "local" or src.device == dst.device
            bulk = (mode == "pull" and not local) or (local and local_bulk_preferred(self.layout))
        self.bulk = bool(bulk)
        if (dst.n_layers, dst.n_heads, dst.head_dim) != (src.n_layers, src.n_heads, src.head_dim):
            raise ValueError("source and destination KV geometry differ")
        self.p_dev, self.d_dev = src.device, dst.device
        same = self.p_dev == self.d_dev
        if same:
            mode = "local"
        elif mode not in ("copy", "push", "pull"):
            raise ValueError(f"unknown mode {mode!r}")
        else:
            enable_peer(self.p_dev.index, self.d_dev.index)
        self.mode = mode
        if min_chunk_bytes:  # short hand-offs: fewer, larger chunks (launch overhead)
            n_chunks = min(n_chunks, max(1, -(-self.layout.fp16_bytes // min_chunk_bytes)))
        self.chunks = layer_chunks(self.layout.n_layers, n_chunks)
        # push: payload lives on D (K1 writes it remotely); pull/local: on P;
        # copy: one buffer on each side.
        self.p_buf = alloc_packed(self.layout, self.d_dev if mode == "push" else self.p_dev)
        self.d_buf = alloc_packed(self.layout, self.d_dev) if mode == "copy" else self.p_buf
        with torch.cuda.device(self.p_dev):
            self.p_stream = torch.cuda.Stream()
            self.k1_done = [torch.cuda.Event() for _ in self.chunks]
        with torch.cuda.device(self.d_dev):
            self.d_stream = torch.cuda.Stream() if not same else self.p_stream
            self.c_stream = torch.cuda.Stream() if mode == "copy" else None
            self.copy_done = [torch.cuda.Event() for _ in self.chunks]
            self.d_idle = torch.cuda.Event()  # the previous run's last K3 (never recorded: no-op)

    @property
    def packed(self) -> PackedKV:
        return self.d_buf

    def run(self, timing: list | None = None) -> None:
        """Enqueue one hand-off (asynchronous; ordered after the current
        streams of both devices, and the current streams wait for it).

        ``timing``: if a list, per chunk a dict of CUDA event pairs recorded on
        the stream each kernel is launched on ({"k1": (start, end), "k3": ...})."""
        with torch.cuda.device(self.p_dev):
            self.p_stream.wait_stream(torch.cuda.current_stream(self.p_dev))
            if self.d_dev != self.p_dev:
                # write-after-read across devices: this run's K1 (pull/push) or
                # copy must not overwrite the payload buffer while the previous
                # run's K3 (or copy) on the decode side may still read it
                self.p_stream.wait_event(self.d_idle)
        if self.d_dev != self.p_dev:
            with torch.cuda.device(self.d_dev):
                self.d_stream.wait_stream(torch.cuda.current_stream(self.d_dev))
                if self.c_stream is not None:
                    self.c_stream.wait_event(self.d_idle)
        for i, (l0, l1) in enumerate(self.chunks):
            ev = {} if timing is not None else None
            with torch.cuda.device(self.p_dev):
                if ev is not None:
                    ev["k1"] = (torch.cuda.Event(enable_timing=True),
                                torch.cuda.Event(enable_timing=True))
                    ev["k1"][0].record(self.p_stream)
                quant_pack_layers(self.src, self.p_buf, l0, l1, self.p_stream)
                if ev is not None:
                    ev["k1"][1].record(self.p_stream)
                self.k1_done[i].record(self.p_stream)
            with torch.cuda.device(self.d_dev):
                if self.mode == "copy":
                    self.c_stream.wait_event(self.k1_done[i])
                    transfer(self.p_buf, self.d_dev, out=self.d_buf, stream=self.c_stream,
                             layers=(l0, l1))
                    self.copy_done[i].record(self.c_stream)
                    self.d_stream.wait_event(self.copy_done[i])
                elif self.mode != "local":
                    self.d_stream.wait_event(self.k1_done[i])
                if ev is not None:
                    ev["k3"] = (torch.cuda.Event(enable_timing=True),
                                torch.cuda.Event(enable_timing=True))
                    ev["k3"][0].record(self.d_stream)
                dequant_scatter_layers(self.d_buf, self.dst, l0, l1, self.d_stream,
                                       bulk=self.bulk)
                if ev is not None:
                    ev["k3"][1].record(self.d_stream)
                    timing.append(ev)
        with torch.cuda.device(self.d_dev):
            torch.cuda.current_stream(self.d_dev).wait_stream(self.d_stream)
            if self.d_dev != self.p_dev:
                self.d_idle.record(self.d_stream)  # every read of p_buf/d_buf done
        if self.d_dev != self.p_dev:
            with torch.cuda.device(self.p_dev):
                torch.cuda.current_stream(self.p_dev).wait_stream(self.p_stream)


def handoff(kv: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
            slot_mapping: torch.Tensor, prec=KvPrecision(4), group_size: int = DEFAULT_GROUP,
            mode: str = "pull", n_chunks: int = 8) -> PackedKV:
    """Hand a dense fp16 [L, 2, T, H, D] KV tensor on the prefill GPU to the
    paged cache on the decode GPU (compress -> NVLink -> decompress)."""
    src = KVPlanes.dense(kv)
    dst = KVPlanes.paged(k_cache, v_cache, slot_mapping)
    plan = HandoffPlan(src, dst, kv.shape[2], prec, group_size, mode, n_chunks)
    plan.run()
    return plan.packed


def device_count() -> int:
    n = ctypes.c_int(0)
    _lib.call("kvx_device_count", ctypes.byref(n))
    return n.value


class HostHandoff:
    """Host-buffer hand-off through the C-ABI (the e2e path bench.py times).

    The CPU reference path reads fp16 KV from host memory and writes the decode
    paged cache to host memory; this class does the same on one GPU:
    per layer chunk, H2D of the KV (copy engine) -> K1 -> K3 -> D2H of the
    decode cache (second copy engine), three streams overlapping chunk i's
    compute with chunk i+1's upload and chunk i-1's download.  Consecutive
    ``run()`` calls pipeline too: a chunk's upload waits only for the previous
    run's K1 of that chunk, its K3 only for the previous run's download of it,
    so run i+1's first uploads overlap run i's last downloads.  Each run ends
    with the caller's current stream waiting for all of it; the first run also
    starts after the caller's stream (the slot mapping copied at construction).
    Host tensors must be pinned for the copies to be asynchronous.
    """

    def __init__(self, kv_host: torch.Tensor, k_cache_host: torch.Tensor,
                 v_cache_host: torch.Tensor, slot_mapping: torch.Tensor, device,
                 prec=KvPrecision(4), group_size: int = DEFAULT_GROUP, n_chunks: int = 8):
        self.device = torch.device(device)
        self.kv_host, self.kc_host, self.vc_host = kv_host, k_cache_host, v_cache_host
        self.kv = torch.empty(kv_host.shape, dtype=torch.float16, device=self.device)
        # device mirror of the host cache: blocks outside the slot mapping keep
        # the host's contents (they are copied back unchanged)
        self.kc = k_cache_host.to(self.device)
        self.vc = v_cache_host.to(self.device)
        self.slots = slot_mapping.to(self.device)
        self.src = KVPlanes.dense(self.kv)
        self.dst = KVPlanes.paged(self.kc, self.vc, self.slots)
        bits = _bits_of(prec)
        self.layout = _layout_for(self.src, kv_host.shape[2], bits, group_size)
        self.packed = alloc_packed(self.layout, self.device)
        self.bulk = local_bulk_preferred(self.layout)  # K3 variant for the local payload
        self.chunks = layer_chunks(self.layout.n_layers, n_chunks)
        with torch.cuda.device(self.device):
            self.h2d, self.comp, self.d2h = (torch.cuda.Stream() for _ in range(3))
            self.up = [torch.cuda.Event() for _ in self.chunks]
            self.done = [torch.cuda.Event() for _ in self.chunks]
            self.read = [torch.cuda.Event() for _ in self.chunks]  # K1 read kv[chunk]
            self.down = [torch.cuda.Event() for _ in self.chunks]  # D2H read kc/vc[chunk]
        self._runs = 0

    @property
    def h2d_bytes(self) -> int:
        return self.kv_host.numel() * 2

    @property
    def d2h_bytes(self) -> int:
        return (self.kc_host.numel() + self.vc_host.numel()) * 2

    def run(self) -> None:
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream()
            first = self._runs == 0
            if first:
                for s in (self.h2d, self.comp, self.d2h):
                    s.wait_stream(cur)
            for i, (l0, l1) in enumerate(self.chunks):
                if not first:
                    self.h2d.wait_event(self.read[i])  # previous run's K1 read kv[chunk]
                with torch.cuda.stream(self.h2d):
                    self.kv[l0:l1].copy_(self.kv_host[l0:l1], non_blocking=True)
                    self.up[i].record(self.h2d)
                self.comp.wait_event(self.up[i])
                quant_pack_layers(self.src, self.packed, l0, l1, self.comp)
                self.read[i].record(self.comp)
                if not first:
                    self.comp.wait_event(self.down[i])  # previous run's D2H read the cache
                dequant_scatter_layers(self.packed, self.dst, l0, l1, self.comp,
                                       bulk=self.bulk)
                self.done[i].record(self.comp)
                self.d2h.wait_event(self.done[i])
                with torch.cuda.stream(self.d2h):
                    self.kc_host[l0:l1].copy_(self.kc[l0:l1], non_blocking=True)
                    self.vc_host[l0:l1].copy_(self.vc[l0:l1], non_blocking=True)
                    self.down[i].record(self.d2h)
            self._runs += 1
            for s in (self.h2d, self.comp, self.d2h):
                cur.wait_stream(s)
