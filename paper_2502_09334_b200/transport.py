"""Multi-process (one process per GPU) prefill -> decode hand-off over NVLink.

The reference models each hand-off as an independent point-to-point delay over
the bottleneck link between the last prefill stage and the first decode stage
(``/root/reference/pkg/src/hetplan/simulate.py:221-235``,
``costs.py:51-65,83-103``); the paper's system pre-builds a pool of
communication groups and has decode replicas pull KV from queues kept in the
prefill replicas' GPU memory (``PAPER.md:859``).  Here:

* pairing: ranks [0, N/2) prefill, [N/2, N) decode, pair
  i -> i + N/2 (1P1D / 2P2D / 4P4D).  Pairs are independent: no collective on
  the data path, NVSwitch gives every pair a full link.
* the channel pool: at setup every rank exports its queue and its doorbell
  page with CUDA IPC and maps its partner's (the analogue of the paper's
  pre-built group pool); nothing is allocated per hand-off.
* transports (``mode``):
    "pull" - K1 on P into P's HBM queue; D's K3-bulk streams the payload over
             NVLink with TMA bulk copies (cp.async.bulk, peer source) into
             shared memory and dequantises straight into D's paged cache.
             The payload crosses NVLink once and D's HBM sees only the fp16
             writes.
    "pull_ldg" - same, but K3 reads the peer payload with per-lane 16-B loads.
    "push" - P's K1 stores the payload straight into D's landing buffer over
             NVLink (fused quantise + transfer); K3 on D reads it locally.
    "copy" - K1 local, copy-engine cudaMemcpyAsync into D's landing buffer,
             K3 local (the non-fused baseline).
    "nccl" - K1 local, an NCCL send/recv per chunk through the C-ABI's NCCL
             pair pool (kvx_nccl_*; a 2-rank communicator per pair), K3 local.
* the default "pull" hand-off is ONE kernel launch per end, issued by the
  native pair object (``kvx_pair_send`` / ``kvx_pair_recv``, include/kvx.h):
  K1 rings per-layer-chunk doorbells in D's memory from the device, D's
  K3-bulk waits for them in-kernel and frees the queue slot in-kernel.  The
  doorbells carry per-slot SEQUENCE NUMBERS (hand-off e uses slot e % Q for
  the v-th time; P waits free >= v - 1 and rings ready = v, D waits
  ready >= v and sets free = v): values only grow, so no flag is ever reset
  and a doorbell left by an earlier, longer use of the slot can never
  satisfy a later wait.  Every launch reads the hand-off's length, slot and
  sequence number from its arguments, so any length and any slot tensor is
  one launch -- no per-shape CUDA graphs, no graph caches.  Consecutive
  pulls are chained with programmatic dependent launch: the next pull
  streams its slot while the previous one drains.  ``recv_many`` drains
  several queued hand-offs with one pull launch (a decode round's pull).
  The prefill end either gates each K1 in the GPU front-end until its slot
  is free (``gate_send``) or, in latency mode, chains the K1s with PDL.
* the kivi format: one fused prefill call ringing K and V chunk doorbells
  in-kernel, one pull kernel for K groups, V rows and residual rows.
* the other paths (pull_ldg, host doorbells, layer-wise streaming, host
  staging) use stream memory operations (cuStreamWriteValue32 /
  cuStreamWaitValue32 GEQ) on the same doorbells, in the GPU front-end.
* failure: every in-kernel wait is bounded by the channel's timeout and can
  be aborted from the host (``PairChannel.abort``); the kernels then record
  the reason in a host-mapped control block and exit, and the channel raises
  PartnerLost (a NoPath) -- no trap, no lost CUDA context.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
from dataclasses import dataclass

import torch

from . import _lib
from .costs import DEFAULT_GROUP, KvPrecision
from .datapath import (KVPlanes, PackedKV, PackedLayout, _round_up, _stream_ptr,
                       dequant_scatter_layers, layer_chunks, layers_per_chunk, pull_supported,
                       quant_pack_layers)
from .errors import PartnerLost

MODES = ("pull", "pull_ldg", "push", "copy", "nccl")
PULL_MODES = ("pull", "pull_ldg")
FLAG_SLOTS = 1024  # 32-bit doorbells per rank (a 4 KB page)
PULL_MAX_CHUNKS = 64
PULL_MAX_QUEUE = 8  # queue slots per pair in the prefill GPU's HBM
PULL_CHUNK_TARGET = 128 << 20  # min fp16 bytes per pull chunk (non-fused paths)
# abort(): the local doorbells are set to this value -- above any sequence
# number a wait can ask for (< 2^28 uses per slot), so every pending wait is
# released, and the kernels read a jump of >= 2^29 as "aborted"
POISON = 0x60000000
DEFAULT_TIMEOUT_S = 60.0


# ---------------------------------------------------------------------------
# Host-side plan (pure Python: unit-tested with gloo on CPU)
# ---------------------------------------------------------------------------

def pairing(world: int):
    """[(prefill_rank, decode_rank)] for N = 2, 4, 8 ... (pair i -> i + N/2)."""
    if world < 2 or world % 2:
        raise ValueError("the hand-off pairs prefill and decode ranks: world must be even >= 2")
    h = world // 2
    return [(i, i + h) for i in range(h)]


def role_of(rank: int, world: int):
    """('prefill'|'decode', pair index, partner rank)."""
    for i, (p, d) in enumerate(pairing(world)):
        if rank == p:
            return "prefill", i, d
        if rank == d:
            return "decode", i, p
    raise ValueError(f"rank {rank} outside world {world}")


def seq_of(e: int, Q: int):
    """(queue slot, sequence number) of hand-off ``e`` (1, 2, ...): slot
    e % Q, used for the v-th time (include/kvx.h, the sequence protocol)."""
    return e % Q, (e - 1) // Q + 1


@dataclass(frozen=True)
class ChannelSpec:
    """What both ends of a pair must agree on (capacity, format, chunking)."""

    n_layers: int
    max_tokens: int
    n_heads: int
    head_dim: int
    bits: int = 4
    group: int = DEFAULT_GROUP
    n_chunks: int = 8
    mode: str = "pull"
    min_chunk_bytes: int = PULL_CHUNK_TARGET  # non-fused pull paths: fewer chunks when short
    format: str = "default"  # "default" (per-token groups) or "kivi" (pull modes only)
    device_doorbells: bool = True  # "pull": K1 itself rings per-chunk doorbells (one launch)
    layerwise: bool = False  # pull: layer-granular chunks (<= 64) for open_send streaming
    # pull: hand-offs the prefill side may queue in its HBM before the decode
    # side has pulled them (PAPER.md:859's KV queues); 2 = double buffering
    queue_depth: int = 2
    # fused pull: hold the prefill launch in the GPU front-end until the slot
    # is free (no SMs held while the decode side lags) / the decode launch
    # until the first chunk is published (no pull sitting on the SMs while
    # the prefill side is idle; costs one launch latency per hand-off --
    # serving loops can poll() instead)
    gate_send: bool = True
    gate_recv: bool = False
    pdl: bool = True  # fused pull: chain consecutive pulls (programmatic dependent launch)
    timeout_s: float = DEFAULT_TIMEOUT_S  # bound of every in-kernel doorbell wait

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        KvPrecision(self.bits)
        if self.n_chunks < 1 or self.n_chunks > FLAG_SLOTS // 4:
            raise ValueError("n_chunks out of range")
        if not 1 <= self.queue_depth <= PULL_MAX_QUEUE:
            raise ValueError(f"queue_depth must be in [1, {PULL_MAX_QUEUE}]")
        if self.format not in ("default", "kivi"):
            raise ValueError("format must be 'default' or 'kivi'")
        if self.format == "kivi" and self.mode not in PULL_MODES:
            raise ValueError("the kivi format is carried by the pull modes")
        if self.n_layers < 1 or self.max_tokens < 1 or self.n_heads < 1:
            raise ValueError("n_layers, max_tokens and n_heads must be >= 1")
        if not self.timeout_s > 0:
            raise ValueError("timeout_s must be > 0")

    def layout(self, n_tokens: int) -> PackedLayout:
        if not 0 <= n_tokens <= self.max_tokens:
            raise ValueError("n_tokens exceeds the channel capacity")
        return PackedLayout(self.n_layers, n_tokens, self.n_heads, self.head_dim, self.bits,
                            self.group)

    def kivi_layout(self, seqlens):
        from .kivi import KiviLayout
        lay = KiviLayout(self.n_layers, self.n_heads, self.head_dim, self.bits, self.group,
                         tuple(int(n) for n in seqlens))
        if lay.n_tokens > self.max_tokens:
            raise ValueError("n_tokens exceeds the channel capacity")
        return lay

    @property
    def capacity_bytes(self) -> int:
        if self.format == "kivi":
            # worst case: every token in the fp16 residual window
            hd = self.n_heads * self.head_dim
            per_layer = (_round_up(self.max_tokens * hd * 2) + _round_up(
                self.max_tokens * hd * self.bits // 8) + 2 * _round_up(
                self.max_tokens * hd // self.group * 2) + 4 * 256 + _round_up(
                self.max_tokens * hd * 2 // self.group))
            return per_layer * self.n_layers + 256
        return self.layout(self.max_tokens).nbytes + 256

    def chunks(self):
        return layer_chunks(self.n_layers, self.n_chunks)

    def check_planes(self, planes: KVPlanes, n_tokens: int, what: str) -> None:
        """The caller's planes must match the channel: the kernels index
        n_layers layers, n_heads heads of head_dim, and slots[t] for every
        t < n_tokens (ValueError otherwise, like decompress_into_paged)."""
        if (planes.n_layers, planes.n_heads, planes.head_dim) != (
                self.n_layers, self.n_heads, self.head_dim):
            raise ValueError(f"{what} geometry (L={planes.n_layers}, H={planes.n_heads}, "
                             f"D={planes.head_dim}) does not match the channel "
                             f"(L={self.n_layers}, H={self.n_heads}, D={self.head_dim})")
        if planes.k.dtype != torch.float16 or planes.v.dtype != torch.float16:
            raise ValueError(f"{what} planes must be fp16")
        if planes.slots is not None and planes.slots.numel() < n_tokens:
            raise ValueError(f"{what} slot mapping has {planes.slots.numel()} entries "
                             f"for {n_tokens} tokens")
        if not 0 <= n_tokens <= self.max_tokens:
            raise ValueError("n_tokens exceeds the channel capacity")


def handoff_chunk_plan(n_layers: int, n_tokens: int, n_heads: int, head_dim: int,
                       layerwise: bool = False):
    """(chunks, layers_per_chunk) of a fused pull hand-off: the native plan
    (kvx_handoff_chunk_plan) both ends derive from the token count."""
    lpc, nc = ctypes.c_int(0), ctypes.c_int(0)
    _lib.call("kvx_handoff_chunk_plan", n_layers, n_tokens, n_heads, head_dim, int(layerwise),
              ctypes.byref(lpc), ctypes.byref(nc))
    return layer_chunks(n_layers, nc.value), lpc.value


def pull_chunk_plan(n_layers: int, fp16_bytes: int, n_chunks: int, min_chunk_bytes: int):
    """(chunks, layers_per_chunk) of a non-fused pull hand-off: at most
    ``n_chunks`` uniform layer chunks, none carrying less than
    ``min_chunk_bytes`` of fp16 KV -- a short prompt goes as ONE chunk
    (per-chunk launch and doorbell overhead would dominate it).  Both ends
    derive it from the token count."""
    want = max(1, -(-int(fp16_bytes) // max(1, int(min_chunk_bytes))))
    n = max(1, min(int(n_chunks), want))
    return layer_chunks(n_layers, n), layers_per_chunk(n_layers, n)


def exchange(obj, group=None):
    """all_gather_object over the control group (gloo)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


# ---------------------------------------------------------------------------
# Device buffers exported / imported with CUDA IPC; the control block
# ---------------------------------------------------------------------------

class IpcBuffer:
    """A kvx_malloc'd device buffer that can be mapped by another process."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _lib.call("kvx_malloc", ctypes.byref(p), int(nbytes))
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)
        _lib.call("kvx_memset_async", self.ptr, 0, self.nbytes, None)
        torch.cuda.synchronize()

    def handle(self) -> bytes:
        n = _lib.load().kvx_ipc_handle_size()
        buf = ctypes.create_string_buffer(n)
        _lib.call("kvx_ipc_get_handle", self.ptr, buf)
        return buf.raw

    def free(self):
        if self.ptr:
            _lib.call("kvx_free", self.ptr)
            self.ptr = 0


def ipc_open(handle: bytes) -> int:
    """Map a partner's buffer (NoPath if this GPU cannot reach it)."""
    p = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(handle, len(handle))
    _lib.call("kvx_ipc_open", buf, ctypes.byref(p))
    return int(p.value)


class Ctl:
    """A channel's host-mapped control block (kvx.h ``kvx_ctl``): abort word,
    status written by the kernels, timeout of their waits."""

    class _S(ctypes.Structure):
        _fields_ = [("abort", ctypes.c_uint32), ("status", ctypes.c_uint32),
                    ("timeout_ns", ctypes.c_uint64)]

    def __init__(self, timeout_s: float = DEFAULT_TIMEOUT_S):
        p = ctypes.c_void_p()
        _lib.call("kvx_ctl_alloc", ctypes.byref(p))
        self.ptr = int(p.value)
        self.s = self._S.from_address(self.ptr)
        self.s.timeout_ns = int(timeout_s * 1e9)

    @property
    def status(self) -> int:
        return int(self.s.status)

    def abort(self) -> None:
        self.s.abort = 1

    def free(self) -> None:
        if self.ptr:
            self.s = None
            _lib.call("kvx_ctl_free", self.ptr)
            self.ptr = 0


def memops_supported() -> bool:
    v = ctypes.c_int(0)
    _lib.call("kvx_stream_memops_supported", ctypes.byref(v))
    return bool(v.value)


def signal(flag_addr: int, value: int, stream) -> None:
    _lib.call("kvx_stream_signal", flag_addr, value & 0xFFFFFFFF, _stream_ptr(stream))


def wait(flag_addr: int, value: int, stream) -> None:
    """GPU front-end wait until the doorbell's sequence number reaches
    ``value`` (wrap-safe GEQ)."""
    _lib.call("kvx_stream_wait", flag_addr, value & 0xFFFFFFFF, _stream_ptr(stream))


def wait_eq(flag_addr: int, value: int, stream) -> None:
    _lib.call("kvx_stream_wait_eq", flag_addr, value & 0xFFFFFFFF, _stream_ptr(stream))


# ---------------------------------------------------------------------------
# The channel
# ---------------------------------------------------------------------------

class PairChannel:
    """One end of a prefill -> decode pair (construct on every rank, collectively).

    prefill end: ``send(src_planes, n_tokens)``; decode end:
    ``recv(dst_planes, n_tokens)``.  Both are asynchronous and ordered on the
    caller's current stream (the default fused pull launches there; the other
    paths run on the channel's streams, after the current stream, and make it
    wait for them), like a collective's work.
    """

    def __init__(self, spec: ChannelSpec, rank: int, world: int, control_group=None,
                 data_group=None, edge: tuple | None = None):
        """``edge=(prefill_rank, decode_rank)`` overrides the default pairing
        (TP regroups, see TPHandoff).  Construction is collective over the
        control group: ranks outside the edge take part in the handle exchange
        and get an inert channel (``role is None``).  ``data_group`` is
        accepted for round-1 callers and unused: the "nccl" mode builds its
        own 2-rank communicator through the C-ABI."""
        self.spec = spec
        self.rank, self.world = rank, world
        self._pair = None
        self.ctl = None
        if edge is None:
            self.role, self.pair, self.peer = role_of(rank, world)
        else:
            p, d = edge
            self.pair = p
            self.role = "prefill" if rank == p else "decode" if rank == d else None
            self.peer = d if rank == p else p
            if self.role is None:
                exchange(None, control_group)
                self.flags, self.local_payload = None, None
                self.peer_flags = self._peer_payload_map = 0
                return
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.Stream(self.device)    # kernels (non-fused paths)
        self.cstream = torch.cuda.Stream(self.device)   # copy engine / NCCL
        self.epoch = 0
        self.Q = spec.queue_depth if spec.mode in PULL_MODES else 1
        self._prev_ranges = None
        self.chunks = spec.chunks()
        n_ev = PULL_MAX_CHUNKS if spec.mode in PULL_MODES else len(self.chunks)
        self.k_done = [torch.cuda.Event() for _ in range(n_ev)]
        self.comm_done = [torch.cuda.Event() for _ in range(n_ev)]
        self.xfer = torch.cuda.Stream(self.device)      # host <-> device staging
        self.x_ready = [torch.cuda.Event() for _ in range(n_ev)]
        self.x_done = [torch.cuda.Event() for _ in range(n_ev)]
        mode = spec.mode
        if mode != "nccl" and not memops_supported():
            raise RuntimeError("stream memory operations unavailable: use mode='nccl'")
        self.ctl = Ctl(spec.timeout_s)
        # local buffers: doorbells (written by the partner) + payload staging
        self.flags = IpcBuffer(FLAG_SLOTS * 4)
        stage_here = (self.role == "prefill" and mode in ("pull", "pull_ldg", "copy", "nccl")) or (
            self.role == "decode" and mode in ("push", "copy", "nccl"))
        self.local_payload = None
        self.slot_bytes = _round_up(spec.capacity_bytes)
        if stage_here:
            if mode == "nccl":  # the NCCL staging buffer (no IPC export needed)
                t = torch.empty(spec.capacity_bytes, dtype=torch.uint8, device=self.device)
                self.local_payload = (t, _round_up(t.data_ptr()))
            else:
                # pull modes keep a queue of Q slots on the prefill side:
                # hand-off e fills slot e % Q while the decode side may still
                # be pulling the previous Q - 1
                b = IpcBuffer(self.slot_bytes * self.Q + 256)
                self.local_payload = (b, _round_up(b.ptr))
        mine = {"flags": self.flags.handle()}
        if mode == "nccl" and self.role == "prefill":
            # a 2-rank NCCL communicator per pair, built through the C-ABI
            # (kvx_nccl_*: the paper's pre-built NCCL groups)
            uid = ctypes.create_string_buffer(_lib.load().kvx_nccl_unique_id_size())
            _lib.call("kvx_nccl_get_unique_id", uid)
            mine["nccl_id"] = uid.raw
        if self.local_payload is not None and mode != "nccl":
            mine["payload"] = self.local_payload[0].handle()
            mine["payload_off"] = self.local_payload[1] - self.local_payload[0].ptr
        allv = exchange(mine, control_group)
        theirs = allv[self.peer]
        self._nccl = None
        if mode == "nccl":
            uid = mine["nccl_id"] if self.role == "prefill" else theirs["nccl_id"]
            comm = ctypes.c_void_p()
            _lib.call("kvx_nccl_pair_init", ctypes.create_string_buffer(uid, len(uid)), 2,
                      0 if self.role == "prefill" else 1, ctypes.byref(comm))
            self._nccl = comm.value
        self.peer_flags = ipc_open(theirs["flags"])
        self.peer_payload = None
        self._peer_payload_map = 0
        if "payload" in theirs:
            self._peer_payload_map = ipc_open(theirs["payload"])
            self.peer_payload = self._peer_payload_map + theirs["payload_off"]
        # where K1 writes / K3 reads
        if self.role == "prefill":
            self.k1_target = self.peer_payload if mode == "push" else self.local_payload[1]
        else:
            self.k3_source = (self.peer_payload if mode in ("pull", "pull_ldg")
                              else self.local_payload[1])
        if mode in PULL_MODES and spec.format == "default" and spec.bits != 16:
            # the native end of the pair: the fused hand-off is one launch
            queue = self.local_payload[1] if self.role == "prefill" else self.k3_source
            h = ctypes.c_void_p()
            _lib.call("kvx_pair_create",
                      _lib.KVX_ROLE_PREFILL if self.role == "prefill" else _lib.KVX_ROLE_DECODE,
                      spec.n_layers, spec.max_tokens, spec.n_heads, spec.head_dim, spec.bits,
                      spec.group, self.Q, int(spec.layerwise), self.flags.ptr, self.peer_flags,
                      queue, self.slot_bytes, self.ctl.ptr, ctypes.byref(h))
            self._pair = h.value
            self._pair_send, self._pair_recv = _pair_calls()
            # the front-end slot gate, or (latency mode) K1s chained with PDL
            # that wait for the slot in-kernel
            self._send_flags = (_lib.KVX_PAIR_GATE if spec.gate_send else
                                _lib.KVX_PAIR_PDL if spec.pdl else 0)
            self._recv_flags = ((_lib.KVX_PAIR_GATE if spec.gate_recv else 0) |
                                (_lib.KVX_PAIR_PDL if spec.pdl else 0))

    # ---- doorbell page: ready[h][c] at h*64 + c, free[h] at 512 + h --------
    def _seq(self, e: int):
        return seq_of(e, self.Q)

    def _half(self, e: int) -> int:
        """Byte offset of the queue slot used by hand-off ``e`` (pull modes)."""
        return (e % self.Q) * self.slot_bytes

    def _pready(self, base: int, h: int, c: int) -> int:
        return base + 4 * (h * PULL_MAX_CHUNKS + c)

    def _pfree(self, base: int, h: int) -> int:
        return base + 4 * (PULL_MAX_QUEUE * PULL_MAX_CHUNKS + h)

    def _fused(self, lay) -> bool:
        """One K1 launch ringing device-side doorbells -> one K3-bulk launch
        waiting on them (both ends decide identically from the layout)."""
        return (self._pair is not None and self.spec.mode == "pull" and
                self.spec.device_doorbells and pull_supported(lay))

    def _fused_n(self, n_tokens: int) -> bool:
        """``_fused`` by token count, memoised: the per-hand-off host path of
        the fused pull does no layout arithmetic or library query."""
        memo = self.__dict__.setdefault("_fused_memo", {})
        f = memo.get(n_tokens)
        if f is None:
            if len(memo) >= 4096:
                memo.clear()
            f = memo[n_tokens] = self._fused(self.spec.layout(n_tokens))
        return f

    def _pull_chunks(self, lay):
        """Chunk plan of a pull hand-off; identical on both ends (it depends
        on the spec and the token count only)."""
        sp = self.spec
        if sp.layerwise or (sp.mode == "pull" and pull_supported(lay)):
            # the plan the native pair (and the in-kernel waits) use
            return handoff_chunk_plan(lay.n_layers, lay.n_tokens, lay.n_heads, lay.head_dim,
                                      sp.layerwise)
        return pull_chunk_plan(lay.n_layers, lay.fp16_bytes, sp.n_chunks, sp.min_chunk_bytes)

    # ---- failure handling ---------------------------------------------------
    def check(self) -> None:
        """Raise PartnerLost if a kernel of this channel gave up waiting
        (aborted, or the partner did not answer within ``spec.timeout_s``).
        Reads the host-mapped status word: no CUDA call, no sync."""
        st = self.ctl.status if self.ctl is not None else 0
        if st:
            why = {_lib.KVX_STATUS_ABORTED: "aborted",
                   _lib.KVX_STATUS_TIMEOUT: f"no answer within {self.spec.timeout_s:g} s"}.get(
                       st, f"status {st}")
            raise PartnerLost(f"rank {self.rank}: hand-off channel with rank {self.peer} "
                              f"lost ({why}); open a new channel")

    def abort(self) -> None:
        """Give up on the partner: every kernel of this channel spinning on a
        doorbell exits (status ABORTED), and every pending GPU front-end wait
        on this rank's doorbells is released (they are set to POISON, which
        the kernels read as an abort) -- no SMs or streams stay blocked, and
        nothing touches the partner's memory.  The channel is dead
        afterwards: check() raises, close() it."""
        if self.ctl is None:
            return
        self.ctl.abort()
        host = torch.full((FLAG_SLOTS,), POISON, dtype=torch.int32).pin_memory()
        side = torch.cuda.Stream(self.device)
        _lib.call("kvx_memcpy_async", self.flags.ptr, host.data_ptr(), FLAG_SLOTS * 4,
                  _stream_ptr(side))
        side.synchronize()

    # ---- prefill side -------------------------------------------------------
    def send(self, src: KVPlanes, n_tokens: int, timing: list | None = None,
             stage_in: tuple | None = None, seqlens=None) -> None:
        """Hand ``src`` to the partner.  ``stage_in=(host_kv, dev_kv)``: upload
        each layer chunk from pinned host memory first (the host-buffer e2e
        path; H2D of chunk c+1 overlaps K1 of chunk c)."""
        if self.role != "prefill":
            raise RuntimeError("send() on the decode end of the channel")
        self.check()
        n_tokens = int(n_tokens)
        self.spec.check_planes(src, n_tokens, "source")
        if n_tokens == 0:
            return  # nothing to hand off (both ends skip it: no epoch consumed)
        if self.spec.format == "kivi":
            self.epoch += 1
            return self._send_kivi(src, n_tokens, seqlens, self.epoch, timing)
        e = self.epoch + 1
        if stage_in is None and self._fused_n(n_tokens):
            # the default path: ONE native launch on the caller's stream
            if timing is None:
                cs = _raw_stream(self.device.index)
                ev = None
            else:
                cur = torch.cuda.current_stream(self.device)
                cs, ev = cur.cuda_stream, _kernel_events(timing, cur, "k1")
            sl = src.slots
            rc = self._pair_send(self._pair, e, src.k.data_ptr(), src.v.data_ptr(),
                                 src.layer_stride, sl.data_ptr() if sl is not None else None,
                                 n_tokens, src.plane_heads or src.n_heads, src.head_offset,
                                 self._send_flags, cs)
            if rc:
                _lib.check(rc, "kvx_pair_send")
            if ev is not None:
                _kernel_events_end(ev, cur)
            self.epoch = e
            return
        self.epoch = e
        lay = self.spec.layout(n_tokens)
        mode = self.spec.mode
        s, cs = self.stream, self.cstream
        cur = torch.cuda.current_stream(self.device)
        if mode in PULL_MODES:
            return self._send_pull(src, lay, e, s, cur, timing, stage_in)
        s.wait_stream(cur)
        payload = PackedKV(lay, self.k1_target, self.device)
        ranges = [(l0 * lay.layer_stride, l1 * lay.layer_stride) for l0, l1 in self.chunks]
        prev = self._prev_ranges
        for c, (l0, l1) in enumerate(self.chunks):
            if stage_in is not None:
                host, devt = stage_in
                self.xfer.wait_event(self.x_done[c])  # K1 of the previous epoch read it
                with torch.cuda.stream(self.xfer):
                    devt[l0:l1].copy_(host[l0:l1], non_blocking=True)
                self.x_ready[c].record(self.xfer)
                s.wait_event(self.x_ready[c])
            g = self._guard(prev, ranges[c])
            if g is not None:
                if mode == "push":
                    # the decode side may still be reading these bytes
                    wait(self._ack(self.flags.ptr, g), e - 1, s)
                else:
                    # local staging still being copied / sent
                    s.wait_event(self.comm_done[g])
            ev = _kernel_events(timing, s, "k1")
            quant_pack_layers(src, payload, l0, l1, s)
            _kernel_events_end(ev, s)
            if stage_in is not None:
                self.x_done[c].record(s)
            addr, nbytes = payload.byte_range(l0, l1)
            if mode == "push":
                signal(self._ready(self.peer_flags, c), e, s)
                continue
            self.k_done[c].record(s)
            cs.wait_event(self.k_done[c])
            if mode == "copy":
                if g is not None:
                    wait(self._ack(self.flags.ptr, g), e - 1, cs)  # D's landing bytes free
                dst = self.peer_payload + (addr - self.k1_target)
                _lib.call("kvx_copy_peer", dst, self.device.index, addr, self.device.index,
                          nbytes, _stream_ptr(cs))
                signal(self._ready(self.peer_flags, c), e, cs)
            else:  # nccl: one ncclSend in a group on the copy stream (kvx_nccl_sendrecv)
                _lib.call("kvx_nccl_sendrecv", self._nccl, addr, nbytes, 1, None, 0, -1,
                          _stream_ptr(cs))
            self.comm_done[c].record(cs)
        self._prev_ranges = ranges
        cur.wait_stream(s)
        cur.wait_stream(cs)
        if stage_in is not None:
            cur.wait_stream(self.xfer)

    def _send_pull(self, src, lay, e, s, cur, timing, stage_in):
        """Non-fused pull send: per-chunk K1 launches + stream-memop doorbells
        (host staging, host doorbells, pull_ldg, shapes the bulk pull cannot
        stage)."""
        h, v = self._seq(e)
        chunks, _ = self._pull_chunks(lay)
        payload = PackedKV(lay, self.k1_target + self._half(e), self.device)
        s.wait_stream(cur)
        if v > 1:
            wait(self._pfree(self.flags.ptr, h), v - 1, s)  # D is done with this slot
        for c, (l0, l1) in enumerate(chunks):
            if stage_in is not None:
                host, devt = stage_in
                self.xfer.wait_event(self.x_done[c])
                with torch.cuda.stream(self.xfer):
                    devt[l0:l1].copy_(host[l0:l1], non_blocking=True)
                self.x_ready[c].record(self.xfer)
                s.wait_event(self.x_ready[c])
            ev = _kernel_events(timing, s, "k1")
            quant_pack_layers(src, payload, l0, l1, s)
            _kernel_events_end(ev, s)
            if stage_in is not None:
                self.x_done[c].record(s)
            signal(self._pready(self.peer_flags, h, c), v, s)
        cur.wait_stream(s)
        if stage_in is not None:
            cur.wait_stream(self.xfer)

    def open_send(self, src: KVPlanes, n_tokens: int) -> "SendSession":
        """Layer-wise hand-off during prefill (pull modes; SURVEY.md 8(f)3,
        PAPER.md:859): returns a session whose ``layers_ready(n)`` quantises
        and publishes every chunk whose layers are all < n, ordered after the
        caller's current stream (the prefill compute that produced them) but
        running on the channel's stream, so it overlaps the next layers'
        compute.  The decode side calls ``recv`` as usual: its one K3-bulk
        launch consumes the chunks as their doorbells ring."""
        if self.role != "prefill" or self.spec.mode not in PULL_MODES:
            raise RuntimeError("open_send needs the prefill end of a pull channel")
        if self.spec.format == "kivi":
            raise ValueError("layer-wise streaming carries the default format only "
                             "(the kivi K groups span a request's tokens, not layers)")
        self.check()
        self.spec.check_planes(src, n_tokens, "source")
        return SendSession(self, src, n_tokens)

    # ---- decode side --------------------------------------------------------
    def poll(self) -> bool:
        """Decode end, pull modes: has the prefill side started publishing the
        next hand-off (its first chunk's doorbell rang)?  A host-side check
        (a 4-byte device-to-host read of this GPU's doorbell page) for a
        serving loop that pulls queued KV between decode rounds without
        launching a pull that would wait for an idle prefill side."""
        if self.role != "decode" or self.spec.mode not in PULL_MODES:
            raise RuntimeError("poll() needs the decode end of a pull channel")
        self.check()
        h, v = self._seq(self.epoch + 1)
        if getattr(self, "_poll_buf", None) is None:
            self._poll_buf = torch.empty(1, dtype=torch.int32, pin_memory=True)
            self._poll_stream = torch.cuda.Stream(self.device)
        _lib.call("kvx_memcpy_async", self._poll_buf.data_ptr(), self._pready(self.flags.ptr, h, 0),
                  4, _stream_ptr(self._poll_stream))
        self._poll_stream.synchronize()
        got = int(self._poll_buf[0]) & 0xFFFFFFFF
        return 0 <= ((got - v) & 0xFFFFFFFF) < (1 << 29)

    def poll_count(self) -> int:
        """Decode end, pull modes: how many of the next hand-offs (at most the
        queue depth) the prefill side has started publishing -- the count a
        decode round hands to ``recv_many``.  One device-to-host read of the
        first-chunk doorbells of every queue slot."""
        if self.role != "decode" or self.spec.mode not in PULL_MODES:
            raise RuntimeError("poll_count() needs the decode end of a pull channel")
        self.check()
        if getattr(self, "_pollq_buf", None) is None:
            self._pollq_buf = torch.empty(PULL_MAX_QUEUE * PULL_MAX_CHUNKS, dtype=torch.int32,
                                          pin_memory=True)
            self._pollq_stream = torch.cuda.Stream(self.device)
        n_words = self.Q * PULL_MAX_CHUNKS
        _lib.call("kvx_memcpy_async", self._pollq_buf.data_ptr(), self._pready(self.flags.ptr, 0, 0),
                  4 * n_words, _stream_ptr(self._pollq_stream))
        self._pollq_stream.synchronize()
        flags = self._pollq_buf[:n_words].tolist()
        n = 0
        for k in range(1, self.Q + 1):  # hand-offs epoch+1, epoch+2, ... in order
            h, v = self._seq(self.epoch + k)
            got = flags[h * PULL_MAX_CHUNKS] & 0xFFFFFFFF
            if not 0 <= ((got - v) & 0xFFFFFFFF) < (1 << 29):
                break
            n += 1
        return n

    def recv(self, dst: KVPlanes, n_tokens: int, timing: list | None = None,
             stage_out: tuple | None = None, seqlens=None, chained: bool = False) -> None:
        """Receive into ``dst``.  ``stage_out=((dev_k, dev_v), (host_k, host_v))``:
        download the decode cache to pinned host memory after the hand-off.
        ``chained`` (fused pull with PDL, default format): the caller promises
        that the previous operation on the current stream is this channel's
        previous ``recv``, and for the whole run of chained recvs since the
        last unchained one, that every slot mapping was ready before the run
        and no two recvs of the run write the same blocks -- the pull then
        writes the cache while earlier pulls drain (kvx.h KVX_PAIR_CHAINED)."""
        if self.role != "decode":
            raise RuntimeError("recv() on the prefill end of the channel")
        self.check()
        n_tokens = int(n_tokens)
        self.spec.check_planes(dst, n_tokens, "destination")
        if n_tokens and dst.slots is None:
            raise ValueError("the decode side needs a slot mapping (paged destination)")
        if n_tokens == 0:
            return
        if self.spec.format == "kivi":
            self.epoch += 1
            return self._recv_kivi(dst, n_tokens, seqlens, self.epoch, timing)
        e = self.epoch + 1
        mode = self.spec.mode
        if stage_out is None and self._fused_n(n_tokens):
            # the default path: ONE native K3-bulk launch on the caller's stream
            if timing is None:
                cs = _raw_stream(self.device.index)
                ev = None
            else:
                cur = torch.cuda.current_stream(self.device)
                cs, ev = cur.cuda_stream, _kernel_events(timing, cur, "k3")
            flags = self._recv_flags
            if chained and flags & _lib.KVX_PAIR_PDL:
                flags |= _lib.KVX_PAIR_CHAINED
            rc = self._pair_recv(self._pair, e, dst.k.data_ptr(), dst.v.data_ptr(),
                                 dst.layer_stride, dst.slots.data_ptr(), n_tokens,
                                 dst.plane_heads or dst.n_heads, dst.head_offset,
                                 flags, cs)
            if rc:
                _lib.check(rc, "kvx_pair_recv")
            if ev is not None:
                _kernel_events_end(ev, cur)
            self.epoch = e
            return
        self.epoch = e
        lay = self.spec.layout(n_tokens)
        s, cs = self.stream, self.cstream
        cur = torch.cuda.current_stream(self.device)
        if mode in PULL_MODES:
            return self._recv_pull(dst, lay, e, s, cur, timing, stage_out)
        s.wait_stream(cur)
        cs.wait_stream(cur)
        payload = PackedKV(lay, self.k3_source, self.device)
        ranges = [(l0 * lay.layer_stride, l1 * lay.layer_stride) for l0, l1 in self.chunks]
        prev = self._prev_ranges
        for c, (l0, l1) in enumerate(self.chunks):
            if mode == "nccl":
                g = self._guard(prev, ranges[c])
                if g is not None:
                    cs.wait_event(self.k_done[g])  # landing bytes consumed by K3
                addr, nbytes = payload.byte_range(l0, l1)
                _lib.call("kvx_nccl_sendrecv", self._nccl, None, 0, -1, addr, nbytes, 0,
                          _stream_ptr(cs))
                self.comm_done[c].record(cs)
                s.wait_event(self.comm_done[c])
            else:
                wait(self._ready(self.flags.ptr, c), e, s)
            if stage_out is not None:
                s.wait_event(self.x_done[c])  # previous epoch's download of these layers
            ev = _kernel_events(timing, s, "k3")
            dequant_scatter_layers(payload, dst, l0, l1, s)
            _kernel_events_end(ev, s)
            if stage_out is not None:
                (dk, dv), (hk, hv) = stage_out
                self.x_ready[c].record(s)
                self.xfer.wait_event(self.x_ready[c])
                with torch.cuda.stream(self.xfer):
                    hk[l0:l1].copy_(dk[l0:l1], non_blocking=True)
                    hv[l0:l1].copy_(dv[l0:l1], non_blocking=True)
                self.x_done[c].record(self.xfer)
            if mode == "nccl":
                self.k_done[c].record(s)
            else:
                signal(self._ack(self.peer_flags, c), e, s)
        self._prev_ranges = ranges
        cur.wait_stream(s)
        cur.wait_stream(cs)
        if stage_out is not None:
            cur.wait_stream(self.xfer)

    def recv_many(self, items, timing: list | None = None) -> None:
        """Decode end, fused pull: receive the next ``len(items)`` hand-offs
        with ONE K3-bulk launch (``kvx_pair_recv_many``) -- the decode side
        draining everything queued after a decode round.
        ``items``: [(dst_planes, n_tokens), ...] in hand-off order, at most the
        queue depth; every destination is the same paged cache (only the slot
        mappings differ).  Hand-offs the bulk pull cannot stage (or any other
        transport) are received one by one instead."""
        if self.role != "decode":
            raise RuntimeError("recv_many() on the prefill end of the channel")
        items = [(d, int(n)) for d, n in items]
        if not items:
            return
        if len(items) > self.Q:
            raise ValueError(f"recv_many: {len(items)} hand-offs > queue depth {self.Q}")
        if self.spec.format == "kivi":
            raise ValueError("recv_many: the kivi format needs each hand-off's seqlens; "
                             "use recv(..., seqlens=...) per hand-off")
        self.check()
        d0 = items[0][0]
        key = (d0.k.data_ptr(), d0.v.data_ptr(), d0.layer_stride, d0.plane_heads or d0.n_heads,
               d0.head_offset)
        batch = True
        for d, n in items:
            self.spec.check_planes(d, n, "destination")
            if d.slots is None:
                raise ValueError("the decode side needs a slot mapping (paged destination)")
            if (d.k.data_ptr(), d.v.data_ptr(), d.layer_stride, d.plane_heads or d.n_heads,
                    d.head_offset) != key:
                raise ValueError("recv_many: every hand-off must land in the same cache")
            batch = batch and n > 0 and self._fused_n(n)
        if not batch:
            for d, n in items:
                self.recv(d, n, timing)
            return
        k = len(items)
        slots = (ctypes.c_void_p * k)(*[d.slots.data_ptr() for d, _ in items])
        ns = (ctypes.c_int64 * k)(*[n for _, n in items])
        if timing is None:
            cs, ev = _raw_stream(self.device.index), None
        else:
            cur = torch.cuda.current_stream(self.device)
            cs, ev = cur.cuda_stream, _kernel_events(timing, cur, "k3")
        e0 = self.epoch + 1
        rc = _lib.load().kvx_pair_recv_many(self._pair, e0, k, d0.k.data_ptr(), d0.v.data_ptr(),
                                            d0.layer_stride, slots, ns, key[3], key[4],
                                            self._recv_flags & _lib.KVX_PAIR_PDL, cs)
        if rc:
            _lib.check(rc, "kvx_pair_recv_many")
        if ev is not None:
            _kernel_events_end(ev, cur)
        self.epoch = e0 + k - 1

    def _recv_pull(self, dst, lay, e, s, cur, timing, stage_out):
        """Pull receive on the channel stream: the bulk kernel with in-kernel
        waits and completion (host staging after it), or per-chunk front-end
        waits + per-lane K3 (pull_ldg, shapes the bulk pull cannot stage)."""
        h, v = self._seq(e)
        chunks, lpc = self._pull_chunks(lay)
        payload = PackedKV(lay, self.k3_source + self._half(e), self.device)
        bulk = self.spec.mode == "pull" and pull_supported(lay)
        s.wait_stream(cur)
        if stage_out is not None:
            s.wait_event(self.x_done[0])  # the previous download read the cache
        if bulk:
            # ONE persistent bulk-pull kernel: its producers wait in-kernel for
            # each chunk's doorbell, its last CTA frees the slot
            ev = _kernel_events(timing, s, "k3")
            dequant_scatter_layers(payload, dst, 0, lay.n_layers, s,
                                   ready=(self._pready(self.flags.ptr, h, 0), v, lpc),
                                   done=(self._done_counter(h), self._pfree(self.peer_flags, h)),
                                   ctl=self.ctl.ptr)
            _kernel_events_end(ev, s)
        else:
            for c, (l0, l1) in enumerate(chunks):
                wait(self._pready(self.flags.ptr, h, c), v, s)
                ev = _kernel_events(timing, s, "k3")
                dequant_scatter_layers(payload, dst, l0, l1, s)
                _kernel_events_end(ev, s)
            signal(self._pfree(self.peer_flags, h), v, s)  # slot consumed
        if stage_out is not None:
            (dk, dv), (hk, hv) = stage_out
            self.x_ready[0].record(s)
            self.xfer.wait_event(self.x_ready[0])
            with torch.cuda.stream(self.xfer):
                hk.copy_(dk, non_blocking=True)
                hv.copy_(dv, non_blocking=True)
            self.x_done[0].record(self.xfer)
        cur.wait_stream(s)
        if stage_out is not None:
            cur.wait_stream(self.xfer)

    def _done_counter(self, h: int) -> int:
        """Device scratch of the Python-launched bulk pull's in-kernel
        completion (per slot, zero between launches; the native pair keeps
        its own)."""
        if getattr(self, "_done", None) is None:
            self._done = torch.zeros(PULL_MAX_QUEUE, dtype=torch.int32, device=self.device)
        return self._done.data_ptr() + 4 * h

    # ---- kivi format over the pull queue (per-chunk doorbells) ----------------
    def _kivi_common(self, n_tokens, seqlens, e):
        from .kivi import kivi_groups
        seqlens = tuple(int(n) for n in (seqlens if seqlens is not None else (n_tokens,)))
        lay = self.spec.kivi_layout(seqlens)
        if lay.n_tokens != n_tokens:
            raise ValueError("seqlens must sum to n_tokens")
        gs, rt = kivi_groups(seqlens, lay.group)
        chunks, lpc = pull_chunk_plan(lay.n_layers, lay.fp16_bytes,
                                      min(self.spec.n_chunks, _lib.KVX_KIVI_V_FLAGS),
                                      self.spec.min_chunk_bytes)
        h, v = self._seq(e)
        return lay, gs, rt, chunks, lpc, h, v

    def _kivi_index(self, gs, rt, stream):
        """Device copies of a batch's group starts / residual tokens, cached per
        batch shape (LRU, 64 entries).  A synchronous upload from pageable
        memory would make the host wait for the channel stream to drain, so a
        hand-off could never be enqueued while the previous one runs."""
        key = (gs.tobytes(), rt.tobytes())
        cache = self.__dict__.setdefault("_kivi_idx", {})
        hit = cache.pop(key, None)
        if hit is None:
            if len(cache) >= 64:
                cache.pop(next(iter(cache)))
            host = torch.from_numpy(np.concatenate([gs, rt]).astype(np.int64)).pin_memory()
            with torch.cuda.stream(stream):
                dev = host.to(self.device, non_blocking=True)
            hit = (dev[:len(gs)], dev[len(gs):], host, dev)
        hit[3].record_stream(stream)  # (re)used on this stream: not freed under it
        cache[key] = hit  # most recently used last
        return hit[0], hit[1]

    def _send_kivi(self, src, n_tokens, seqlens, e, timing=None):
        """The fused kivi prefill side: K per-channel, residual and V
        quantisers over the whole hand-off, ringing the K and V chunk
        doorbells from inside the kernels (kvx_quant_pack_kivi_signal); the
        launches are held in the GPU front-end until the queue slot is free."""
        lay, gs, rt, chunks, lpc, h, v = self._kivi_common(n_tokens, seqlens, e)
        s = torch.cuda.current_stream(self.device)
        gs_d, rt_d = self._kivi_index(gs, rt, s)
        base = self.k1_target + self._half(e)
        offs = (ctypes.c_int64 * 7)(*lay.offsets)
        if getattr(self, "_kivi_cnt", None) is None:  # K and V chunk arrivals per slot
            self._kivi_cnt = torch.zeros((PULL_MAX_QUEUE, 2 * PULL_MAX_CHUNKS), dtype=torch.int32,
                                         device=self.device)
        k, vv = src.ptrs(0)
        ev = _kernel_events(timing, s, "k1")
        _lib.call("kvx_quant_pack_kivi_signal", k, vv, src.layer_stride, lay.n_layers, n_tokens,
                  lay.n_heads, lay.head_dim, lay.group, lay.bits,
                  gs_d.data_ptr() if len(gs) else None, len(gs),
                  rt_d.data_ptr() if len(rt) else None, len(rt),
                  base, lay.layer_stride, offs, self._kivi_cnt[h].data_ptr(),
                  self._pready(self.peer_flags, h, 0), lpc, v,
                  self._pfree(self.flags.ptr, h) if v > 1 else None, v - 1, self.ctl.ptr,
                  s.cuda_stream)
        _kernel_events_end(ev, s)

    def _recv_kivi(self, dst, n_tokens, seqlens, e, timing=None):
        """Kivi decode side on the caller's stream: ONE bulk pull kernel for the
        per-channel K groups, the per-token V rows and the fp16 residual rows,
        waiting in-kernel for the K / V doorbells; its last CTA frees the
        queue slot (no stream memop between hand-offs)."""
        lay, gs, rt, chunks, lpc, h, v = self._kivi_common(n_tokens, seqlens, e)
        cur = torch.cuda.current_stream(self.device)
        gs_d, rt_d = self._kivi_index(gs, rt, cur)
        rdst = dst.slots[rt_d].contiguous() if len(rt) else None
        base = self.k3_source + self._half(e)
        offs = (ctypes.c_int64 * 7)(*lay.offsets)
        cs = cur.cuda_stream

        def args(l0, l1):
            k, vv = dst.ptrs(l0)
            return (base + l0 * lay.layer_stride, lay.layer_stride, offs, dst.slots_ptr,
                    gs_d.data_ptr() if len(gs) else None, len(gs),
                    rdst.data_ptr() if rdst is not None else None, len(rt), l1 - l0,
                    n_tokens, lay.n_heads, lay.head_dim, lay.group, lay.bits, k, vv,
                    dst.layer_stride)

        if self.spec.mode == "pull":
            # TMA bulk-staged kernels over the whole hand-off, waiting in-kernel
            # for each chunk's doorbell
            ev = _kernel_events(timing, cur, "k3")
            # ONE pull kernel (K groups, V rows, residual rows) that frees the
            # slot itself; no PDL (measured slower for the kivi pull: config 3
            # 2,387 vs 2,484 GB/s, profiles/r02_bench/k1default_n2.log)
            _lib.call("kvx_pull_dequant_scatter_paged_kivi", *args(0, lay.n_layers),
                      self._pready(self.flags.ptr, h, 0), v, lpc, self._done_counter(h),
                      self._pfree(self.peer_flags, h), self.ctl.ptr, 0, cs)
            _kernel_events_end(ev, cur)
        else:  # "pull_ldg": per-chunk stream waits, per-lane peer loads
            for c, (l0, l1) in enumerate(chunks):
                # the chunk's V doorbell publishes all of it (K, residual, V)
                wait(self._pready(self.flags.ptr, h, _lib.KVX_KIVI_V_FLAGS + c), v, cur)
                _lib.call("kvx_dequant_scatter_paged_kivi", *args(l0, l1), cs)
            signal(self._pfree(self.peer_flags, h), v, cur)

    # flags of the push / copy / nccl modes: slot c = "chunk c of epoch e
    # ready" (written by P into D's flags); slot FLAG_SLOTS//2 + c = "chunk c
    # of epoch e consumed" (D -> P); values are epochs (GEQ waits)
    def _ready(self, base: int, c: int) -> int:
        return base + 4 * c

    def _ack(self, base: int, c: int) -> int:
        return base + 4 * (FLAG_SLOTS // 2 + c)

    @staticmethod
    def _guard(prev, new_range):
        """Index of the last previous-epoch chunk overlapping ``new_range``
        (chunks complete in order, so waiting for it covers all earlier ones)."""
        if not prev:
            return None
        hits = [i for i, (a, _) in enumerate(prev) if a < new_range[1]]
        return max(hits) if hits else None

    def close(self):
        """Unmap the partner's buffers and free ours (call after a barrier)."""
        if self.role is None:
            return
        if self.ctl is None or not self.ctl.status:
            torch.cuda.synchronize(self.device)
        if self._pair is not None:
            _lib.call("kvx_pair_destroy", self._pair)
            self._pair = None
        if getattr(self, "_nccl", None):
            _lib.call("kvx_nccl_pair_destroy", self._nccl)
            self._nccl = None
        if self.peer_flags:
            _lib.call("kvx_ipc_close", self.peer_flags)
            self.peer_flags = 0
        if self._peer_payload_map:
            _lib.call("kvx_ipc_close", self._peer_payload_map)
            self._peer_payload_map = 0
            self.peer_payload = None
        if self.local_payload is not None and isinstance(self.local_payload[0], IpcBuffer):
            self.local_payload[0].free()
        self.local_payload = None
        self.flags.free()
        if self.ctl is not None:
            self.ctl.free()
            self.ctl = None


def _pair_calls():
    """(send, recv) callables for kvx_pair_send / kvx_pair_recv: the CPython
    fast-call shims (csrc/kvx_fast.c) bound to the loaded library, or its
    ctypes functions when the shim is not built.  Same library, same calls."""
    L = _lib.load()
    try:
        from . import _kvx_fast
    except ImportError:
        return L.kvx_pair_send, L.kvx_pair_recv
    _kvx_fast.bind(ctypes.cast(L.kvx_pair_send, ctypes.c_void_p).value,
                   ctypes.cast(L.kvx_pair_recv, ctypes.c_void_p).value)
    return _kvx_fast.pair_send, _kvx_fast.pair_recv


try:  # the caller's current stream as a raw cudaStream_t (no torch.cuda.Stream object)
    _raw_stream_fn = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover - older torch
    _raw_stream_fn = None


def _raw_stream(device_index: int) -> int:
    if _raw_stream_fn is not None:
        return _raw_stream_fn(device_index)
    return torch.cuda.current_stream(device_index).cuda_stream


def _kernel_events(timing, stream, name):
    if timing is None:
        return None
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    return (timing, name, a, b)


def _kernel_events_end(ev, stream):
    if ev is None:
        return
    timing, name, a, b = ev
    b.record(stream)
    timing.append((name, a, b))


class SendSession:
    """See PairChannel.open_send."""

    def __init__(self, ch: PairChannel, src: KVPlanes, n_tokens: int):
        self.ch, self.src = ch, src
        self.lay = ch.spec.layout(n_tokens)
        ch.epoch += 1
        self.h, self.v = ch._seq(ch.epoch)
        self.chunks, _ = ch._pull_chunks(self.lay)
        self.payload = PackedKV(self.lay, ch.k1_target + ch._half(ch.epoch), ch.device)
        self.next = 0
        s = ch.stream
        s.wait_stream(torch.cuda.current_stream(ch.device))
        if self.v > 1:  # decode side done with this slot's previous use
            wait(ch._pfree(ch.flags.ptr, self.h), self.v - 1, s)

    def layers_ready(self, n_layers_done: int) -> None:
        ch, s = self.ch, self.ch.stream
        s.wait_stream(torch.cuda.current_stream(ch.device))  # after the layers' producer
        while self.next < len(self.chunks) and self.chunks[self.next][1] <= n_layers_done:
            l0, l1 = self.chunks[self.next]
            quant_pack_layers(self.src, self.payload, l0, l1, s)
            signal(ch._pready(ch.peer_flags, self.h, self.next), self.v, s)
            self.next += 1

    def close(self) -> None:
        self.layers_ready(self.lay.n_layers)
        torch.cuda.current_stream(self.ch.device).wait_stream(self.ch.stream)


class TPHandoff:
    """Hand-off between TP-sharded replicas with possibly different TP degrees
    (SURVEY.md 8(e)).  KV heads are split evenly by TP rank on both sides;
    every (prefill rank, decode rank) pair whose head ranges overlap becomes
    one point-to-point edge (a PairChannel over the overlap): the prefill rank
    packs its head window, the decode rank pulls it and scatters it into its
    own head window -- the head-range remap on the pull side, no collective.
    Matched TP degrees reduce to one edge per rank pair.  Construct on every
    rank of the control group (collective)."""

    def __init__(self, n_layers: int, max_tokens: int, n_kv_heads: int, head_dim: int,
                 prefill_ranks, decode_ranks, rank: int, world: int, control_group=None,
                 bits: int = 4, group: int = DEFAULT_GROUP, n_chunks: int = 8,
                 mode: str = "pull"):
        tp_p, tp_d = len(prefill_ranks), len(decode_ranks)
        if n_kv_heads % tp_p or n_kv_heads % tp_d:
            raise ValueError("KV heads must split evenly over both TP groups")
        hp, hd = n_kv_heads // tp_p, n_kv_heads // tp_d
        self.rank = rank
        self.edges = []  # (channel, src window offset, dst window offset, n heads)
        for i, pr in enumerate(prefill_ranks):
            for j, dr in enumerate(decode_ranks):
                a, b = max(i * hp, j * hd), min((i + 1) * hp, (j + 1) * hd)
                if a >= b:
                    continue
                if pr == dr:
                    raise ValueError("a rank cannot hand heads to itself: use datapath.HandoffPlan")
                spec = ChannelSpec(n_layers, max_tokens, b - a, head_dim, bits, group, n_chunks,
                                   mode)
                ch = PairChannel(spec, rank, world, control_group, edge=(pr, dr))
                self.edges.append((ch, a - i * hp, a - j * hd, b - a))

    def send(self, src: KVPlanes, n_tokens: int) -> None:
        """Prefill rank: ``src`` holds this rank's hp heads."""
        for ch, so, _, n in self.edges:
            if ch.role == "prefill":
                ch.send(src.window(so, n), n_tokens)

    def recv(self, dst: KVPlanes, n_tokens: int) -> None:
        """Decode rank: ``dst`` is this rank's paged cache (hd heads per token row)."""
        for ch, _, do, n in self.edges:
            if ch.role == "decode":
                ch.recv(dst.window(do, n), n_tokens)

    def check(self) -> None:
        for ch, *_ in self.edges:
            if ch.role is not None:
                ch.check()

    def close(self) -> None:
        for ch, *_ in self.edges:
            ch.close()
