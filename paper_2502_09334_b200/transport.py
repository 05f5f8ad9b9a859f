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
* the channel pool: at setup every rank exports its staging buffers and its
  doorbell flags with CUDA IPC and maps its partner's (the analogue of the
  paper's pre-built group pool); nothing is allocated per hand-off.
* transports (``mode``):
    "pull" - K1 on P into P's HBM; D's K3-bulk streams the payload over NVLink
             with TMA bulk copies (cp.async.bulk, peer source) into shared
             memory and dequantises straight into D's paged cache.  The
             payload crosses NVLink once and D's HBM sees only the fp16 writes.
    "pull_ldg" - same, but K3 reads the peer payload with per-lane 16-B loads.
    "push" - P's K1 stores the payload straight into D's landing buffer over
             NVLink (fused quantise + transfer); K3 on D reads it locally.
    "copy" - K1 local, copy-engine cudaMemcpyAsync into D's landing buffer,
             K3 local (the non-fused baseline).
    "nccl" - K1 local, torch.distributed (NCCL) send/recv per chunk, K3 local.
* chunk pipeline: layers are cut into chunks and every chunk has a 32-bit
  doorbell in D's memory, so K1 of chunk c+1, the link and K3 of chunk c
  overlap.  In the default "pull" mode ONE K1 launch rings the doorbells from
  the device (fence + st.release.sys over NVLink, by the last warp to finish
  the chunk) and ONE K3-bulk launch waits for them in-kernel (bounded
  ld.acquire polling by its producer warps); its last CTA releases the queue
  queue slot back to P; P waits for that release (in the GPU front-end, and
  again in-kernel) before it reuses the slot.  P's queue holds
  ``ChannelSpec.queue_depth`` slots (default 2; hand-off e uses slot e % Q).
  The flags take constant values per (slot, parity) and are never reset, so
  both ends of a hand-off are single CUDA-graph launches with no memop or
  memset nodes (see PairChannel._parity).  The non-fused paths use stream
  memory operations (cuStreamWriteValue32 / cuStreamWaitValue32) on the same
  doorbells, in the GPU front-end.  No host round trips per chunk.
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

MODES = ("pull", "pull_ldg", "push", "copy", "nccl")
PULL_MODES = ("pull", "pull_ldg")
FLAG_SLOTS = 1024  # 32-bit doorbells per rank (a 4 KB page)
PULL_MAX_CHUNKS = 64
PULL_MAX_QUEUE = 8  # queue slots per pair in the prefill GPU's HBM
PULL_CHUNK_TARGET = 128 << 20  # min fp16 bytes per pull chunk
K1_WARPS_EST = 148 * 2 * 8     # resident K1 warps on a B200 (2 x 256-thread CTAs per SM)


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
    min_chunk_bytes: int = PULL_CHUNK_TARGET  # pull modes: smaller hand-offs use fewer chunks
    format: str = "default"  # "default" (per-token groups) or "kivi" (pull modes only)
    device_doorbells: bool = True  # "pull": K1 itself rings per-chunk doorbells (one launch)
    layerwise: bool = False  # pull: layer-granular chunks (<= 64) for open_send streaming
    # pull: hand-offs the prefill side may queue in its HBM before the decode
    # side has pulled them (PAPER.md:859's KV queues); 2 = double buffering
    queue_depth: int = 2

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


def pull_chunk_plan(n_layers: int, fp16_bytes: int, n_chunks: int, min_chunk_bytes: int):
    """(chunks, layers_per_chunk) of one pull hand-off: at most ``n_chunks``
    uniform layer chunks, none carrying less than ``min_chunk_bytes`` of fp16
    KV -- a short prompt goes as ONE chunk (per-chunk launch and doorbell
    overhead would dominate it).  Both ends derive it from the token count."""
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
# Device buffers exported / imported with CUDA IPC
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
    p = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(handle, len(handle))
    _lib.call("kvx_ipc_open", buf, ctypes.byref(p))
    return int(p.value)


def memops_supported() -> bool:
    v = ctypes.c_int(0)
    _lib.call("kvx_stream_memops_supported", ctypes.byref(v))
    return bool(v.value)


def signal(flag_addr: int, value: int, stream) -> None:
    _lib.call("kvx_stream_signal", flag_addr, value & 0xFFFFFFFF, _stream_ptr(stream))


def wait(flag_addr: int, value: int, stream) -> None:
    _lib.call("kvx_stream_wait", flag_addr, value & 0xFFFFFFFF, _stream_ptr(stream))


def wait_eq(flag_addr: int, value: int, stream) -> None:
    _lib.call("kvx_stream_wait_eq", flag_addr, value & 0xFFFFFFFF, _stream_ptr(stream))


# ---------------------------------------------------------------------------
# The channel
# ---------------------------------------------------------------------------

class PairChannel:
    """One end of a prefill -> decode pair (construct on every rank, collectively).

    prefill end: ``send(src_planes, n_tokens)``; decode end:
    ``recv(dst_planes, n_tokens)``.  Both enqueue asynchronously on the
    channel's stream, ordered after the caller's current stream, and make the
    caller's current stream wait for completion (like a collective's work).
    """

    def __init__(self, spec: ChannelSpec, rank: int, world: int, control_group=None,
                 data_group=None, graphs: bool = True, edge: tuple | None = None):
        """``edge=(prefill_rank, decode_rank)`` overrides the default pairing
        (TP regroups, see TPHandoff).  Construction is collective over the
        control group: ranks outside the edge take part in the handle exchange
        and get an inert channel (``role is None``)."""
        self.spec = spec
        self.rank, self.world = rank, world
        if edge is None:
            self.role, self.pair, self.peer = role_of(rank, world)
        else:
            p, d = edge
            self.pair = p
            self.role = "prefill" if rank == p else "decode" if rank == d else None
            self.peer = d if rank == p else p
            if self.role is None:
                exchange(None, control_group)
                self.graphs, self.flags, self.local_payload = False, None, None
                self.peer_flags = self._peer_payload_map = 0
                return
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.Stream(self.device)    # kernels
        self.cstream = torch.cuda.Stream(self.device)   # copy engine / NCCL
        self.data_group = data_group
        self.epoch = 0
        self.Q = spec.queue_depth if spec.mode in PULL_MODES else 1
        self._prev_ranges = None
        self.chunks = spec.chunks()
        self.lpc = layers_per_chunk(spec.n_layers, spec.n_chunks)
        n_ev = PULL_MAX_CHUNKS if spec.mode in PULL_MODES else len(self.chunks)
        self.k_done = [torch.cuda.Event() for _ in range(n_ev)]
        self.comm_done = [torch.cuda.Event() for _ in range(n_ev)]
        self.xfer = torch.cuda.Stream(self.device)      # host <-> device staging
        self.x_ready = [torch.cuda.Event() for _ in range(n_ev)]
        self.x_done = [torch.cuda.Event() for _ in range(n_ev)]
        mode = spec.mode
        if mode != "nccl" and not memops_supported():
            raise RuntimeError("stream memory operations unavailable: use mode='nccl'")
        # local buffers: doorbells (written by the partner) + payload staging
        self.flags = IpcBuffer(FLAG_SLOTS * 4)
        self.graphs = bool(graphs) and mode in PULL_MODES
        # per queue slot: K1's chunk arrival counters + CTA exit counter, and
        # K3-bulk's done counter (zero between launches) -- per slot, so
        # hand-offs on different slots never share scratch even if the caller
        # issues them from different streams
        self.counters = torch.zeros((self.Q, PULL_MAX_CHUNKS + 1), dtype=torch.int32,
                                    device=self.device)
        self.done_counter = torch.zeros(self.Q, dtype=torch.int32, device=self.device)
        self._graphs, self._seen = {}, set()
        if mode in PULL_MODES:
            if len(self.chunks) > PULL_MAX_CHUNKS:
                raise ValueError(f"pull modes support at most {PULL_MAX_CHUNKS} chunks")
            # every flag starts at 0: every queue slot free for its first
            # use (parity 0), no chunk published (see _parity)
        stage_here = (self.role == "prefill" and mode in ("pull", "pull_ldg", "copy", "nccl")) or (
            self.role == "decode" and mode in ("push", "copy", "nccl"))
        self.local_payload = None
        if stage_here:
            if mode == "nccl":  # NCCL needs a torch tensor
                t = torch.empty(spec.capacity_bytes, dtype=torch.uint8, device=self.device)
                self.local_payload = (t, _round_up(t.data_ptr()))
            else:
                # pull modes keep a queue of Q slots on the prefill side:
                # hand-off e fills slot e % Q while the decode side may still
                # be pulling the previous Q - 1
                b = IpcBuffer(_round_up(spec.capacity_bytes) * self.Q)
                self.local_payload = (b, _round_up(b.ptr))
        mine = {"flags": self.flags.handle()}
        if self.local_payload is not None and mode != "nccl":
            mine["payload"] = self.local_payload[0].handle()
            mine["payload_off"] = self.local_payload[1] - self.local_payload[0].ptr
        allv = exchange(mine, control_group)
        theirs = allv[self.peer]
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

    def _slot(self, e: int) -> int:
        """Queue slot used by hand-off ``e`` (pull modes)."""
        return e % self.Q

    def _half(self, e: int) -> int:
        """Byte offset of the payload slot used by hand-off ``e`` (pull modes)."""
        return (e % self.Q) * _round_up(self.spec.capacity_bytes)

    # pull-mode doorbells are never reset (no lost wake-ups): hand-off e uses
    # queue slot h = e % Q for the u-th time, u = (e - 1) // Q, parity p = u & 1.
    # ready[h][c] lives on D: P sets it to p ^ 1 once chunk c is in slot h.
    # free[h] lives on P: D sets it to p ^ 1 once it has consumed the slot;
    # P's next use of slot h (parity p ^ 1) waits for free[h] == p ^ 1.
    # Each side also keeps p in its own memory (state[h]); the fused kernels
    # read it there and flip it, so their CUDA graphs do not depend on p.
    # The stream-memop paths bake p in (their graphs are keyed by it) and flip
    # state[h] with a memop.
    def _parity(self, e: int) -> int:
        return ((e - 1) // self.Q) & 1

    def _pready(self, base: int, h: int, c: int) -> int:
        return base + 4 * (h * PULL_MAX_CHUNKS + c)

    def _pfree(self, base: int, h: int) -> int:
        return base + 4 * (PULL_MAX_QUEUE * PULL_MAX_CHUNKS + h)

    def _pstate(self, h: int) -> int:
        return self.flags.ptr + 4 * (PULL_MAX_QUEUE * PULL_MAX_CHUNKS + PULL_MAX_QUEUE + h)

    def _fused(self, lay) -> bool:
        """One K1 launch ringing device-side doorbells -> one K3-bulk launch
        waiting on them (both ends decide identically from the layout)."""
        return (self.spec.mode == "pull" and self.spec.device_doorbells and
                pull_supported(lay))

    def _pull_chunks(self, lay):
        if self.spec.layerwise:  # streaming during prefill: publish as layers finish
            n = min(lay.n_layers, PULL_MAX_CHUNKS)
            return layer_chunks(lay.n_layers, n), layers_per_chunk(lay.n_layers, n)
        if self._fused(lay):
            # layer-granular doorbells, but every K1 warp should own several
            # items per chunk (one fence + atomic per warp per chunk)
            cpr = lay.n_heads * lay.head_dim // 32
            items = lay.n_layers * 2 * lay.n_tokens * (-(-cpr // 32))
            n = max(1, min(lay.n_layers, PULL_MAX_CHUNKS, items // (4 * K1_WARPS_EST)))
            return layer_chunks(lay.n_layers, n), layers_per_chunk(lay.n_layers, n)
        return pull_chunk_plan(lay.n_layers, lay.fp16_bytes, self.spec.n_chunks,
                               self.spec.min_chunk_bytes)

    def _wait_half_free(self, h: int, p: int, stream) -> None:
        """Hold the prefill side in the GPU front-end (a stream memop, no SMs
        held) until the decode side has released queue half h.  The fused K1
        re-checks in-kernel, but it must not sit spinning on every SM of a
        prefill GPU that has compute to run while the decode side lags."""
        wait_eq(self._pfree(self.flags.ptr, h), p, stream)

    def _send_pull(self, src, lay, e, s, cur, timing, stage_in):
        h, p = self._slot(e), self._parity(e)
        chunks, lpc = self._pull_chunks(lay)
        key = ("send", lay.n_tokens, h, p, src.k.data_ptr(), src.slots_ptr)
        if self._graph_ok(key, timing, stage_in):
            self._wait_half_free(h, p, cur)
            return self._replay(key, s, cur)
        payload = PackedKV(lay, self.k1_target + self._half(e), self.device)

        fused = self._fused(lay) and stage_in is None
        if fused:
            self._wait_half_free(h, p, cur)  # outside the graph: it depends on p
        # the fused graph reads the parity from device state: valid for both
        keys = [key, key[:3] + (p ^ 1,) + key[4:]] if fused else [key]

        def body():
            if fused:
                # ONE launch: every CTA waits in-kernel for D to be done with
                # this half, then quantises and rings the chunk doorbells
                ev = _kernel_events(timing, s, "k1")
                k, v = src.ptrs(0)
                c0, sc0, z0 = payload.ptrs(0)
                _lib.call("kvx_quant_pack_signal", k, v, src.layer_stride, src.slots_ptr,
                          lay.n_layers, lay.n_tokens, lay.n_heads, lay.head_dim, lay.group,
                          lay.bits, c0, sc0, z0, lay.layer_stride, *src.window_args,
                          self.counters[h].data_ptr(), self._pready(self.peer_flags, h, 0), lpc,
                          self._pfree(self.flags.ptr, h), self._pstate(h), _stream_ptr(s))
                _kernel_events_end(ev, s)
                return
            wait_eq(self._pfree(self.flags.ptr, h), p, s)     # D is done with this half
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
                signal(self._pready(self.peer_flags, h, c), p ^ 1, s)
            signal(self._pstate(h), p ^ 1, s)

        self._run_or_capture(keys, body, s, cur, capturable=timing is None and stage_in is None)
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
        assert self.role == "prefill" and self.spec.mode in PULL_MODES
        return SendSession(self, src, n_tokens)

    def _recv_pull(self, dst, lay, e, s, cur, timing, stage_out):
        h, p = self._slot(e), self._parity(e)
        chunks, lpc = self._pull_chunks(lay)
        key = ("recv", lay.n_tokens, h, p, dst.slots_ptr, dst.k.data_ptr())
        if self._graph_ok(key, timing, stage_out):
            return self._replay(key, s, cur)
        payload = PackedKV(lay, self.k3_source + self._half(e), self.device)
        bulk = self.spec.mode == "pull" and pull_supported(lay)
        keys = [key, key[:3] + (p ^ 1,) + key[4:]] if bulk else [key]

        def body():
            if stage_out is not None:
                for c in range(len(chunks)):
                    s.wait_event(self.x_done[c])
            if bulk:
                # ONE persistent bulk-pull kernel per hand-off: its producer
                # threads wait in-kernel for each chunk's doorbell
                ev = _kernel_events(timing, s, "k3")
                dequant_scatter_layers(payload, dst, 0, lay.n_layers, s,
                                       ready=(self._pready(self.flags.ptr, h, 0), lpc),
                                       done=(self.done_counter[h].data_ptr(),
                                             self._pfree(self.peer_flags, h), self._pstate(h)))
                _kernel_events_end(ev, s)
            else:
                for c, (l0, l1) in enumerate(chunks):
                    wait_eq(self._pready(self.flags.ptr, h, c), p ^ 1, s)
                    ev = _kernel_events(timing, s, "k3")
                    dequant_scatter_layers(payload, dst, l0, l1, s)
                    _kernel_events_end(ev, s)
            if not bulk:  # (the bulk kernel frees the half and flips the parity itself)
                signal(self._pfree(self.peer_flags, h), p ^ 1, s)  # half consumed
                signal(self._pstate(h), p ^ 1, s)
            if stage_out is not None:
                (dk, dv), (hk, hv) = stage_out
                self.x_ready[0].record(s)
                self.xfer.wait_event(self.x_ready[0])
                with torch.cuda.stream(self.xfer):
                    hk.copy_(dk, non_blocking=True)
                    hv.copy_(dv, non_blocking=True)
                for c in range(len(chunks)):
                    self.x_done[c].record(self.xfer)

        self._run_or_capture(keys, body, s, cur, capturable=timing is None and stage_out is None)
        if stage_out is not None:
            cur.wait_stream(self.xfer)

    # ---- kivi format over the pull queue (per-chunk doorbells) ----------------
    def _kivi_common(self, n_tokens, seqlens, e):
        from .kivi import kivi_groups
        seqlens = tuple(int(n) for n in (seqlens if seqlens is not None else (n_tokens,)))
        lay = self.spec.kivi_layout(seqlens)
        if lay.n_tokens != n_tokens:
            raise ValueError("seqlens must sum to n_tokens")
        gs, rt = kivi_groups(seqlens, lay.group)
        chunks, lpc = pull_chunk_plan(lay.n_layers, lay.fp16_bytes, self.spec.n_chunks,
                                      self.spec.min_chunk_bytes)
        self._kivi_lpc = lpc
        return lay, gs, rt, chunks, self._slot(e), self._parity(e)

    def _kivi_index(self, gs, rt, stream):
        """Device copies of a batch's group starts / residual tokens, cached per
        batch shape.  A synchronous upload from pageable memory would make the
        host wait for the channel stream to drain, so a hand-off could never
        be enqueued while the previous one runs."""
        key = (gs.tobytes(), rt.tobytes())
        cache = self.__dict__.setdefault("_kivi_idx", {})
        hit = cache.get(key)
        if hit is None:
            if len(cache) >= 64:
                cache.pop(next(iter(cache)))
            host = torch.from_numpy(np.concatenate([gs, rt]).astype(np.int64)).pin_memory()
            with torch.cuda.stream(stream):
                dev = host.to(self.device, non_blocking=True)
            dev.record_stream(stream)
            hit = cache[key] = (dev[:len(gs)], dev[len(gs):], host)
        return hit[0], hit[1]

    def _send_kivi(self, src, n_tokens, seqlens, e):
        lay, gs, rt, chunks, h, p = self._kivi_common(n_tokens, seqlens, e)
        s, cur = self.stream, torch.cuda.current_stream(self.device)
        s.wait_stream(cur)
        gs_d, rt_d = self._kivi_index(gs, rt, s)
        base = self.k1_target + self._half(e)
        offs = (ctypes.c_int64 * 7)(*lay.offsets)
        wait_eq(self._pfree(self.flags.ptr, h), p, s)
        for c, (l0, l1) in enumerate(chunks):
            k, v = src.ptrs(l0)
            _lib.call("kvx_quant_pack_kivi", k, v, src.layer_stride, l1 - l0, n_tokens,
                      lay.n_heads, lay.head_dim, lay.group, lay.bits,
                      gs_d.data_ptr() if len(gs) else None, len(gs),
                      rt_d.data_ptr() if len(rt) else None, len(rt),
                      base + l0 * lay.layer_stride, lay.layer_stride, offs, _stream_ptr(s))
            signal(self._pready(self.peer_flags, h, c), p ^ 1, s)
        signal(self._pstate(h), p ^ 1, s)
        cur.wait_stream(s)

    def _recv_kivi(self, dst, n_tokens, seqlens, e):
        lay, gs, rt, chunks, h, p = self._kivi_common(n_tokens, seqlens, e)
        s, cur = self.stream, torch.cuda.current_stream(self.device)
        s.wait_stream(cur)
        gs_d, rt_d = self._kivi_index(gs, rt, s)
        with torch.cuda.stream(s):
            rdst = dst.slots[rt_d].contiguous()
        base = self.k3_source + self._half(e)
        offs = (ctypes.c_int64 * 7)(*lay.offsets)

        def args(l0, l1):
            k, v = dst.ptrs(l0)
            return (base + l0 * lay.layer_stride, lay.layer_stride, offs, dst.slots_ptr,
                    gs_d.data_ptr() if len(gs) else None, len(gs),
                    rdst.data_ptr() if rdst.numel() else None, rdst.numel(), l1 - l0,
                    n_tokens, lay.n_heads, lay.head_dim, lay.group, lay.bits, k, v,
                    dst.layer_stride)

        if self.spec.mode == "pull":
            # TMA bulk-staged kernels over the whole hand-off, waiting in-kernel
            # for each chunk's doorbell (a handful of launches per hand-off)
            _lib.call("kvx_pull_dequant_scatter_paged_kivi", *args(0, lay.n_layers),
                      self._pready(self.flags.ptr, h, 0), self._kivi_lpc, self._pstate(h),
                      _stream_ptr(s))
        else:  # "pull_ldg": per-chunk stream waits, per-lane peer loads
            for c, (l0, l1) in enumerate(chunks):
                wait_eq(self._pready(self.flags.ptr, h, c), p ^ 1, s)
                _lib.call("kvx_dequant_scatter_paged_kivi", *args(l0, l1), _stream_ptr(s))
        signal(self._pfree(self.peer_flags, h), p ^ 1, s)
        signal(self._pstate(h), p ^ 1, s)
        rdst.record_stream(s)
        cur.wait_stream(s)

    # ---- CUDA graphs: a hand-off of a given size is one graph launch ----------
    def _graph_ok(self, key, timing, staging) -> bool:
        return self.graphs and timing is None and staging is None and key in self._graphs

    def _replay(self, key, s, cur):
        self._graphs[key].replay()  # graph launches are ordered on the current stream

    def _run_or_capture(self, keys, body, s, cur, capturable: bool):
        """Run ``body`` eagerly the first time, capture it the second time
        (registered under every key in ``keys``), replay it afterwards."""
        s.wait_stream(cur)
        if self.graphs and capturable and any(k in self._seen for k in keys):
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                    body()
            except Exception:  # noqa: BLE001 - capture unsupported here: stay eager
                self.graphs = False
                body()
                cur.wait_stream(s)
                return
            for k in keys:
                self._graphs[k] = g
            cur.wait_stream(s)
            g.replay()
            return
        else:
            body()
            if capturable:
                self._seen.update(keys)  # eager once (attributes, caches), capture next time
        cur.wait_stream(s)

    # flags: slot c = "chunk c of epoch e ready" (written by P into D's flags);
    #        slot FLAG_SLOTS//2 + c = "chunk c of epoch e consumed" (D -> P)
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

    def send(self, src: KVPlanes, n_tokens: int, timing: list | None = None,
             stage_in: tuple | None = None, seqlens=None) -> None:
        """Hand ``src`` to the partner.  ``stage_in=(host_kv, dev_kv)``: upload
        each layer chunk from pinned host memory first (the host-buffer e2e
        path; H2D of chunk c+1 overlaps K1 of chunk c)."""
        assert self.role == "prefill"
        if n_tokens == 0:
            return  # nothing to hand off (both ends skip it: no epoch consumed)
        if timing is None and stage_in is None and self._graphs:
            # fast path: a captured hand-off of this size/half/buffers is ONE
            # graph launch on the caller's stream (no extra stream syncs)
            e = self.epoch + 1
            h, p = self._slot(e), self._parity(e)
            g = self._graphs.get(("send", n_tokens, h, p, src.k.data_ptr(), src.slots_ptr))
            if g is not None:
                self.epoch += 1
                self._wait_half_free(h, p, torch.cuda.current_stream(self.device))
                g.replay()
                return
        if self.spec.format == "kivi":
            self.epoch += 1
            return self._send_kivi(src, n_tokens, seqlens, self.epoch)
        lay = self.spec.layout(n_tokens)
        self.epoch += 1
        e = self.epoch
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
            else:  # nccl
                import torch.distributed as dist
                t = self.local_payload[0]
                off = addr - t.data_ptr()
                with torch.cuda.stream(cs):
                    dist.send(t[off:off + nbytes], self.peer, group=self.data_group)
            self.comm_done[c].record(cs)
        self._prev_ranges = ranges
        cur.wait_stream(s)
        cur.wait_stream(cs)
        if stage_in is not None:
            cur.wait_stream(self.xfer)

    def poll(self) -> bool:
        """Decode end, pull modes: has the prefill side started publishing the
        next hand-off (its first chunk's doorbell rang)?  A host-side check
        (a 4-byte device-to-host read of this GPU's doorbell page) for a
        serving loop that pulls queued KV between decode rounds without
        launching a pull that would wait for an idle prefill side."""
        assert self.role == "decode" and self.spec.mode in PULL_MODES
        e = self.epoch + 1
        h, p = self._slot(e), self._parity(e)
        if getattr(self, "_poll_buf", None) is None:
            self._poll_buf = torch.empty(1, dtype=torch.int32, pin_memory=True)
            self._poll_stream = torch.cuda.Stream(self.device)
        _lib.call("kvx_memcpy_async", self._poll_buf.data_ptr(), self._pready(self.flags.ptr, h, 0),
                  4, _stream_ptr(self._poll_stream))
        self._poll_stream.synchronize()
        return int(self._poll_buf[0]) == (p ^ 1)

    def recv(self, dst: KVPlanes, n_tokens: int, timing: list | None = None,
             stage_out: tuple | None = None, seqlens=None) -> None:
        """Receive into ``dst``.  ``stage_out=((dev_k, dev_v), (host_k, host_v))``:
        download each finished layer chunk of the cache to pinned host memory
        (D2H of chunk c overlaps K3 of chunk c+1)."""
        assert self.role == "decode"
        if n_tokens == 0:
            return
        if timing is None and stage_out is None and self._graphs:
            e = self.epoch + 1
            g = self._graphs.get(("recv", n_tokens, self._slot(e), self._parity(e), dst.slots_ptr,
                                  dst.k.data_ptr()))
            if g is not None:
                self.epoch += 1
                g.replay()
                return
        if self.spec.format == "kivi":
            self.epoch += 1
            return self._recv_kivi(dst, n_tokens, seqlens, self.epoch)
        lay = self.spec.layout(n_tokens)
        self.epoch += 1
        e = self.epoch
        mode = self.spec.mode
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
                import torch.distributed as dist
                g = self._guard(prev, ranges[c])
                if g is not None:
                    cs.wait_event(self.k_done[g])  # landing bytes consumed by K3
                t = self.local_payload[0]
                addr, nbytes = payload.byte_range(l0, l1)
                off = addr - t.data_ptr()
                with torch.cuda.stream(cs):
                    dist.recv(t[off:off + nbytes], self.peer, group=self.data_group)
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

    def close(self):
        """Unmap the partner's buffers and free ours (call after a barrier)."""
        if self.role is None:
            return
        torch.cuda.synchronize(self.device)
        self._graphs, self._seen = {}, set()  # their kernels point at the buffers freed below
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


# ---------------------------------------------------------------------------
# bench.py N > 1
# ---------------------------------------------------------------------------


class SendSession:
    """See PairChannel.open_send."""

    def __init__(self, ch: PairChannel, src: KVPlanes, n_tokens: int):
        self.ch, self.src = ch, src
        self.lay = ch.spec.layout(n_tokens)
        ch.epoch += 1
        self.h, self.p = ch._slot(ch.epoch), ch._parity(ch.epoch)
        self.chunks, _ = ch._pull_chunks(self.lay)
        self.payload = PackedKV(self.lay, ch.k1_target + ch._half(ch.epoch), ch.device)
        self.next = 0
        s = ch.stream
        s.wait_stream(torch.cuda.current_stream(ch.device))
        wait_eq(ch._pfree(ch.flags.ptr, self.h), self.p, s)  # decode side done with this half

    def layers_ready(self, n_layers_done: int) -> None:
        ch, s = self.ch, self.ch.stream
        s.wait_stream(torch.cuda.current_stream(ch.device))  # after the layers' producer
        while self.next < len(self.chunks) and self.chunks[self.next][1] <= n_layers_done:
            l0, l1 = self.chunks[self.next]
            quant_pack_layers(self.src, self.payload, l0, l1, s)
            signal(ch._pready(ch.peer_flags, self.h, self.next), self.p ^ 1, s)
            self.next += 1

    def close(self) -> None:
        self.layers_ready(self.lay.n_layers)
        signal(self.ch._pstate(self.h), self.p ^ 1, self.ch.stream)
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
                 mode: str = "pull", graphs: bool = True):
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
                ch = PairChannel(spec, rank, world, control_group, graphs=graphs,
                                 edge=(pr, dr))
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

    def close(self) -> None:
        for ch, *_ in self.edges:
            ch.close()
