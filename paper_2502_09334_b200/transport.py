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
* chunk pipeline: layers are cut into chunks; per chunk P signals a 32-bit
  doorbell in D's memory (cuStreamWriteValue32, fenced) and D's stream waits on
  it in the front-end (cuStreamWaitValue32 GEQ epoch), so K1 of chunk c+1, the
  link and K3 of chunk c overlap.  D acks each chunk back into P's memory so
  the next hand-off never overwrites a chunk still being read.  No spinning
  kernels, no host round trips per chunk.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import _lib
from .costs import DEFAULT_GROUP, KvPrecision
from .datapath import (KVPlanes, PackedKV, PackedLayout, _round_up, _stream_ptr,
                       dequant_scatter_layers, layer_chunks, layers_per_chunk, pull_supported,
                       quant_pack_layers)

MODES = ("pull", "pull_ldg", "push", "copy", "nccl")
PULL_MODES = ("pull", "pull_ldg")
FLAG_SLOTS = 256  # 32-bit doorbells per rank
PULL_MAX_CHUNKS = 64
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

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        KvPrecision(self.bits)
        if self.n_chunks < 1 or self.n_chunks > FLAG_SLOTS:
            raise ValueError("n_chunks out of range")
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
                 data_group=None, graphs: bool = True):
        self.spec = spec
        self.rank, self.world = rank, world
        self.role, self.pair, self.peer = role_of(rank, world)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.Stream(self.device)    # kernels
        self.cstream = torch.cuda.Stream(self.device)   # copy engine / NCCL
        self.data_group = data_group
        self.epoch = 0
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
        self.counters = torch.zeros(PULL_MAX_CHUNKS, dtype=torch.int32, device=self.device)
        self._graphs, self._seen = {}, set()
        if mode in PULL_MODES:
            if len(self.chunks) > PULL_MAX_CHUNKS:
                raise ValueError(f"pull modes support at most {PULL_MAX_CHUNKS} chunks")
            if self.role == "prefill":  # both queue halves start free
                one = torch.ones(2, dtype=torch.int32, device=self.device)
                _lib.call("kvx_copy_peer", self._pfree(self.flags.ptr, 0), self.device.index,
                          one.data_ptr(), self.device.index, 8, None)
                torch.cuda.synchronize(self.device)
        stage_here = (self.role == "prefill" and mode in ("pull", "pull_ldg", "copy", "nccl")) or (
            self.role == "decode" and mode in ("push", "copy", "nccl"))
        self.local_payload = None
        if stage_here:
            if mode == "nccl":  # NCCL needs a torch tensor
                t = torch.empty(spec.capacity_bytes, dtype=torch.uint8, device=self.device)
                self.local_payload = (t, _round_up(t.data_ptr()))
            else:
                # pull modes double-buffer the prefill-side queue: hand-off e
                # fills half e % 2 while the decode side may still read e - 1
                halves = 2 if mode in PULL_MODES else 1
                b = IpcBuffer(_round_up(spec.capacity_bytes) * halves)
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

    def _half(self, e: int) -> int:
        """Byte offset of the payload half used by hand-off ``e`` (pull modes)."""
        return (e & 1) * _round_up(self.spec.capacity_bytes)

    # pull-mode doorbells use constant values (0/1) so a hand-off is
    # graph-capturable: ready[h][c] lives on D (set to 1 by P after K1 of
    # chunk c into half h, reset to 0 by D after consuming the half);
    # free[h] lives on P (1 = D is done with half h; P clears it before reuse).
    def _pready(self, base: int, h: int, c: int) -> int:
        return base + 4 * (h * PULL_MAX_CHUNKS + c)

    def _pfree(self, base: int, h: int) -> int:
        return base + 4 * (2 * PULL_MAX_CHUNKS + h)

    def _fused(self, lay) -> bool:
        """One K1 launch ringing device-side doorbells -> one K3-bulk launch
        waiting on them (both ends decide identically from the layout)."""
        return (self.spec.mode == "pull" and self.spec.device_doorbells and
                pull_supported(lay))

    def _pull_chunks(self, lay):
        if self._fused(lay):
            # layer-granular doorbells, but every K1 warp should own several
            # items per chunk (one fence + atomic per warp per chunk)
            cpr = lay.n_heads * lay.head_dim // 32
            items = lay.n_layers * 2 * lay.n_tokens * (-(-cpr // 32))
            n = max(1, min(lay.n_layers, PULL_MAX_CHUNKS, items // (4 * K1_WARPS_EST)))
            return layer_chunks(lay.n_layers, n), layers_per_chunk(lay.n_layers, n)
        return pull_chunk_plan(lay.n_layers, lay.fp16_bytes, self.spec.n_chunks,
                               self.spec.min_chunk_bytes)

    def _send_pull(self, src, lay, e, s, cur, timing, stage_in):
        h = e & 1
        chunks, lpc = self._pull_chunks(lay)
        key = ("send", lay.n_tokens, h, src.k.data_ptr(), src.slots_ptr)
        if self._graph_ok(key, timing, stage_in):
            return self._replay(key, s, cur)
        payload = PackedKV(lay, self.k1_target + self._half(e), self.device)

        fused = self._fused(lay) and stage_in is None

        def body():
            wait(self._pfree(self.flags.ptr, h), 1, s)        # D is done with this half
            signal(self._pfree(self.flags.ptr, h), 0, s)      # claim it
            if fused:
                ev = _kernel_events(timing, s, "k1")
                k, v = src.ptrs(0)
                c0, sc0, z0 = payload.ptrs(0)
                _lib.call("kvx_quant_pack_signal", k, v, src.layer_stride, src.slots_ptr,
                          lay.n_layers, lay.n_tokens, lay.n_heads, lay.head_dim, lay.group,
                          lay.bits, c0, sc0, z0, lay.layer_stride, self.counters.data_ptr(),
                          self._pready(self.peer_flags, h, 0), lpc, _stream_ptr(s))
                _kernel_events_end(ev, s)
                return
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
                signal(self._pready(self.peer_flags, h, c), 1, s)

        self._run_or_capture(key, body, s, cur, capturable=timing is None and stage_in is None)
        if stage_in is not None:
            cur.wait_stream(self.xfer)

    def _recv_pull(self, dst, lay, e, s, cur, timing, stage_out):
        h = e & 1
        chunks, lpc = self._pull_chunks(lay)
        key = ("recv", lay.n_tokens, h, dst.slots_ptr, dst.k.data_ptr())
        if self._graph_ok(key, timing, stage_out):
            return self._replay(key, s, cur)
        payload = PackedKV(lay, self.k3_source + self._half(e), self.device)
        bulk = self.spec.mode == "pull" and pull_supported(lay)

        def body():
            if stage_out is not None:
                for c in range(len(chunks)):
                    s.wait_event(self.x_done[c])
            if bulk:
                # ONE persistent bulk-pull kernel per hand-off: its producer
                # threads wait in-kernel for each chunk's doorbell
                ev = _kernel_events(timing, s, "k3")
                dequant_scatter_layers(payload, dst, 0, lay.n_layers, s,
                                       ready=(self._pready(self.flags.ptr, h, 0), 1, lpc))
                _kernel_events_end(ev, s)
            else:
                for c, (l0, l1) in enumerate(chunks):
                    wait(self._pready(self.flags.ptr, h, c), 1, s)
                    ev = _kernel_events(timing, s, "k3")
                    dequant_scatter_layers(payload, dst, l0, l1, s)
                    _kernel_events_end(ev, s)
            _lib.call("kvx_memset_async", self._pready(self.flags.ptr, h, 0), 0,
                      4 * len(chunks), _stream_ptr(s))
            signal(self._pfree(self.peer_flags, h), 1, s)     # half consumed
            if stage_out is not None:
                (dk, dv), (hk, hv) = stage_out
                self.x_ready[0].record(s)
                self.xfer.wait_event(self.x_ready[0])
                with torch.cuda.stream(self.xfer):
                    hk.copy_(dk, non_blocking=True)
                    hv.copy_(dv, non_blocking=True)
                for c in range(len(chunks)):
                    self.x_done[c].record(self.xfer)

        self._run_or_capture(key, body, s, cur, capturable=timing is None and stage_out is None)
        if stage_out is not None:
            cur.wait_stream(self.xfer)

    # ---- kivi format over the pull queue (per-chunk doorbells, LDG kernels) ---
    def _kivi_common(self, n_tokens, seqlens, e):
        from .kivi import kivi_groups
        seqlens = tuple(int(n) for n in (seqlens if seqlens is not None else (n_tokens,)))
        lay = self.spec.kivi_layout(seqlens)
        if lay.n_tokens != n_tokens:
            raise ValueError("seqlens must sum to n_tokens")
        gs, rt = kivi_groups(seqlens, lay.group)
        chunks, _ = pull_chunk_plan(lay.n_layers, lay.fp16_bytes, self.spec.n_chunks,
                                    self.spec.min_chunk_bytes)
        return lay, gs, rt, chunks, e & 1

    def _send_kivi(self, src, n_tokens, seqlens, e):
        lay, gs, rt, chunks, h = self._kivi_common(n_tokens, seqlens, e)
        s, cur = self.stream, torch.cuda.current_stream(self.device)
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            gs_d = torch.from_numpy(gs).to(self.device, non_blocking=False)
            rt_d = torch.from_numpy(rt).to(self.device, non_blocking=False)
        base = self.k1_target + self._half(e)
        offs = (ctypes.c_int64 * 7)(*lay.offsets)
        wait(self._pfree(self.flags.ptr, h), 1, s)
        signal(self._pfree(self.flags.ptr, h), 0, s)
        for c, (l0, l1) in enumerate(chunks):
            k, v = src.ptrs(l0)
            _lib.call("kvx_quant_pack_kivi", k, v, src.layer_stride, l1 - l0, n_tokens,
                      lay.n_heads, lay.head_dim, lay.group, lay.bits,
                      gs_d.data_ptr() if len(gs) else None, len(gs),
                      rt_d.data_ptr() if len(rt) else None, len(rt),
                      base + l0 * lay.layer_stride, lay.layer_stride, offs, _stream_ptr(s))
            signal(self._pready(self.peer_flags, h, c), 1, s)
        gs_d.record_stream(s)
        rt_d.record_stream(s)
        cur.wait_stream(s)

    def _recv_kivi(self, dst, n_tokens, seqlens, e):
        lay, gs, rt, chunks, h = self._kivi_common(n_tokens, seqlens, e)
        s, cur = self.stream, torch.cuda.current_stream(self.device)
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            gs_d = torch.from_numpy(gs).to(self.device)
            rdst = dst.slots[torch.from_numpy(rt).to(self.device)].contiguous()
        base = self.k3_source + self._half(e)
        offs = (ctypes.c_int64 * 7)(*lay.offsets)
        for c, (l0, l1) in enumerate(chunks):
            wait(self._pready(self.flags.ptr, h, c), 1, s)
            k, v = dst.ptrs(l0)
            _lib.call("kvx_dequant_scatter_paged_kivi", base + l0 * lay.layer_stride,
                      lay.layer_stride, offs, dst.slots_ptr,
                      gs_d.data_ptr() if len(gs) else None, len(gs),
                      rdst.data_ptr() if rdst.numel() else None, rdst.numel(), l1 - l0,
                      n_tokens, lay.n_heads, lay.head_dim, lay.group, lay.bits, k, v,
                      dst.layer_stride, _stream_ptr(s))
        _lib.call("kvx_memset_async", self._pready(self.flags.ptr, h, 0), 0, 4 * len(chunks),
                  _stream_ptr(s))
        signal(self._pfree(self.peer_flags, h), 1, s)
        gs_d.record_stream(s)
        rdst.record_stream(s)
        cur.wait_stream(s)

    # ---- CUDA graphs: a hand-off of a given size is one graph launch ----------
    def _graph_ok(self, key, timing, staging) -> bool:
        return self.graphs and timing is None and staging is None and key in self._graphs

    def _replay(self, key, s, cur):
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            self._graphs[key].replay()
        cur.wait_stream(s)

    def _run_or_capture(self, key, body, s, cur, capturable: bool):
        s.wait_stream(cur)
        if self.graphs and capturable and key in self._seen:
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
                    body()
            except Exception:  # noqa: BLE001 - capture unsupported here: stay eager
                self.graphs = False
                body()
                cur.wait_stream(s)
                return
            self._graphs[key] = g
            with torch.cuda.stream(s):
                g.replay()
        else:
            body()
            if capturable:
                self._seen.add(key)  # eager once (attributes, caches), capture next time
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

    def recv(self, dst: KVPlanes, n_tokens: int, timing: list | None = None,
             stage_out: tuple | None = None, seqlens=None) -> None:
        """Receive into ``dst``.  ``stage_out=((dev_k, dev_v), (host_k, host_v))``:
        download each finished layer chunk of the cache to pinned host memory
        (D2H of chunk c overlaps K3 of chunk c+1)."""
        assert self.role == "decode"
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
        torch.cuda.synchronize(self.device)
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

def _verify_last(ch, trace, tok, it, L, H, D, spec, ctrl, kv=None, dec=None):
    """Bit-exact check of 3 layers x 32 sampled tokens of the last hand-off at
    full size: the prefill rank ships its source rows, the decode rank runs the
    C oracle on them and compares with its paged cache.  Returns the AND over
    all pairs (every rank gets it)."""
    import numpy as np

    last = (it["i"] - 1) % len(tok)
    T_last = tok[last]
    rng = np.random.default_rng(1234 + last)
    toks = np.sort(rng.choice(T_last, size=min(32, T_last), replace=False))
    layers = sorted({0, L // 2, L - 1})
    mine = None
    if ch.role == "prefill":
        rows = kv[layers][:, :, torch.from_numpy(toks).to(kv.device)]  # [nl, 2, n, H, D]
        mine = rows.cpu().numpy()
    else:
        kc, vc, pl = dec
        planes = pl if trace is None else pl[last]
        sl = planes.slots[torch.from_numpy(toks).to(kc.device)]
        ks = kc[layers].reshape(len(layers), -1, H, D)[:, sl]
        vs = vc[layers].reshape(len(layers), -1, H, D)[:, sl]
        mine = torch.stack([ks, vs], 1).cpu().numpy()
    allv = exchange(mine, ctrl)
    ok = True
    if ch.role == "decode":
        from oracle import kvq_oracle_c as C  # the checker, never the measured path
        src = allv[ch.peer]
        c, s_, z = C.quant_pack(np.ascontiguousarray(src).reshape(-1, D), spec.bits, spec.group)
        want = C.unpack_dequant(c, s_, z, spec.bits, spec.group, D).reshape(src.shape)
        ok = bool(np.array_equal(want.view(np.uint16), mine.view(np.uint16)))
        if not ok and os.environ.get("KVX_VERIFY_DEBUG"):
            bad = want.view(np.uint16) != mine.view(np.uint16)
            print(f"[verify] rank {ch.rank}: {int(bad.sum())}/{bad.size} mismatches; per layer "
                  f"{bad.reshape(len(layers), -1).sum(1).tolist()}; per kv {bad.sum((0, 2, 3, 4)).tolist()}"
                  f"; per token {bad.sum((0, 1, 3, 4)).tolist()}; max|d| "
                  f"{float(np.abs(want.astype(np.float32) - mine.astype(np.float32)).max())}",
                  flush=True)
    return all(exchange(ok, ctrl))


def _calibration(spec, T, ms_large, ms_small, t_small=16):
    """(alpha, beta) of t = alpha + V/beta with V the reference's modelled
    volume 2*b*s*h*bits/8*L (costs.py:102) -- what calibrate.cluster_dict and
    measured_kv_comm_cost consume."""
    from .calibrate import fit_alpha_beta
    v_large = spec.layout(T).fp16_bytes * spec.bits / 16
    v_small = spec.layout(t_small).fp16_bytes * spec.bits / 16
    try:
        alpha, beta = fit_alpha_beta(ms_small * 1e-3, v_small, ms_large * 1e-3, v_large)
    except ValueError:
        return None
    return {"alpha_us": round(alpha * 1e6, 2), "beta_GBps_of_modelled_volume": round(beta / 1e9, 1),
            "small_handoff_us": round(ms_small * 1e3, 2), "small_tokens": t_small,
            "note": "t = alpha + (2*b*s*h*bits/8*L)/beta, per pair, CUDA-graph replayed"}


def bench_pairs(args, torch_mod, rank: int, world: int, emit) -> None:
    """Weak-scaling pair benchmark: every pair hands off the same workload."""
    import json
    import torch.distributed as dist

    import bench as B

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    wl = args.workload or B.default_pair_workload(world)
    trace = None
    if wl in B.TRACE_MODELS:
        L, H, D = B.TRACE_MODELS[wl]
        trace = B.make_trace(args.warmup + args.steps + 2, seed=0)
        T = B.TRACE_CAP
    else:
        L, H, D, b, s = B.WORKLOADS[wl]
        T = b * s
    mode = args.mode
    n_chunks = args.chunks or 8
    spec = ChannelSpec(L, T, H, D, args.bits, args.group, n_chunks, mode,
                       format=getattr(args, "format", "default"))
    ch = PairChannel(spec, rank, world, control_group=ctrl, graphs=not args.no_graphs)
    lay = spec.layout(T)
    # per step token counts (fixed workload, or the trace's batches)
    tok = [T] * (args.warmup + args.steps + 2) if trace is None else [sum(x) for x in trace]
    seqs = ([(s,) * b] * len(tok)) if trace is None else [tuple(x) for x in trace]
    it = {"i": 0}
    kivi = spec.format == "kivi"

    def next_t():
        t = tok[it["i"] % len(tok)]
        it["i"] += 1
        return t

    if ch.role == "prefill":
        kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=ch.pair)
        planes = KVPlanes.dense(kv)
        def step(timing=None):
            i = it["i"] % len(tok)
            t = next_t()
            if kivi:
                ch.send(planes, t, seqlens=seqs[i])
            else:
                ch.send(planes, t, timing)
    else:
        slots, nb = B.paged_slots(torch, T, dev, seed=ch.pair)
        kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
        vc = torch.zeros_like(kc)
        if trace is None:
            planes = KVPlanes.paged(kc, vc, slots)

            def step(timing=None):
                i = it["i"] % len(tok)
                t = next_t()
                if kivi:
                    ch.recv(planes, t, seqlens=seqs[i])
                else:
                    ch.recv(planes, t, timing)
        else:
            # each batch gets its own random block placement (requests start on
            # a block boundary, as a paged allocator hands them out)
            import numpy as np
            rng = np.random.default_rng(ch.pair + 7)
            per_batch = []
            for lens in trace:
                nblk = sum((n + B.BLOCK - 1) // B.BLOCK for n in lens)
                blocks = rng.permutation(nb)[:nblk]
                sl, bi = [], 0
                for n in lens:
                    t = np.arange(n)
                    sl.append(blocks[bi + t // B.BLOCK] * B.BLOCK + t % B.BLOCK)
                    bi += (n + B.BLOCK - 1) // B.BLOCK
                per_batch.append(torch.from_numpy(np.concatenate(sl).astype(np.int64)).to(dev))
            planes_b = [KVPlanes.paged(kc, vc, sl) for sl in per_batch]

            def step(timing=None):
                i = it["i"] % len(tok)
                if kivi:
                    ch.recv(planes_b[i], next_t(), seqlens=seqs[i])
                else:
                    ch.recv(planes_b[i], next_t(), timing)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with B.ClockSampler(local) as clk:
        t0.record()
        for _ in range(args.steps):
            step()  # CUDA-graph replay per hand-off once warmed up (pull modes)
        t1.record()
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    # per-kernel durations: a separate eager pass with CUDA events on the
    # launching streams (events cannot sit inside the captured graph)
    timing = []
    n_kt = max(1, min(args.steps, 5))
    for _ in range(n_kt):
        step(timing)
    torch.cuda.synchronize()
    dist.barrier()
    kern = {}
    for name, a, b_ in timing:
        kern[name] = kern.get(name, 0.0) + a.elapsed_time(b_) / n_kt
    launches = len(timing) / n_kt * args.steps
    # full-size parity (outside the timed region): sampled token rows of the
    # last hand-off, decode cache vs the CPU oracle applied to the source rows
    verified = None
    if not getattr(args, "no_verify", False) and not kivi:
        verified = _verify_last(ch, trace, tok, it, L, H, D, spec, ctrl,
                                kv if ch.role == "prefill" else None,
                                (kc, vc, planes if trace is None else planes_b)
                                if ch.role == "decode" else None)
    # alpha-beta calibration of this very channel (graph-replayed pull): a
    # 16-token hand-off against the main one -> kv_comm_cost's (alpha, beta)
    # for the reference's volume at this bit-width
    cal_small_ms = 0.0
    if trace is None and not kivi:
        t_small = 16
        if ch.role == "prefill":
            small = lambda: ch.send(planes, t_small)  # noqa: E731
        else:
            sl_small = KVPlanes.paged(kc, vc, planes.slots[:t_small])
            small = lambda: ch.recv(sl_small, t_small)  # noqa: E731
        for _ in range(3):
            small()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_cal = 50
        c0.record()
        for _ in range(n_cal):
            small()
        c1.record()
        torch.cuda.synchronize()
        cal_small_ms = c0.elapsed_time(c1) / n_cal
        dist.barrier()
    # e2e through the same public API with host buffers: pinned host KV on the
    # prefill side (H2D inside the step), pinned host paged cache on the decode
    # side (D2H inside the step)
    e2e_ms, h2d, d2h = 0.0, 0, 0
    if not args.no_e2e and not kivi:
        if ch.role == "prefill":
            host = torch.empty(kv.shape, dtype=torch.float16, pin_memory=True)
            host.copy_(kv)
            stage = dict(stage_in=(host, kv))
            h2d = host.numel() * 2
            e2e_step = lambda: ch.send(planes, next_t(), None, **stage)  # noqa: E731
        else:
            hk = torch.empty(kc.shape, dtype=torch.float16, pin_memory=True)
            hv = torch.empty(vc.shape, dtype=torch.float16, pin_memory=True)
            stage = dict(stage_out=((kc, vc), (hk, hv)))
            d2h = (hk.numel() + hv.numel()) * 2
            e2e_step = (lambda: ch.recv(planes, next_t(), None, **stage)) if trace is None else (
                lambda: ch.recv(planes_b[it["i"] % len(tok)], next_t(), None, **stage))
        n_e2e = max(1, min(args.steps, args.e2e_steps))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_e2e):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / n_e2e
        dist.barrier()
    stats = torch.tensor([ms, kern.get("k1", 0.0), kern.get("k3", 0.0), e2e_ms, h2d, d2h,
                          launches, cal_small_ms], dtype=torch.float64, device=dev)
    gathered = [torch.zeros_like(stats) for _ in range(world)]
    dist.all_gather(gathered, stats)
    clocks = exchange(clk.summary(), ctrl)
    if rank == 0:
        g = torch.stack(gathered).cpu()
        ms_max = float(g[:, 0].max())
        k1 = float(g[:, 1].max())
        k3 = float(g[:, 2].max())
        pairs = world // 2
        if kivi:
            timed = range(args.warmup, args.warmup + args.steps)
            fp16 = sum(spec.kivi_layout(seqs[i % len(tok)]).fp16_bytes for i in timed) / len(timed)
            wire_mean = sum(spec.kivi_layout(seqs[i % len(tok)]).wire_bytes
                            for i in timed) / len(timed)
        elif trace is None:
            fp16 = lay.fp16_bytes
        else:  # mean fp16 bytes of the timed batches
            timed = tok[args.warmup:args.warmup + args.steps]
            fp16 = sum(spec.layout(t).fp16_bytes for t in timed) / len(timed)
            wire_mean = sum(spec.layout(t).wire_bytes for t in timed) / len(timed)
        value = pairs * fp16 / (ms_max * 1e-3) / 1e9
        wire = lay.wire_bytes if (trace is None and not kivi) else wire_mean
        link_gbs = wire / (ms_max * 1e-3) / 1e9  # per pair
        hbm, peak_kind = B.peaks()
        k3_link = wire / (k3 * 1e-3) / 1e9 if k3 > 0 else None
        sm = [c["sm_mhz"] for c in clocks if c.get("sm_mhz")]
        reasons = sorted({r for c in clocks for r in c.get("reasons", [])})
        r = dict(
            value=value, ms=ms_max, workload=wl, fp16_bytes=fp16 * pairs, wire_bytes=wire * pairs,
            launches=int(g[:, 6].sum()),  # kvx kernels launched in the timed region
            clocks={"sm_mhz": min(sm) if sm else None,
                    "sm_max_mhz": max((c.get("sm_max_mhz") or 0) for c in clocks) or None,
                    "reasons": reasons, "per_rank_median_sm_mhz": sm},
            e2e=None if (args.no_e2e or kivi) else {
                "value": round(pairs * fp16 / (float(g[:, 3].max()) * 1e-3) / 1e9, 3),
                "unit": "GB/s", "h2d_bytes_per_step": int(g[:, 4].sum()),
                "d2h_bytes_per_step": int(g[:, 5].sum()),
                "ms_per_step": round(float(g[:, 3].max()), 3),
                "path": "pinned host KV -(H2D)-> K1 on P -(NVLink)-> K3 on D -(D2H)-> pinned "
                        "host paged cache, per layer chunk"},
            cpu=None,
            roofline={"bound": "nvlink", "kernel": "pull_dequant_scatter_paged (TMA bulk pull "
                      "over NVLink)" if mode == "pull" else f"hand-off ({mode})",
                      "achieved": round(link_gbs, 1), "peak": B.NVLINK_GBS,
                      "peak_kind": "measured peer copy, B200_PROFILING.md (900 nominal)",
                      "unit": "GB/s", "frac": round(link_gbs / B.NVLINK_GBS, 4), "traffic": None,
                      "k1_ms": round(k1, 4), "k3_ms": round(k3, 4),
                      "k3_link_gbs": round(k3_link, 1) if k3_link else None,
                      "frac_of_nominal_900": round(link_gbs / 900.0, 4),
                      "hbm_peak": hbm},
            calibration=_calibration(spec, T, ms_max, float(g[:, 7].max())) if (
                trace is None and not kivi) else None,
            extra={"mode": mode, "n_chunks": len(spec.chunks()), "pairs": pairs,
                   "format": spec.format,
                   "cuda_graphs": bool(ch.graphs),
                   "verified_sampled_rows_bit_exact": verified,
                   **({"trace_batches_timed": tok[args.warmup:args.warmup + args.steps],
                       "trace": "lengths log-uniform [128, 8192], 1-16 req/batch, <=16384 "
                                "tokens/batch, rng(0)"} if trace is not None else {}),
                   "pairing": pairing(world), "parallelism": f"{pairs}P{pairs}D"},
        )
        emit(args, r, world)
    dist.barrier()
    ch.close()
    dist.destroy_process_group()
