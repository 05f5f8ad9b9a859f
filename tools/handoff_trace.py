"""Timeline of small fused hand-offs from %globaltimer stamps inside the
kernels (trace build: python -m paper_2502_09334_b200.build --variant trace
KVX_TRACE).  Prefill rank: K1-signal launch start, free seen, last doorbell
rung, last CTA out.  Decode rank: K3-bulk start, doorbell seen, release
issued, release done.  The clocks of the two GPUs are aligned by assuming the
two doorbell directions have equal latency.

    KVX_LIB=paper_2502_09334_b200/_kvx_trace.so torchrun --nproc-per-node 2 \\
        --master-addr 127.0.0.1 tools/handoff_trace.py [--tokens 16]"""
import argparse
import ctypes
import json
import os
import statistics as st
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_09334_b200 import _lib  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel, exchange  # noqa: E402


def read_trace(kind):
    lib = _lib.load()
    fn = lib.kvx_trace_read
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint)]
    buf = np.zeros((4096, 4), np.uint64)
    n = ctypes.c_uint(0)
    _lib.check(fn(kind, buf.ctypes.data, ctypes.byref(n)))
    return buf[: n.value].astype(np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--queue-depth", type=int, default=2)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-gate-send", action="store_true")
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--heads", type=int, default=8)
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    L, H, D, T = a.layers, a.heads, 128, a.tokens
    ch = PairChannel(ChannelSpec(L, T, H, D, 4, 128, 8, "pull", queue_depth=a.queue_depth,
                                 pdl=not a.no_pdl, gate_send=not a.no_gate_send),
                     rank, 2, control_group=ctrl)
    if ch.role == "prefill":
        kv = torch.randn((L, 2, T, H, D), device=dev).half()
        planes = KVPlanes.dense(kv)
        step = lambda: ch.send(planes, T)  # noqa: E731
    else:
        kc = torch.zeros((L, T // 16 + 4, 16, H, D), dtype=torch.float16, device=dev)
        planes = KVPlanes.paged(kc, torch.zeros_like(kc), torch.arange(T, device=dev))
        step = lambda: ch.recv(planes, T)  # noqa: E731
    for _ in range(a.steps):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    tr = read_trace(0 if ch.role == "prefill" else 1)
    allt = exchange(tr.tolist(), ctrl)
    if rank == 0:
        # rows are indexed by the hand-off's epoch (1..steps; row 0 unused)
        k1 = np.array(allt[0], np.int64)[1:]  # start, free seen, rung, out    (P clock)
        k3 = np.array(allt[1], np.int64)[1:]  # start, ready seen, release, released (D clock)
        n = min(len(k1), len(k3))
        k1, k3 = k1[:n], k3[:n]
        s = slice(n // 2, n)  # steady state
        fwd = k3[s, 1] - k1[s, 2]                 # doorbell P->D  = L + d
        back = k1[2:, 1][n // 2 - 2:] - k3[:-2, 3][n // 2 - 2:]  # free D->P for e+2 = L - d
        d = (st.median(fwd) - st.median(back)) / 2
        med = lambda x: round(float(st.median(x)) / 1e3, 2)  # noqa: E731
        out = {
            "tokens": T, "launches": n,
            "period_us": med(np.diff(k3[s, 3])),
            "one_way_doorbell_us": med((fwd + back[: len(fwd)]) / 2),
            "k1_launch_to_free_seen_us": med(k1[s, 1] - k1[s, 0]),
            "k1_free_seen_to_rung_us": med(k1[s, 2] - k1[s, 1]),
            "k1_rung_to_out_us": med(k1[s, 3] - k1[s, 2]),
            "k1_gap_prev_out_to_start_us": med(k1[n // 2 + 1:, 0] - k1[n // 2:-1, 3]),
            "k3_launch_to_ready_seen_us": med(k3[s, 1] - k3[s, 0]),
            "k3_ready_seen_to_release_us": med(k3[s, 2] - k3[s, 1]),
            "k3_release_store_us": med(k3[s, 3] - k3[s, 2]),
            "k3_gap_prev_out_to_start_us": med(k3[n // 2 + 1:, 0] - k3[n // 2:-1, 3]),
            "k3_start_minus_k1_rung_us": med(k3[s, 0] - d - k1[s, 2]),
            "queue_depth": a.queue_depth, "pdl": not a.no_pdl, "layers": L, "heads": H,
            "gate_send": not a.no_gate_send,
        }
        # three consecutive steady-state hand-offs on one (prefill) clock, us
        # relative to the first K1's start
        i0 = n // 2
        t0 = k1[i0, 0]
        out["timeline_us"] = [
            {"epoch": int(i0 + 1 + j),
             "k1": [round((x - t0) / 1e3, 2) for x in k1[i0 + j]],
             "k3": [round((x - d - t0) / 1e3, 2) for x in k3[i0 + j]]} for j in range(3)]
        print(json.dumps(out), flush=True)
    dist.barrier()
    ch.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
