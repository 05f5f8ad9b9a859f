"""A decode replica pulling queued KV between decode rounds (torchrun, 2 ranks;
the paper's serving loop).

The prefill rank produces one prompt's KV every --prefill-us (a sleep kernel
stands in for the prefill compute) and hands it off into its HBM queue
(queue_depth slots).  The decode rank runs decode rounds (an HBM-bound read of
a --round-gb buffer stands in for attention over the KV cache); between rounds
it polls the channel and pulls every hand-off that is ready -- never
launching a pull that would wait for the prefill side.  Reports, on the
decode GPU: rounds run, hand-offs pulled, mean round time, and the mean time a
pull added to the round it followed.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      tools/decode_rounds.py [--prompts 24 --prefill-us 3000 --round-gb 4]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prompts", type=int, default=24)
    ap.add_argument("--prefill-us", type=float, default=3000.0)
    ap.add_argument("--round-gb", type=float, default=4.0)
    ap.add_argument("--queue-depth", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=None,
                    help="prompt length (default: a config-4 pair, 2 x 4096)")
    ap.add_argument("--drain", action="store_true",
                    help="after each round pull everything queued with ONE launch "
                         "(poll_count + recv_many) instead of one pull per hand-off")
    ap.add_argument("--latency-mode", action="store_true",
                    help="prefill side without the front-end gate (PDL-chained K1)")
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    L, H, D, b, s = B.WORKLOADS["cfg4_70b_gqa_pair"]
    T = a.tokens or b * s
    ch = PairChannel(ChannelSpec(L, T, H, D, 4, 128, 8, "pull", queue_depth=a.queue_depth,
                                 gate_send=not a.latency_mode),
                     rank, 2, control_group=ctrl)
    if ch.role == "prefill":
        kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=0)
        planes = KVPlanes.dense(kv)
        for _ in range(2 * a.queue_depth):  # warm-up hand-offs (graph capture on both ends)
            ch.send(planes, T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)  # clocks up before calibrating the sleep kernel
        e0.record(); torch.cuda._sleep(10_000_000); e1.record(); torch.cuda.synchronize()
        cycles = int(a.prefill_us * 10_000_000 / (e0.elapsed_time(e1) * 1e3))
        dist.barrier(ctrl)
        e0.record()
        for _ in range(a.prompts):
            torch.cuda._sleep(cycles)  # "prefill" of the next prompt
            ch.send(planes, T)
        e1.record()
        torch.cuda.synchronize()
        res = {"prefill_span_ms": round(e0.elapsed_time(e1), 2)}
        dist.barrier(ctrl)
        exchange_res = [None, None]
        dist.all_gather_object(exchange_res, res, group=ctrl)
    else:
        # one block range per queue slot, so a drained batch lands in distinct blocks
        need = (T + B.BLOCK - 1) // B.BLOCK
        nb = need * a.queue_depth + 64
        kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
        vc = torch.zeros_like(kc)
        perm = torch.randperm(nb, generator=torch.Generator().manual_seed(1))
        tt = torch.arange(T)
        planes_q = [KVPlanes.paged(kc, vc, (perm[j * need + tt // B.BLOCK] * B.BLOCK +
                                            tt % B.BLOCK).to(dev)) for j in range(a.queue_depth)]
        planes = planes_q[0]
        cache = torch.randn(int(a.round_gb * 2**29), device=dev).half()
        for _ in range(2 * a.queue_depth):  # warm-up pulls, and the round kernel
            ch.recv(planes, T)
            cache.sum(dtype=torch.float32)
        torch.cuda.synchronize()
        rounds, pulled, launches, t_round, t_pull = 0, 0, 0, [], []
        dist.barrier(ctrl)
        t0 = time.perf_counter()
        s0 = torch.cuda.Event(enable_timing=True)
        s0.record()
        while pulled < a.prompts and time.perf_counter() - t0 < 60:
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record(); cache.sum(dtype=torch.float32); r1.record()
            r1.synchronize()
            t_round.append(r0.elapsed_time(r1))
            rounds += 1
            if a.drain:  # everything queued, one pull launch
                n = min(ch.poll_count(), a.prompts - pulled)
                if n:
                    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    p0.record(); ch.recv_many([(planes_q[j], T) for j in range(n)]); p1.record()
                    p1.synchronize()
                    t_pull.append(p0.elapsed_time(p1))
                    pulled += n
                    launches += 1
                continue
            while pulled < a.prompts and ch.poll():  # pull whatever the queue holds
                p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                p0.record(); ch.recv(planes, T); p1.record()
                p1.synchronize()
                t_pull.append(p0.elapsed_time(p1))
                pulled += 1
                launches += 1
        s1 = torch.cuda.Event(enable_timing=True)
        s1.record()
        s1.synchronize()
        span_ms = s0.elapsed_time(s1)
        dist.barrier(ctrl)
        exchange_res = [None, None]
        dist.all_gather_object(exchange_res, {}, group=ctrl)
        print(json.dumps({"workload": f"70b_gqa_{T}tok", "prompts": a.prompts,
                          "drain": a.drain, "pull_launches": launches,
                          "latency_mode": a.latency_mode,
                          **exchange_res[0], "decode_span_ms": round(span_ms, 2),
                          "prefill_us": a.prefill_us, "queue_depth": a.queue_depth,
                          "decode_rounds": rounds, "pulled": pulled,
                          "round_ms_mean": round(statistics.mean(t_round), 3),
                          "pull_ms_mean": round(statistics.mean(t_pull), 3) if t_pull else None,
                          "pull_ms_per_handoff": round(sum(t_pull) / max(1, pulled), 4),
                          "pull_ms_max": round(max(t_pull), 3) if t_pull else None}), flush=True)
    dist.barrier()
    ch.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
