"""TP-sharded hand-off throughput (torchrun, 4 ranks): 70B GQA KV (80 layers,
8 KV heads x 128, 8192 tokens) between TP-sharded prefill and decode
replicas, SURVEY.md 8(e).  Every (prefill rank, decode rank) pair whose head
ranges overlap is one NVLink edge (TPHandoff); fan-in and fan-out regroups
share a GPU's link between edges.

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
      tools/tp_bench.py

Prints one JSON line per scenario: GB/s of fp16-equivalent KV handed off
(the whole replica's KV per step), max over ranks of CUDA-event time.
--paged-src: the prefill ranks hand off from their own paged caches (a slot
mapping per token) instead of dense KV.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import TPHandoff  # noqa: E402


def main():
    paged_src = "--paged-src" in sys.argv
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    L, H, D, T = 80, 8, 128, 8192
    steps = 20
    scenarios = {"tp2->tp2": ([0, 1], [2, 3]), "tp2->tp1 (fan-in)": ([0, 1], [2]),
                 "tp1->tp2 (fan-out)": ([0], [2, 3]), "tp1->tp1": ([0], [2])}
    for name, (pr, dr) in scenarios.items():
        tp = TPHandoff(L, T, H, D, pr, dr, rank, world, ctrl)
        if rank in pr:
            hp = H // len(pr)
            if paged_src:
                sl, nbp = B.paged_slots(torch, T, dev, seed=rank)
                pk = torch.randn((L, nbp, B.BLOCK, hp, D), device=dev).half()
                src = KVPlanes.paged(pk, torch.randn_like(pk), sl)
            else:
                src = KVPlanes.dense(B.synthetic_kv_device(torch, L, T, hp, D, dev, seed=rank))
            step = lambda: tp.send(src, T)  # noqa: E731
        elif rank in dr:
            hd = H // len(dr)
            slots, nb = B.paged_slots(torch, T, dev)
            kc = torch.zeros((L, nb, B.BLOCK, hd, D), dtype=torch.float16, device=dev)
            planes = KVPlanes.paged(kc, torch.zeros_like(kc), slots)
            step = lambda: tp.recv(planes, T)  # noqa: E731
        else:
            step = None
        for _ in range(6):
            if step:
                step()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            if step:
                step()
        b.record()
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b) / steps], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.barrier()
        if rank == 0:
            fp16 = L * 2 * T * H * D * 2
            print(json.dumps({"scenario": name, "prefill_source": "paged" if paged_src else "dense",
                              "prefill_ranks": pr, "decode_ranks": dr,
                              "edges": len(tp.edges) if rank in pr or rank in dr else None,
                              "ms_per_step": round(float(ms), 4),
                              "GBps_fp16_eq": round(fp16 / (float(ms) * 1e-3) / 1e9, 1)}),
                  flush=True)
        for ch, *_ in tp.edges:
            ch.close()
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
