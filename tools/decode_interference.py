"""What a pull costs the decode GPU's own work (torchrun, 2 ranks).

The paper's decode replicas pull queued KV from prefill GPUs between decode
rounds.  A pull is NVLink-bound, but its K3 writes the fp16
cache into the decode GPU's HBM at ~2.8 TB/s and holds a CTA per SM.  This
tool measures, on the decode GPU's clock:

  round_alone  : one synthetic decode round (an HBM-bound read of a
                 --round-gb fp16 buffer, like attention over the KV cache)
  pull_alone   : one config-4 pair hand-off (70B GQA, 8192 tokens)
  both         : the round on the compute stream with a pull issued at the
                 same time on the channel's stream -> round and pull times

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      tools/decode_interference.py [--round-gb 4]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round-gb", type=float, default=4.0)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    L, H, D, b, s = B.WORKLOADS["cfg4_70b_gqa_pair"]
    T = b * s
    ch = PairChannel(ChannelSpec(L, T, H, D, 4, 128, 8, "pull"), rank, world, control_group=ctrl)
    res = {}
    if ch.role == "prefill":
        kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=0)
        planes = KVPlanes.dense(kv)
        for _ in range(6 + 2 * a.reps):  # the decode side pulls this many hand-offs
            ch.send(planes, T)
        torch.cuda.synchronize()
    else:
        slots, nb = B.paged_slots(torch, T, dev)
        kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
        planes = KVPlanes.paged(kc, torch.zeros_like(kc), slots)
        cache = torch.randn(int(a.round_gb * 2**29), device=dev).half()  # round_gb GB fp16
        comp, pull = torch.cuda.Stream(), torch.cuda.Stream()

        def ev():
            return torch.cuda.Event(enable_timing=True)

        def decode_round():
            return cache.sum(dtype=torch.float32)

        for _ in range(6):  # warm-up incl. graph capture of the recv
            with torch.cuda.stream(pull):
                ch.recv(planes, T)
            with torch.cuda.stream(comp):
                decode_round()
        torch.cuda.synchronize()
        alone, palone, r_both, p_both = [], [], [], []
        for _ in range(a.reps):
            e0, e1 = ev(), ev()
            with torch.cuda.stream(comp):
                e0.record(); decode_round(); e1.record()
            torch.cuda.synchronize()
            alone.append(e0.elapsed_time(e1))
            e0, e1 = ev(), ev()
            with torch.cuda.stream(pull):
                e0.record(); ch.recv(planes, T); e1.record()
            torch.cuda.synchronize()
            palone.append(e0.elapsed_time(e1))
            r0, r1, p0, p1 = ev(), ev(), ev(), ev()
            with torch.cuda.stream(pull):
                p0.record(); ch.recv(planes, T); p1.record()
            with torch.cuda.stream(comp):
                r0.record(); decode_round(); r1.record()
            torch.cuda.synchronize()
            r_both.append(r0.elapsed_time(r1))
            p_both.append(p0.elapsed_time(p1))
        med = statistics.median
        res = {"round_gb": a.round_gb, "round_alone_ms": round(med(alone), 3),
               "pull_alone_ms": round(med(palone), 3),
               "round_with_pull_ms": round(med(r_both), 3),
               "pull_with_round_ms": round(med(p_both), 3),
               "round_hbm_gbs_alone": round(a.round_gb * 1e9 / 1e9 / (med(alone) / 1e3), 1)}
        print(json.dumps({"workload": "cfg4_70b_gqa_pair", **res}), flush=True)
    dist.barrier()
    ch.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
