"""Exposed hand-off latency after prefill (torchrun, 2 ranks): how long after
the prefill GPU finishes its LAST layer is the KV fully in the decode GPU's
paged cache?  (This is what the hand-off adds to time-to-first-token.)

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      tools/prefill_overlap.py [--layer-us 500]

Prefill is simulated on the prefill GPU by a fixed-duration kernel per layer
(torch.cuda._sleep); its KV is the config-4 pair tensor (70B GQA, 8192 tokens).
Measured on the prefill GPU's clock: event after the last layer -> event after
the decode side frees the queue half (its K3 finished).

  after   : hand-off starts when prefill ends (ch.send)
  stream  : layer-wise hand-off during prefill (ch.open_send / layers_ready)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench as B  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel, exchange, wait  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer-us", type=float, default=500.0)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    L, H, D, b, s = B.WORKLOADS["cfg4_70b_gqa_pair"]
    T = b * s
    # calibrate the sleep kernel: cycles per microsecond
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(); torch.cuda._sleep(10_000_000); t1.record(); torch.cuda.synchronize()
    cyc_per_us = 10_000_000 / (t0.elapsed_time(t1) * 1e3)
    layer_cycles = int(a.layer_us * cyc_per_us)
    out = {}
    for mode in ("after", "stream"):
        spec = ChannelSpec(L, T, H, D, 4, 128, 8, "pull", layerwise=(mode == "stream"))
        ch = PairChannel(spec, rank, world, control_group=ctrl)
        if ch.role == "prefill":
            kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=0)
            planes = KVPlanes.dense(kv)
        else:
            slots, nb = B.paged_slots(torch, T, dev)
            kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
            vc = torch.zeros_like(kc)
            planes = KVPlanes.paged(kc, vc, slots)
        lat = []
        for rep in range(a.reps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            if ch.role == "prefill":
                e_end, e_done = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if mode == "stream":
                    sess = ch.open_send(planes, T)
                for l in range(L):
                    torch.cuda._sleep(layer_cycles)  # "layer l"
                    if mode == "stream":
                        sess.layers_ready(l + 1)
                e_end.record()
                if mode == "stream":
                    sess.close()
                else:
                    ch.send(planes, T)
                # the decode side sets free[h] = v when its K3 has consumed
                # the slot (the sequence protocol)
                h, v = ch._seq(ch.epoch)
                cur = torch.cuda.current_stream()
                wait(ch._pfree(ch.flags.ptr, h), v, cur)
                e_done.record()
                torch.cuda.synchronize()
                if rep:
                    lat.append(e_end.elapsed_time(e_done) * 1e3)
            else:
                ch.recv(planes, T)
                torch.cuda.synchronize()
        dist.barrier()
        res = exchange(lat, ctrl)[0]
        out[mode] = {"exposed_us_median": sorted(res)[len(res) // 2], "samples_us": [round(x, 1) for x in res]}
        ch.close()
    if rank == 0:
        print(json.dumps({"workload": "cfg4_70b_gqa_pair", "layers": L, "layer_us": a.layer_us,
                          **out}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
