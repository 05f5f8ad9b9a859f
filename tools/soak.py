"""Soak test of the pair protocol (torchrun, 2 ranks): thousands of hand-offs
with random lengths, fresh slot tensors, random decode-round batching
(`recv_many` of 1..Q queued hand-offs, or chained recvs), both prefill modes (front-end gate /
latency mode) and queue depths, for a wall-clock budget.  Every hand-off's
destination blocks are distinct within a round; every CHECK_EVERY-th round is
compared on every byte against the local K1 -> K3 on the decode GPU (itself
oracle-pinned).  Prints one JSON line: hand-offs, rounds, checks, mismatches.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      tools/soak.py --seconds 300
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _mp  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel, exchange  # noqa: E402

CHECK_EVERY = 7


def run_config(rank, world, dev, ctrl, Q, gate, L, H, D, Tmax, seconds, seed):
    spec = ChannelSpec(L, Tmax, H, D, 4, 128, 8, "pull", queue_depth=Q, gate_send=gate)
    ch = PairChannel(spec, rank, world, control_group=ctrl)
    bs = 16
    nb = Q * (Tmax // bs + 1) + 8
    rng = np.random.default_rng(seed)  # the same stream on both ranks
    if ch.role == "decode":
        kc = torch.zeros((L, nb, bs, H, D), dtype=torch.float16, device=dev)
        vc = torch.zeros_like(kc)
    handoffs = rounds = checks = bad = 0
    t_end = time.time() + seconds
    stop = False
    while not stop:
        k = int(rng.integers(1, Q + 1))
        Ts = [int(x) for x in rng.integers(1, Tmax + 1, size=k)]
        seeds = [int(x) for x in rng.integers(0, 1 << 30, size=k)]
        check = rounds % CHECK_EVERY == 0
        kvs = []
        for T, sd in zip(Ts, seeds):
            g = torch.Generator(device=dev).manual_seed(sd)
            kvs.append(torch.randn((L, 2, T, H, D), generator=g, device=dev).half())
        if ch.role == "prefill":
            for kv, T in zip(kvs, Ts):
                ch.send(KVPlanes.dense(kv), T)
        else:
            perm = torch.from_numpy(rng.permutation(nb)).to(dev)
            items, b0 = [], 0
            for T in Ts:
                t = torch.arange(T, device=dev)
                sl = perm[b0 + t // bs] * bs + t % bs
                b0 += (T + bs - 1) // bs
                items.append((KVPlanes.paged(kc, vc, sl), T))
            if check:
                kc.zero_()
                vc.zero_()
            use_many = k > 1 and rng.random() < 0.5
            chain = rng.random() < 0.5
            if use_many:
                ch.recv_many(items)
            elif chain:
                # chained pulls (kvx.h KVX_PAIR_CHAINED): the slot mappings are
                # made and the round's blocks are distinct, so every recv after
                # the first may write while the previous one drains
                torch.cuda.current_stream().synchronize()
                for i, it in enumerate(items):
                    ch.recv(*it, chained=i > 0)
            else:
                for it in items:
                    ch.recv(*it)
            if check:
                rk = torch.zeros_like(kc)
                rv = torch.zeros_like(vc)
                for kv, (pl, T) in zip(kvs, items):
                    a, b = _mp.local_reference(kv, kc.shape, pl.slots)
                    m = pl.slots
                    # merge: each hand-off owns distinct blocks
                    rk.view(L, -1, H, D)[:, m] = a.view(L, -1, H, D)[:, m]
                    rv.view(L, -1, H, D)[:, m] = b.view(L, -1, H, D)[:, m]
                torch.cuda.synchronize()
                checks += 1
                if not (torch.equal(kc, rk) and torch.equal(vc, rv)):
                    bad += 1
                    print(f"MISMATCH rank={rank} round={rounds} Ts={Ts}", flush=True)
        # both ranks draw the next round from the same stream; the decode
        # rank also drew the block permutation, so advance the prefill side
        if ch.role == "prefill":
            rng.permutation(nb)
            if k > 1:
                rng.random()
            rng.random()
        handoffs += k
        rounds += 1
        if rounds % 50 == 0:
            stop = exchange(time.time() > t_end, ctrl)[0]
    torch.cuda.synchronize()
    ch.check()
    dist.barrier(ctrl)
    ch.close()
    return {"Q": Q, "gate_send": gate, "handoffs": handoffs, "rounds": rounds,
            "checks": checks, "mismatches": bad}


def run_kivi(rank, world, dev, ctrl, L, H, D, Tmax, seconds, seed):
    """kivi format: ragged batches of 1-4 requests (residual rows in most),
    one fused prefill call and one pull kernel per hand-off; every round
    checked against the local kivi round trip (compress_kivi ->
    decompress_kivi_into_paged, oracle-pinned in tests/test_gpu_kivi.py)."""
    from paper_2502_09334_b200.kivi import compress_kivi, decompress_kivi_into_paged
    spec = ChannelSpec(L, Tmax, H, D, 4, 32, 8, "pull", format="kivi", queue_depth=2)
    ch = PairChannel(spec, rank, world, control_group=ctrl)
    bs = 16
    nb = Tmax // bs + 8
    rng = np.random.default_rng(seed)
    if ch.role == "decode":
        kc = torch.zeros((L, nb, bs, H, D), dtype=torch.float16, device=dev)
        vc = torch.zeros_like(kc)
        rk = torch.zeros_like(kc)
        rv = torch.zeros_like(kc)
    handoffs = checks = bad = 0
    t_end = time.time() + seconds
    stop = False
    while not stop:
        n_req = int(rng.integers(1, 5))
        seq = tuple(int(x) for x in rng.integers(1, Tmax // 4 + 1, size=n_req))
        T = sum(seq)
        sd = int(rng.integers(0, 1 << 30))
        g = torch.Generator(device=dev).manual_seed(sd)
        kv = torch.randn((L, 2, T, H, D), generator=g, device=dev).half()
        perm = rng.permutation(nb * bs)[:T]
        if ch.role == "prefill":
            ch.send(KVPlanes.dense(kv), T, seqlens=seq)
        else:
            sl = torch.from_numpy(perm.astype(np.int64)).to(dev)
            kc.zero_(); vc.zero_(); rk.zero_(); rv.zero_()
            ch.recv(KVPlanes.paged(kc, vc, sl), T, seqlens=seq)
            decompress_kivi_into_paged(compress_kivi(kv, 4, 32, seq), rk, rv, sl)
            torch.cuda.synchronize()
            checks += 1
            if not (torch.equal(kc, rk) and torch.equal(vc, rv)):
                bad += 1
                print(f"MISMATCH kivi rank={rank} seq={seq}", flush=True)
        handoffs += 1
        if handoffs % 20 == 0:
            stop = exchange(time.time() > t_end, ctrl)[0]
    torch.cuda.synchronize()
    ch.check()
    dist.barrier(ctrl)
    ch.close()
    return {"format": "kivi", "handoffs": handoffs, "checks": checks, "mismatches": bad}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120.0)
    a = ap.parse_args()
    rank, world, dev, ctrl, _ = _mp.init()
    out = []
    configs = [(2, True), (4, False), (8, False), (3, True)]
    share = a.seconds / (len(configs) + 1)
    for i, (Q, gate) in enumerate(configs):
        out.append(run_config(rank, world, dev, ctrl, Q, gate, L=8, H=8, D=128, Tmax=2048,
                              seconds=share, seed=1000 + i))
    out.append(run_kivi(rank, world, dev, ctrl, L=8, H=8, D=128, Tmax=2048, seconds=share,
                        seed=99))
    res = exchange(out, ctrl)
    if rank == 0:
        dec = res[1]
        print(json.dumps({"soak": dec, "total_handoffs": sum(r["handoffs"] for r in dec),
                          "total_checks": sum(r["checks"] for r in dec),
                          "total_mismatches": sum(r["mismatches"] for r in dec)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
