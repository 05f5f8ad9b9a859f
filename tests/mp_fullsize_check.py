"""torchrun worker for tests/test_gpu_multiproc.py::test_fullsize_pairs: the
bench's pair workloads at FULL size through the default transport (the fused
native pull), checked on EVERY byte of the decode cache against a local
K1 -> K3 round trip of the same KV on the decode GPU (itself bit-exact
against the oracle in tests/test_gpu_parity.py).  Exits non-zero on any
mismatch."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _mp  # noqa: E402
import bench as B  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel  # noqa: E402


def main():
    workloads = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg4_70b_gqa_pair"]
    rank, world, dev, ctrl, _ = _mp.init()
    failures = 0
    for wl in workloads:
        L, H, D, b, s = B.WORKLOADS[wl]
        T = b * s
        ch = PairChannel(ChannelSpec(L, T, H, D, 4, 128, 8, "pull"), rank, world,
                         control_group=ctrl)
        # the prefill rank's KV, regenerated bit-identically on the decode rank
        kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=ch.pair)
        if ch.role == "prefill":
            for _ in range(3):  # three hand-offs over both queue slots
                ch.send(KVPlanes.dense(kv), T)
            torch.cuda.synchronize()
            ch.check()
            del kv
        else:
            slots, nb = B.paged_slots(torch, T, dev, seed=ch.pair)
            kc = torch.full((L, nb, B.BLOCK, H, D), -7.0, dtype=torch.float16, device=dev)
            vc = torch.full_like(kc, -7.0)
            for _ in range(3):
                ch.recv(KVPlanes.paged(kc, vc, slots), T)
            torch.cuda.synchronize()
            ch.check()
            rk = torch.full_like(kc, -7.0)  # untouched blocks keep the sentinel
            rv = torch.full_like(vc, -7.0)
            from paper_2502_09334_b200 import KvPrecision, compress, decompress_into_paged
            packed = compress(kv, KvPrecision(4), 128)
            del kv
            decompress_into_paged(packed, rk, rv, slots)
            del packed
            same = torch.equal(kc, rk) and torch.equal(vc, rv)
            torch.cuda.synchronize()
            if not same:
                failures += 1
                print(f"MISMATCH {wl} rank={rank}", flush=True)
            elif ch.pair == 0:
                print(f"{wl}: whole decode cache bit-exact ({kc.numel() * 4} B compared, "
                      f"native pair={ch._pair is not None})", flush=True)
            del kc, vc, rk, rv
        dist.barrier()
        ch.close()
        del ch
        torch.cuda.empty_cache()
    f = _mp.total(failures, ctrl)
    if rank == 0:
        print(f"mp_fullsize_check failures={f}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if f else 0)


if __name__ == "__main__":
    main()
