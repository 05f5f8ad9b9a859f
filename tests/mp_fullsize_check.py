"""torchrun worker for tests/test_gpu_multiproc.py::test_fullsize_pairs: the
bench's pair workloads at FULL size through the default transport (fused
pull, CUDA-graph replayed), checked on sampled rows against the C oracle:
3 layers x 32 tokens of the last hand-off, bit-exact.  Exits non-zero on any
mismatch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench as B  # noqa: E402
from oracle import kvq_oracle_c as C  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel, exchange  # noqa: E402


def main():
    workloads = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg4_70b_gqa_pair"]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    failures = 0
    for wl in workloads:
        L, H, D, b, s = B.WORKLOADS[wl]
        T = b * s
        ch = PairChannel(ChannelSpec(L, T, H, D, 4, 128, 8, "pull"), rank, world,
                         control_group=ctrl)
        if ch.role == "prefill":
            kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=ch.pair)
            for _ in range(3):  # eager, capture, replay
                ch.send(KVPlanes.dense(kv), T)
            torch.cuda.synchronize()
            toks = np.sort(np.random.default_rng(7).choice(T, 32, replace=False))
            layers = sorted({0, L // 2, L - 1})
            mine = kv[layers][:, :, torch.from_numpy(toks).to(dev)].cpu().numpy()
        else:
            slots, nb = B.paged_slots(torch, T, dev, seed=ch.pair)
            kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
            vc = torch.zeros_like(kc)
            for _ in range(3):
                ch.recv(KVPlanes.paged(kc, vc, slots), T)
            torch.cuda.synchronize()
            toks = np.sort(np.random.default_rng(7).choice(T, 32, replace=False))
            layers = sorted({0, L // 2, L - 1})
            sl = slots[torch.from_numpy(toks).to(dev)]
            mine = torch.stack([kc[layers].reshape(len(layers), -1, H, D)[:, sl],
                                vc[layers].reshape(len(layers), -1, H, D)[:, sl]], 1).cpu().numpy()
        allv = exchange(mine, ctrl)
        if ch.role == "decode":
            src = allv[ch.peer]
            c, sc, z = C.quant_pack(np.ascontiguousarray(src).reshape(-1, D), 4, 128)
            want = C.unpack_dequant(c, sc, z, 4, 128, D).reshape(src.shape)
            if not np.array_equal(want.view(np.uint16), mine.view(np.uint16)):
                failures += 1
                print(f"MISMATCH {wl} rank={rank}", flush=True)
            elif ch.pair == 0:
                print(f"{wl}: sampled rows bit-exact (graphs={ch.graphs})", flush=True)
        dist.barrier()
        ch.close()
        del ch
        torch.cuda.empty_cache()
    f = torch.tensor([failures], device=dev)
    dist.all_reduce(f)
    if rank == 0:
        print(f"mp_fullsize_check failures={int(f.item())}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if f.item() else 0)


if __name__ == "__main__":
    main()
