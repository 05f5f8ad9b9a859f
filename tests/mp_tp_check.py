"""torchrun worker (4 ranks) for tests/test_gpu_multiproc.py::test_tp_regroup:
TP-sharded replicas with mismatched TP degrees -- every
decode rank's paged cache must equal the oracle on its own heads."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _mp  # noqa: E402
from oracle import kvq_oracle as O  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import TPHandoff  # noqa: E402


def main():
    rank, world, dev, ctrl, _ = _mp.init()
    L, H, D, bs = 4, 8, 128, 16
    failures = 0
    scenarios = [([0], [1, 2]), ([0, 1], [2]), ([0, 1], [2, 3]), ([3], [0, 1]), ([1, 2, 3, 0], [0, 2])]
    for si, (pr, dr) in enumerate(scenarios):
        for mode in ("pull", "pull_ldg"):
            tp = TPHandoff(L, 256, H, D, pr, dr, rank, world, ctrl, n_chunks=2, mode=mode)
            for epoch, T in enumerate((256, 100, 256)):
                seed = 31 * si + epoch
                kv_full = O.synthetic_kv(L, T, H, D, seed=seed)
                if rank in pr:
                    i = pr.index(rank)
                    hp = H // len(pr)
                    mine = np.ascontiguousarray(kv_full[:, :, :, i * hp:(i + 1) * hp])
                    tp.send(KVPlanes.dense(torch.from_numpy(mine).to(dev)), T)
                    torch.cuda.synchronize()
                if rank in dr:
                    j = dr.index(rank)
                    hd = H // len(dr)
                    nb = T // bs + 2
                    slots = O.synthetic_slots(T, bs, nb, seed=seed)
                    kc = torch.zeros((L, nb, bs, hd, D), dtype=torch.float16, device=dev)
                    vc = torch.zeros_like(kc)
                    tp.recv(KVPlanes.paged(kc, vc, torch.from_numpy(slots).to(dev)), T)
                    torch.cuda.synchronize()
                    sub = np.ascontiguousarray(kv_full[:, :, :, j * hd:(j + 1) * hd])
                    c, s, z = O.quant_pack(sub.reshape(-1, D), 4, 128)
                    rows = O.unpack_dequant(c, s, z, 4, 128, D).reshape(L, 2, T, hd, D)
                    okc = np.zeros((L, nb, bs, hd, D), np.float16); ovc = okc.copy()
                    O.scatter_paged(rows, slots, okc, ovc)
                    if not (np.array_equal(kc.cpu().numpy().view(np.uint16), okc.view(np.uint16))
                            and np.array_equal(vc.cpu().numpy().view(np.uint16), ovc.view(np.uint16))):
                        failures += 1
                        print(f"MISMATCH tp {pr}->{dr} mode={mode} rank={rank} T={T}", flush=True)
            dist.barrier()
            tp.close()
    # routing (the reference's x/y fractions, simulate.py:112-127): every
    # prefill rank sends a different request subset to each decode rank over
    # its own edge channel; decode ranks receive from both prefill ranks into
    # disjoint slots of one paged cache
    from paper_2502_09334_b200.transport import ChannelSpec, PairChannel
    P, Dr = [0, 1], [2, 3]
    edges = [(p, d) for p in P for d in Dr]
    chans = {e: PairChannel(ChannelSpec(L, 256, H, D, 4, 128, 2, "pull"), rank, world, ctrl,
                            edge=e) for e in edges}
    T_req = 64  # tokens per request; each prefill rank holds 4 requests
    nb = 2 * len(P) * T_req // bs + 4
    for epoch in range(3):
        if rank in P:
            i = P.index(rank)
            kv = O.synthetic_kv(L, 4 * T_req, H, D, seed=900 + 10 * epoch + i)
            kvd = torch.from_numpy(kv).to(dev)
            kc_src = kvd[:, 0]  # dense planes viewed as a "paged" source with token gather
            for j, d in enumerate(Dr):
                # requests 2j, 2j+1 of this prefill rank go to decode rank d
                toks = torch.arange(2 * j * T_req, (2 * j + 2) * T_req, device=dev)
                src = KVPlanes(kvd[:, 0], kvd[:, 1], kvd.stride(0), L, H, D, toks)
                chans[(rank, d)].send(src, 2 * T_req)
            torch.cuda.synchronize()
        if rank in Dr:
            j = Dr.index(rank)
            kc = torch.zeros((L, nb, bs, H, D), dtype=torch.float16, device=dev)
            vc = torch.zeros_like(kc)
            okc = np.zeros((L, nb, bs, H, D), np.float16); ovc = okc.copy()
            for i, p in enumerate(P):
                slots = np.arange(2 * T_req, dtype=np.int64) + (i * 2 * T_req)  # disjoint
                chans[(p, rank)].recv(KVPlanes.paged(kc, vc, torch.from_numpy(slots).to(dev)),
                                      2 * T_req)
                kv = O.synthetic_kv(L, 4 * T_req, H, D, seed=900 + 10 * epoch + i)
                sub = np.ascontiguousarray(kv[:, :, 2 * j * T_req:(2 * j + 2) * T_req])
                c, s_, z = O.quant_pack(sub.reshape(-1, D), 4, 128)
                O.scatter_paged(O.unpack_dequant(c, s_, z, 4, 128, D).reshape(sub.shape), slots,
                                okc, ovc)
            torch.cuda.synchronize()
            if not (np.array_equal(kc.cpu().numpy().view(np.uint16), okc.view(np.uint16)) and
                    np.array_equal(vc.cpu().numpy().view(np.uint16), ovc.view(np.uint16))):
                failures += 1
                print(f"MISMATCH routed rank={rank} epoch={epoch}", flush=True)
    dist.barrier()
    for ch in chans.values():
        ch.close()
    f = _mp.total(failures, ctrl)
    if rank == 0:
        print(f"mp_tp_check failures={f}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if f else 0)


if __name__ == "__main__":
    main()
