"""Host cost of enqueuing one fused hand-off (the alpha the CPU adds).

Two ranks (one pair).  Each rank times, per call, in a loop the GPU cannot
fall behind on (16-token hand-offs, queue depth 8, the partner running the
same loop):
  api      PairChannel.send / recv (the public call)
  native   the kvx_pair_send / kvx_pair_recv ctypes call with its arguments
           precomputed (no Python validation, no torch stream query)
  stream   torch.cuda.current_stream(device) alone
  check    ChannelSpec.check_planes alone

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/host_overhead.py
"""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_09334_b200.datapath import KVPlanes  # noqa: E402
from paper_2502_09334_b200.transport import ChannelSpec, PairChannel, exchange  # noqa: E402


def per_call(fn, n):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    rank = int(os.environ["RANK"])
    same = os.environ.get("KVX_MP_SAME_GPU") == "1"
    torch.cuda.set_device(0 if same else rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("gloo")
    L, H, D, T = 80, 8, 128, 16
    ch = PairChannel(ChannelSpec(L, 1024, H, D, 4, 128, 8, "pull", queue_depth=8), rank, 2)
    n = 200
    if ch.role == "prefill":
        kv = torch.randn((L, 2, T, H, D), device=dev).half()
        planes = KVPlanes.dense(kv)
        api = lambda: ch.send(planes, T)  # noqa: E731
        k, v = planes.ptrs(0)
        ph, ho = planes.window_args
        cs = torch.cuda.current_stream(dev).cuda_stream

        def native():
            ch.epoch += 1
            ch._pair_send(ch._pair, ch.epoch, k, v, planes.layer_stride, None, T, ph, ho,
                          ch._send_flags, cs)
    else:
        kc = torch.zeros((L, T // 16 + 4, 16, H, D), dtype=torch.float16, device=dev)
        planes = KVPlanes.paged(kc, torch.zeros_like(kc), torch.arange(T, device=dev))
        api = lambda: ch.recv(planes, T)  # noqa: E731
        k, v = planes.ptrs(0)
        ph, ho = planes.window_args
        cs = torch.cuda.current_stream(dev).cuda_stream
        sp = planes.slots_ptr

        def native():
            ch.epoch += 1
            ch._pair_recv(ch._pair, ch.epoch, k, v, planes.layer_stride, sp, T, ph, ho,
                          ch._recv_flags, cs)
    res = {}
    for name, fn in (("api", api), ("native", native)):
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        res[name] = round(per_call(fn, n), 2)
        torch.cuda.synchronize()
        dist.barrier()
    res["stream"] = round(per_call(lambda: torch.cuda.current_stream(dev), 10000), 2)
    res["check"] = round(per_call(lambda: ch.spec.check_planes(planes, T, "x"), 10000), 2)
    allr = exchange({ch.role: res})
    if rank == 0:
        print(json.dumps({"tokens": T, "us_per_call": {k: v for d in allr for k, v in d.items()}}))
    dist.barrier()
    ch.close()


if __name__ == "__main__":
    main()
