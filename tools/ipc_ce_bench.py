"""Copy-engine pulls across processes (CUDA IPC), vs the in-process ceiling
in tools/nvlink_bench.cu: rank 1 reads 1 GiB of rank 0's IPC buffer with
1/2/4/8 cudaMemcpyPeerAsync calls spread over as many streams.
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ipc_ce_bench.py"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_09334_b200 import _lib  # noqa: E402
from paper_2502_09334_b200.transport import IpcBuffer, exchange, ipc_open  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(rank)
    n = 1 << 30
    buf = IpcBuffer(n)
    hs = exchange(buf.handle())
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    if rank == 1:
        peer = ipc_open(hs[0])
        out = {}
        for k in (1, 2, 4, 8):
            streams = [torch.cuda.Stream() for _ in range(k)]
            cur = torch.cuda.current_stream()

            def go():
                step = n // k
                for i, s in enumerate(streams):
                    s.wait_stream(cur)
                    _lib.call("kvx_copy_peer", dst.data_ptr() + i * step, 1, peer + i * step, 1,
                              step, s.cuda_stream)
                for s in streams:
                    cur.wait_stream(s)

            go()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(5):
                a.record(); go(); b.record(); torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b))
            out[f"ce_pull_ipc_{k}streams_GBps"] = round(n / (best * 1e-3) / 1e9, 1)
        print(json.dumps(out), flush=True)
    dist.barrier()


if __name__ == "__main__":
    main()
