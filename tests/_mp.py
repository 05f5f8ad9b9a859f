"""Process-group setup shared by the torchrun workers (tests/mp_*.py).

KVX_MP_SAME_GPU=1 puts every rank on cuda:0: two (or four) processes, each
with its own CUDA context time-sliced on one B200, talking over CUDA IPC --
the transport's whole protocol (IPC maps, doorbells, queue slots, in-kernel
waits) on a 1-GPU box.  NCCL cannot pair two ranks on one device, so there
the default group is gloo and NCCL-only modes are skipped."""
import os

import torch
import torch.distributed as dist


def init():
    """(rank, world, device, control group, same_gpu)."""
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    same_gpu = os.environ.get("KVX_MP_SAME_GPU", "0") == "1"
    local = 0 if same_gpu else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if same_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    return rank, world, dev, ctrl, same_gpu


def total(failures: int, ctrl) -> int:
    f = torch.tensor([failures])
    dist.all_reduce(f, group=ctrl)
    return int(f.item())


def local_reference(kv, kc_shape, slots, bits=4, group=128):
    """The decode-side cache a hand-off of ``kv`` must produce, computed on
    this GPU by the local K1 -> K3 round trip (itself bit-exact against the
    oracle in tests/test_gpu_parity.py) -- a whole-tensor check at sizes the
    CPU oracle cannot finish in seconds."""
    from paper_2502_09334_b200 import KvPrecision, compress, decompress_into_paged
    rk = torch.zeros(kc_shape, dtype=torch.float16, device=kv.device)
    rv = torch.zeros_like(rk)
    packed = compress(kv, KvPrecision(bits), group)
    decompress_into_paged(packed, rk, rv, slots)
    return rk, rv
