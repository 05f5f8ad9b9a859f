"""Single-process, two-GPU hand-off for ncu NVLink counters (one kernel of
interest per run; no in-kernel cross-GPU waits, so ncu replay is safe):

  pull      K3-bulk on GPU 1 reading GPU 0's payload (TMA cp.async.bulk)
  pull_ldg  per-lane K3 on GPU 1 reading GPU 0's payload (LDG.128)
  push      K1 on GPU 0 storing the payload into GPU 1 (STG over NVLink)

  python tools/nvlink_profile.py pull [workload]   (default: config 4 pair, 70B GQA)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench as B  # noqa: E402
from paper_2502_09334_b200 import KvPrecision  # noqa: E402
from paper_2502_09334_b200.datapath import HandoffPlan, KVPlanes  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "pull"
    wl = sys.argv[2] if len(sys.argv) > 2 else "cfg4_70b_gqa_pair"
    L, H, D, b, s = B.WORKLOADS[wl]
    T = b * s
    p, d = torch.device("cuda", 0), torch.device("cuda", 1)
    kv = B.synthetic_kv_device(torch, L, T, H, D, p)
    slots, nb = B.paged_slots(torch, T, d)
    kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=d)
    vc = torch.zeros_like(kc)
    plan = HandoffPlan(KVPlanes.dense(kv), KVPlanes.paged(kc, vc, slots), T, KvPrecision(4), 128,
                       mode="push" if mode == "push" else "pull", n_chunks=1,
                       bulk=(mode == "pull"))
    for _ in range(3):
        plan.run()
    torch.cuda.synchronize(p)
    torch.cuda.synchronize(d)
    print(f"{mode}: payload {plan.layout.wire_bytes} B, fp16 {plan.layout.fp16_bytes} B")


if __name__ == "__main__":
    main()
