"""Small hand-off workload for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): K1, K3, K3-bulk (TMA + mbarrier ring), the
16-bit passthrough and the kivi kernels on one GPU."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import kvq_oracle as O  # noqa: E402
from paper_2502_09334_b200 import compress, decompress_into_paged  # noqa: E402
from paper_2502_09334_b200.kivi import compress_kivi, decompress_kivi_into_paged  # noqa: E402


def main():
    L, T, H, D, bs = 3, 300, 8, 128, 16
    kv = torch.from_numpy(O.synthetic_kv(L, T, H, D, seed=1)).cuda()
    nb = (T + bs - 1) // bs + 2
    slots = torch.from_numpy(O.synthetic_slots(T, bs, nb, seed=1)).cuda()
    slots[7] = -1
    kc = torch.zeros((L, nb, bs, H, D), dtype=torch.float16, device="cuda")
    vc = torch.zeros_like(kc)
    for bits in (2, 4, 8, 16):
        p = compress(kv, bits, 64 if bits != 16 else 128)
        decompress_into_paged(p, kc, vc, slots)
        if bits != 16:
            decompress_into_paged(p, kc, vc, slots, bulk=True)
    p = compress_kivi(kv, 4, 32, (100, 64, 136))
    decompress_kivi_into_paged(p, kc, vc, torch.arange(T, device="cuda"))
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
