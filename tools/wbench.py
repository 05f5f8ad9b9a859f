"""HBM ceilings by traffic mix on one B200, with torch's own kernels (no math):
pure write (fill), pure read (sum), copy (1:1), and K3's 1 read : 4 write mix
(a copy of a 1/4-size source repeated into a 4x destination).  CUDA events,
best of 10; bytes = algorithmic reads + writes."""
import json
import torch


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


N = 4 << 30  # 4 Gi fp16 = 8 GiB
x = torch.empty(N, dtype=torch.float16, device="cuda")
y = torch.empty(N, dtype=torch.float16, device="cuda")
q = torch.empty(N // 4, dtype=torch.float16, device="cuda").fill_(1)
out = {}
ms = t(lambda: x.fill_(0.5)); out["write (fill)"] = 2 * N / ms / 1e9
ms = t(lambda: x.sum(dtype=torch.float32)); out["read (sum)"] = 2 * N / ms / 1e9
ms = t(lambda: y.copy_(x)); out["copy 1:1"] = 4 * N / ms / 1e9
yv = y.view(4, N // 4)
ms = t(lambda: yv.copy_(q.expand(4, N // 4))); out["1 read : 4 write (broadcast copy)"] = (2 * N // 4 + 2 * N) / ms / 1e9
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
