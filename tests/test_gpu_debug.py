"""The KVX_DEBUG build (`python -m paper_2502_09334_b200.build --variant debug
KVX_DEBUG`): the sanitizer stand-in while compute-sanitizer is closed on the
pool.  Device-side checks: every token position a kernel reads or writes lies
inside the plane the caller's layer stride describes, and no doorbell is ever
ahead of the sequence value awaited.  Run in subprocesses: a failed check is
a __trap (a sticky CUDA error)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_SO = os.path.join(ROOT, "paper_2502_09334_b200", "_kvx_debug.so")

GOOD = r'''
import sys, torch, numpy as np
sys.path.insert(0, {root!r})
from oracle import kvq_oracle as O
from paper_2502_09334_b200 import KvPrecision, compress, decompress_into_paged
dev = torch.device("cuda", 0)
L, T, H, D, bs = 4, 100, 8, 128, 16
kv = torch.from_numpy(O.synthetic_kv(L, T, H, D, seed=1)).to(dev)
nb = (T + bs - 1) // bs + 2
slots = torch.from_numpy(O.synthetic_slots(T, bs, nb, seed=1)).to(dev)
kc = torch.zeros((L, nb, bs, H, D), dtype=torch.float16, device=dev)
vc = torch.zeros_like(kc)
decompress_into_paged(compress(kv, KvPrecision(4), 128), kc, vc, slots)
{tail}
torch.cuda.synchronize()
print("debug build ok")
'''


def _run(tail: str):
    env = dict(os.environ, KVX_LIB=DEBUG_SO)
    code = GOOD.format(root=ROOT, tail=tail)
    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                          timeout=300, env=env)


@pytest.fixture(scope="module")
def debug_so(cuda):
    if not os.path.exists(DEBUG_SO):
        from paper_2502_09334_b200 import build
        build.build(variant="debug", defines=("KVX_DEBUG",))
    return DEBUG_SO


@pytest.mark.gpu
def test_debug_build_passes_valid_handoffs(debug_so):
    r = _run("")
    assert r.returncode == 0 and "debug build ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_debug_build_traps_out_of_range_slot(debug_so):
    """A slot past the cache (the C-ABI cannot see the cache's size; the debug
    build derives it from the layer stride) is caught on the device."""
    tail = ("bad = slots.clone(); bad[7] = nb * bs + 5\n"
            "decompress_into_paged(compress(kv, KvPrecision(4), 128), kc, vc, bad)")
    r = _run(tail)
    assert r.returncode != 0, r.stdout
    out = r.stdout + r.stderr
    # the device printf, or at least the trap it raises (the printf buffer is
    # flushed at the failing synchronize on current drivers)
    assert "kvx debug: token 7 -> position" in out or "illegal instruction" in out, out[-2000:]
