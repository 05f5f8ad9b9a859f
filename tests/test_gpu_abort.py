"""Failure detection of the hand-off: a pull
whose doorbells never ring must not trap or hang the GPU.  On one GPU:

* a spinning K3-bulk is aborted from the host (control block abort word):
  the kernel exits, the status says ABORTED, the CUDA context keeps working;
* a wait that outlives the channel timeout exits with status TIMEOUT;
* poisoned doorbells (PairChannel.abort releasing front-end waits) read as
  an abort, and a K1 waiting for its queue slot gives up the same way.
"""
import time

import numpy as np
import pytest

from oracle import kvq_oracle as O

pytestmark = pytest.mark.gpu


def _case(torch, L=4, T=64, H=8, D=128):
    from paper_2502_09334_b200.datapath import KVPlanes, PackedLayout, alloc_packed
    dev = torch.device("cuda", 0)
    lay = PackedLayout(L, T, H, D, 4, 128)
    payload = alloc_packed(lay, dev)
    nb = T // 16 + 2
    kc = torch.zeros((L, nb, 16, H, D), dtype=torch.float16, device=dev)
    vc = torch.zeros_like(kc)
    slots = torch.from_numpy(O.synthetic_slots(T, 16, nb, seed=3)).to(dev)
    return lay, payload, KVPlanes.paged(kc, vc, slots), kc


def _pull(torch, lay, payload, dst, flags, done, ctl, value=1):
    from paper_2502_09334_b200.datapath import dequant_scatter_layers
    fp = flags.data_ptr()
    s = torch.cuda.Stream()
    dequant_scatter_layers(payload, dst, 0, lay.n_layers, s, ready=(fp, value, 1),
                           done=(done.data_ptr(), fp + 4 * 100), ctl=ctl.ptr)
    return s


def test_abort_spinning_pull(cuda):
    torch = cuda
    from paper_2502_09334_b200 import _lib
    from paper_2502_09334_b200.transport import Ctl
    lay, payload, dst, kc = _case(torch)
    flags = torch.zeros(128, dtype=torch.int32, device="cuda:0")   # never rung
    done = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    ctl = Ctl(timeout_s=30.0)
    s = _pull(torch, lay, payload, dst, flags, done, ctl)
    time.sleep(0.2)
    assert not s.query(), "the pull should still be waiting for its doorbells"
    t0 = time.perf_counter()
    ctl.abort()
    s.synchronize()  # returns: the kernel wound down
    assert time.perf_counter() - t0 < 5.0
    assert ctl.status == _lib.KVX_STATUS_ABORTED
    assert int(flags[100].item()) == 0, "an aborted pull must not free the slot"
    assert int(done.item()) == 0, "completion counter left non-zero"
    assert not kc.any(), "an aborted pull wrote the cache"
    # the context survives: ordinary work still runs
    x = torch.arange(1 << 20, device="cuda:0", dtype=torch.float32)
    assert float(x.sum().item()) == float(np.arange(1 << 20, dtype=np.float64).sum())
    ctl.free()


def test_pull_wait_times_out(cuda):
    torch = cuda
    from paper_2502_09334_b200 import _lib
    from paper_2502_09334_b200.transport import Ctl
    lay, payload, dst, kc = _case(torch)
    flags = torch.zeros(128, dtype=torch.int32, device="cuda:0")
    done = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    ctl = Ctl(timeout_s=0.3)
    t0 = time.perf_counter()
    _pull(torch, lay, payload, dst, flags, done, ctl).synchronize()
    dt = time.perf_counter() - t0
    assert 0.25 < dt < 10.0, dt
    assert ctl.status == _lib.KVX_STATUS_TIMEOUT
    ctl.free()


def test_poisoned_doorbell_reads_as_abort(cuda):
    torch = cuda
    from paper_2502_09334_b200 import _lib
    from paper_2502_09334_b200.transport import POISON, Ctl
    lay, payload, dst, kc = _case(torch)
    flags = torch.zeros(128, dtype=torch.int32, device="cuda:0")
    flags[:64] = POISON  # what PairChannel.abort() writes into its own page
    done = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    ctl = Ctl(timeout_s=30.0)
    _pull(torch, lay, payload, dst, flags, done, ctl, value=5).synchronize()
    assert ctl.status == _lib.KVX_STATUS_ABORTED
    assert not kc.any()
    ctl.free()


def test_k1_slot_wait_gives_up(cuda):
    """K1 with doorbells waiting for a queue slot the decode side never frees."""
    torch = cuda
    from paper_2502_09334_b200 import _lib
    from paper_2502_09334_b200.datapath import KVPlanes, _stream_ptr
    from paper_2502_09334_b200.transport import Ctl
    lay, payload, _, _ = _case(torch)
    kv = torch.from_numpy(O.synthetic_kv(lay.n_layers, lay.n_tokens, 8, 128, seed=1)).cuda()
    src = KVPlanes.dense(kv)
    flags = torch.zeros(128, dtype=torch.int32, device="cuda:0")
    counters = torch.zeros(65, dtype=torch.int32, device="cuda:0")
    ctl = Ctl(timeout_s=0.3)
    s = torch.cuda.Stream()
    k, v = src.ptrs(0)
    c0, s0, z0 = payload.ptrs(0)
    # the slot's 2nd use (v = 2) waits free >= 1; free stays 0
    _lib.call("kvx_quant_pack_signal", k, v, src.layer_stride, None, lay.n_layers, lay.n_tokens,
              8, 128, 128, 4, c0, s0, z0, lay.layer_stride, *src.window_args,
              counters.data_ptr(), flags.data_ptr(), 1, 2, flags.data_ptr() + 400, 1, ctl.ptr,
              _stream_ptr(s))
    s.synchronize()
    assert ctl.status == _lib.KVX_STATUS_TIMEOUT
    assert not flags[:64].any(), "a K1 that never got its slot rang a doorbell"
    ctl.free()
