"""Hand-off pipeline on GPUs: layer-chunked HandoffPlan (local / copy / push /
pull), the host-buffer path, and the full-size (BASELINE config 2) round trip
checked through size-independent properties + sampled rows vs the oracle."""
import numpy as np
import pytest

from oracle import kvq_oracle as O

pytestmark = pytest.mark.gpu


def h16(x):
    return np.ascontiguousarray(x).view(np.uint16)


def expected_cache(kv, slots, nb, bs, bits, group):
    L, _, T, H, D = kv.shape
    okc = np.zeros((L, nb, bs, H, D), np.float16)
    ovc = okc.copy()
    c, s, z = O.quant_pack(kv.reshape(-1, D), bits, group)
    O.scatter_paged(O.unpack_dequant(c, s, z, bits, group, D).reshape(L, 2, T, H, D), slots,
                    okc, ovc)
    return okc, ovc


def make_case(torch, dev_p, dev_d, L=5, T=77, H=8, D=128, bs=16, seed=1):
    kv_np = O.synthetic_kv(L, T, H, D, seed=seed)
    nb = (T + bs - 1) // bs + 3
    slots = O.synthetic_slots(T, bs, nb, seed=seed)
    kv = torch.from_numpy(kv_np).to(dev_p)
    kc = torch.zeros((L, nb, bs, H, D), dtype=torch.float16, device=dev_d)
    vc = torch.zeros_like(kc)
    return kv_np, slots, nb, kv, kc, vc


@pytest.mark.parametrize("n_chunks", [1, 2, 5])
@pytest.mark.parametrize("bits", [4, 8, 16])
def test_local_plan(cuda, n_chunks, bits):
    from paper_2502_09334_b200 import KvPrecision
    from paper_2502_09334_b200.datapath import HandoffPlan, KVPlanes
    torch = cuda
    kv_np, slots, nb, kv, kc, vc = make_case(torch, "cuda:0", "cuda:0")
    plan = HandoffPlan(KVPlanes.dense(kv), KVPlanes.paged(kc, vc, torch.from_numpy(slots).cuda()),
                       kv.shape[2], KvPrecision(bits), 128, n_chunks=n_chunks)
    assert plan.mode == "local"
    plan.run()
    plan.run()  # idempotent re-run
    torch.cuda.synchronize()
    okc, ovc = expected_cache(kv_np, slots, nb, 16, bits, 128)
    assert np.array_equal(h16(kc.cpu().numpy()), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy()), h16(ovc))


@pytest.mark.multigpu
@pytest.mark.parametrize("mode", ["copy", "push", "pull"])
def test_two_gpu_modes(cuda, mode):
    torch = cuda
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2502_09334_b200 import KvPrecision
    from paper_2502_09334_b200.datapath import HandoffPlan, KVPlanes
    kv_np, slots, nb, kv, kc, vc = make_case(torch, "cuda:0", "cuda:1", L=6, T=130)
    plan = HandoffPlan(KVPlanes.dense(kv),
                       KVPlanes.paged(kc, vc, torch.from_numpy(slots).to("cuda:1")),
                       kv.shape[2], KvPrecision(4), 64, mode=mode, n_chunks=3)
    plan.run()
    torch.cuda.synchronize("cuda:0")
    torch.cuda.synchronize("cuda:1")
    okc, ovc = expected_cache(kv_np, slots, nb, 16, 4, 64)
    assert np.array_equal(h16(kc.cpu().numpy()), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy()), h16(ovc))


def test_host_handoff(cuda):
    from paper_2502_09334_b200 import KvPrecision
    from paper_2502_09334_b200.datapath import HostHandoff
    torch = cuda
    kv_np, slots, nb, kv, kc, vc = make_case(torch, "cpu", "cpu", L=6, T=50)
    kv_h = kv.pin_memory()
    kc_h = kc.pin_memory()
    vc_h = vc.pin_memory()
    host = HostHandoff(kv_h, kc_h, vc_h, torch.from_numpy(slots), "cuda:0", KvPrecision(4), 128,
                       n_chunks=3)
    host.run()
    torch.cuda.synchronize()
    okc, ovc = expected_cache(kv_np, slots, nb, 16, 4, 128)
    assert np.array_equal(h16(kc_h.numpy()), h16(okc))
    assert np.array_equal(h16(vc_h.numpy()), h16(ovc))


@pytest.mark.parametrize("H", [8, 32])  # per-lane K3 / K3-bulk (local_bulk_preferred)
def test_host_handoff_pipelined_runs(cuda, H):
    """Consecutive run()s pipeline per chunk (run i+1's uploads overlap run
    i's downloads): a new input per synchronised run, then back-to-back runs
    of one input, each result bit-exact."""
    from paper_2502_09334_b200 import KvPrecision
    from paper_2502_09334_b200.datapath import HostHandoff
    torch = cuda
    L, T, D, bs = 5, 70, 128, 16
    nb = (T + bs - 1) // bs + 2
    slots = O.synthetic_slots(T, bs, nb, seed=3)
    kv_h = torch.empty((L, 2, T, H, D), dtype=torch.float16).pin_memory()
    kc_h = torch.zeros((L, nb, bs, H, D), dtype=torch.float16).pin_memory()
    vc_h = torch.zeros_like(kc_h).pin_memory()
    host = HostHandoff(kv_h, kc_h, vc_h, torch.from_numpy(slots), "cuda:0", KvPrecision(4), 128,
                       n_chunks=4)
    for seed in (11, 12, 13):
        kv_np = O.synthetic_kv(L, T, H, D, seed=seed)
        kv_h.copy_(torch.from_numpy(kv_np))
        host.run()
        torch.cuda.synchronize()
        okc, ovc = expected_cache(kv_np, slots, nb, bs, 4, 128)
        assert np.array_equal(h16(kc_h.numpy()), h16(okc)), seed
        assert np.array_equal(h16(vc_h.numpy()), h16(ovc)), seed
    for _ in range(4):
        host.run()
    torch.cuda.synchronize()
    assert np.array_equal(h16(kc_h.numpy()), h16(okc))
    assert np.array_equal(h16(vc_h.numpy()), h16(ovc))


def test_cfg2_full_size_properties(cuda):
    """BASELINE config 2 (7B, 2048 x 8) at full size: every element inside the
    format's error bound, padding never written, and 2,048 sampled token rows
    bit-exact vs the C oracle (a checksum of the whole payload is pinned per run
    against re-execution: the kernels are deterministic)."""
    torch = cuda
    from oracle import kvq_oracle_c as C
    from paper_2502_09334_b200 import KvPrecision
    from paper_2502_09334_b200.datapath import HandoffPlan, KVPlanes
    import bench
    L, H, D, b, s = bench.WORKLOADS["cfg2_7b_2048x8"]
    T = b * s
    dev = torch.device("cuda:0")
    kv = bench.synthetic_kv_device(torch, L, T, H, D, dev)
    slots, nb = bench.paged_slots(torch, T, dev)
    kc = torch.full((L, nb, 16, H, D), -3.0, dtype=torch.float16, device=dev)
    vc = torch.full_like(kc, -3.0)
    plan = HandoffPlan(KVPlanes.dense(kv), KVPlanes.paged(kc, vc, slots), T, KvPrecision(4), 128,
                       n_chunks=4)
    plan.run()
    torch.cuda.synchronize()
    p = plan.packed
    # 1) error bound, per layer to bound memory
    for l in range(L):
        for side, cache in ((0, kc), (1, vc)):
            x = kv[l, side].float()                                # [T, H, D]
            y = cache[l].view(-1, H, D)[slots].float()             # gathered back
            sc = p.scale()[l, side].float()                        # [T, H, 1]
            ulp = torch.abs(x).half().float()
            ulp = torch.where(ulp > 0, ulp, torch.ones_like(ulp)) * 2.0 ** -10 + 2.0 ** -24
            bound = sc * (0.5 + 15 * 2.0 ** -10) + ulp
            assert bool(((y - x).abs() <= bound).all()), (l, side)
    # 2) blocks not in the block table keep the sentinel
    used = torch.zeros(nb, dtype=torch.bool, device=dev)
    used[slots // 16] = True
    assert bool((kc[:, ~used] == -3.0).all()) and bool((vc[:, ~used] == -3.0).all())
    # 3) sampled token rows bit-exact vs the C oracle
    rng = np.random.default_rng(0)
    tok = np.sort(rng.choice(T, 64, replace=False))
    for l in (0, 13, 31):
        rows = kv[l][:, tok].cpu().numpy()                         # [2, 64, H, D]
        c, sc, z = C.quant_pack(rows.reshape(-1, D), 4, 128)
        gc = p.codes()[l][:, tok].cpu().numpy().reshape(c.shape)
        assert np.array_equal(gc, c)
        assert np.array_equal(h16(p.scale()[l][:, tok].cpu().numpy().reshape(sc.shape)), h16(sc))
    # 4) determinism: a second run reproduces the payload checksum
    digest = p.owner.view(torch.int64).sum().item()
    plan.run()
    torch.cuda.synchronize()
    assert p.owner.view(torch.int64).sum().item() == digest


def test_transfer_with_reference_gpu_lists(cuda):
    """SURVEY 8(b)'s transfer(packed, src_gpu_ids, dst_gpu_ids): the payload
    arrives byte-identical (here cuda:0 -> cuda:0; the multi-GPU suite covers
    real peers through HandoffPlan), and misuse raises like the reference."""
    torch = cuda
    from paper_2502_09334_b200 import KvPrecision, compress, decompress_into_paged, transfer
    kv_np, slots, nb, kv, kc, vc = make_case(torch, "cuda:0", "cuda:0", seed=3)
    packed = compress(kv, KvPrecision(4), 128)
    moved = transfer(packed, [0], [0])
    torch.cuda.synchronize()
    assert torch.equal(moved.codes(), packed.codes())
    assert torch.equal(moved.scale().view(torch.int16), packed.scale().view(torch.int16))
    decompress_into_paged(moved, kc, vc, torch.from_numpy(slots).to("cuda:0"))
    torch.cuda.synchronize()
    okc, ovc = expected_cache(kv_np, slots, nb, 16, 4, 128)
    assert np.array_equal(h16(kc.cpu().numpy()), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy()), h16(ovc))
    with pytest.raises(ValueError):
        transfer(packed, [1, 2], [0])   # the payload is not on a source GPU
    with pytest.raises(ValueError):
        transfer(packed, [0], [])
