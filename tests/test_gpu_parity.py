"""GPU parity: K1 (quant+pack) and K3 (dequant+paged scatter) through the C-ABI
vs the CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): packed codes bit-exact; scale/zero bit-exact
(stricter than the 1-ulp allowance); dequantised K/V bit-exact with the
oracle's single-rounding definition (stricter than a max-abs tolerance; the
tolerance the format guarantees vs the fp16 input is checked separately).
"""
import numpy as np
import pytest

from oracle import kvq_oracle as O

pytestmark = pytest.mark.gpu


def h16(x):
    return np.ascontiguousarray(x).view(np.uint16)


def run_k1(torch, kv_np, bits, group):
    from paper_2502_09334_b200 import compress
    kv = torch.from_numpy(kv_np).cuda()
    p = compress(kv, bits, group)
    torch.cuda.synchronize()
    return p


def oracle_payload(kv_np, bits, group):
    L, _, T, H, D = kv_np.shape
    c, s, z = O.quant_pack(kv_np.reshape(-1, D), bits, group)
    if bits == 16:
        return c.reshape(L, 2, T, H, -1), None, None
    ng = D // group
    return (c.reshape(L, 2, T, H, -1), s.reshape(L, 2, T, H, ng), z.reshape(L, 2, T, H, ng))


SHAPES = [  # (L, T, H, D)
    (1, 1, 1, 128),
    (3, 300, 8, 128),    # several bulk spans per layer, partial last span
    (2, 3, 8, 128),
    (3, 17, 32, 128),
    (2, 64, 40, 128),    # 13B head count (non power of two)
    (4, 33, 8, 64),      # head_dim 64
    (2, 5, 6, 256),      # head_dim 256
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bits", [2, 4, 8, 16])
@pytest.mark.parametrize("group", [32, 64, 128])
def test_quant_pack_bit_exact(cuda, shape, bits, group):
    L, T, H, D = shape
    if bits == 16 and group != 128:
        pytest.skip("16-bit is passthrough")
    if D % group:
        pytest.skip("group must divide head_dim")
    kv = O.synthetic_kv(L, T, H, D, seed=L * 100 + T)
    p = run_k1(cuda, kv, bits, group)
    oc, os_, oz = oracle_payload(kv, bits, group)
    assert np.array_equal(p.codes().cpu().numpy(), oc)
    if bits != 16:
        assert np.array_equal(h16(p.scale().cpu().numpy()), h16(os_))
        assert np.array_equal(h16(p.zero().cpu().numpy()), h16(oz))


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_edge_case_groups(cuda, bits):
    """Hand-built groups (ramp, constant, +-0, +-65504, subnormals, outlier)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "groups.npz"))
    x = g["x"]  # [8, 128]
    kv = np.broadcast_to(x.reshape(1, 1, 8, 1, 128), (1, 2, 8, 1, 128)).copy()
    p = run_k1(cuda, kv, bits, 128)
    codes = p.codes().cpu().numpy().reshape(2, 8, -1)
    assert np.array_equal(codes[0], g[f"codes{bits}"]) and np.array_equal(codes[1], g[f"codes{bits}"])
    assert np.array_equal(h16(p.scale().cpu().numpy().reshape(2, 8)[0]), h16(g[f"scale{bits}"][:, 0]))
    assert np.array_equal(h16(p.zero().cpu().numpy().reshape(2, 8)[0]), h16(g[f"zero{bits}"][:, 0]))


def random_bit_patterns(rng, shape):
    x = rng.integers(0, 0x10000, size=shape, dtype=np.uint16).view(np.float16)
    return np.where(np.isfinite(x), x, np.float16(0)).astype(np.float16)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_random_bit_patterns_bit_exact(cuda, bits):
    """Every finite fp16 (subnormals, huge ranges) -- exercises clamping/saturation."""
    rng = np.random.default_rng(bits)
    kv = random_bit_patterns(rng, (2, 2, 50, 8, 128))
    from paper_2502_09334_b200 import decompress_into_paged
    p = run_k1(cuda, kv, bits, 64)
    oc, os_, oz = oracle_payload(kv, bits, 64)
    assert np.array_equal(p.codes().cpu().numpy(), oc)
    assert np.array_equal(h16(p.scale().cpu().numpy()), h16(os_))
    kc = cuda.zeros((2, 4, 16, 8, 128), dtype=cuda.float16, device="cuda")
    vc = cuda.zeros_like(kc)
    slots = cuda.arange(50, dtype=cuda.int64, device="cuda")
    decompress_into_paged(p, kc, vc, slots)
    want = O.unpack_dequant(oc.reshape(-1, oc.shape[-1]), os_.reshape(-1, 2), oz.reshape(-1, 2),
                            bits, 64, 128).reshape(2, 2, 50, 8, 128)
    got_k = kc.view(2, 64, 8, 128)[:, :50].cpu().numpy()
    got_v = vc.view(2, 64, 8, 128)[:, :50].cpu().numpy()
    assert np.array_equal(h16(got_k), h16(want[:, 0])) and np.array_equal(h16(got_v), h16(want[:, 1]))
    assert np.isfinite(got_k).all()


def paged_case(torch, L, T, H, D, bs, nb, seed, pad=()):
    slots = O.synthetic_slots(T, bs, nb, seed=seed)
    for i in pad:
        slots[i] = -1
    sentinel = np.float16(-7.0)
    kc = torch.full((L, nb, bs, H, D), float(sentinel), dtype=torch.float16, device="cuda")
    vc = torch.full_like(kc, float(sentinel))
    return slots, kc, vc


@pytest.mark.parametrize("bulk", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bits", [2, 4, 8, 16])
def test_dequant_scatter_paged_bit_exact(cuda, shape, bits, bulk):
    """K3 (per-lane loads) and K3-bulk (TMA cp.async.bulk staging)."""
    from paper_2502_09334_b200 import decompress_into_paged
    L, T, H, D = shape
    group = 64 if D == 64 else 128
    kv = O.synthetic_kv(L, T, H, D, seed=7 + T)
    bs, nb = 16, (T + 15) // 16 + 3
    slots, kc, vc = paged_case(cuda, L, T, H, D, bs, nb, seed=T, pad=(0,) if T > 2 else ())
    p = run_k1(cuda, kv, bits, group)
    decompress_into_paged(p, kc, vc, cuda.from_numpy(slots).cuda(), bulk=bulk)
    cuda.cuda.synchronize()
    # oracle: same dequant + scatter into sentinel-filled caches
    okc = np.full((L, nb, bs, H, D), -7.0, np.float16); ovc = okc.copy()
    c, s, z = O.quant_pack(kv.reshape(-1, D), bits, group)
    rows = O.unpack_dequant(c, s, z, bits, group, D).reshape(L, 2, T, H, D)
    O.scatter_paged(rows, slots, okc, ovc)
    assert np.array_equal(h16(kc.cpu().numpy()), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy()), h16(ovc))


def test_paged_source_gather(cuda):
    """compress_paged gathers the prefill replica's paged cache by slot."""
    from paper_2502_09334_b200 import compress_paged
    L, T, H, D, bs, nb = 3, 45, 8, 128, 16, 6
    kv = O.synthetic_kv(L, T, H, D, seed=4)
    slots = O.synthetic_slots(T, bs, nb, seed=4)
    kc = np.zeros((L, nb * bs, H, D), np.float16); vc = kc.copy()
    kc[:, slots] = kv[:, 0]; vc[:, slots] = kv[:, 1]
    t = cuda
    p = compress_paged(t.from_numpy(kc.reshape(L, nb, bs, H, D)).cuda(),
                       t.from_numpy(vc.reshape(L, nb, bs, H, D)).cuda(),
                       t.from_numpy(slots).cuda(), 4, 128)
    oc, os_, oz = oracle_payload(kv, 4, 128)
    assert np.array_equal(p.codes().cpu().numpy(), oc)
    assert np.array_equal(h16(p.zero().cpu().numpy()), h16(oz))


def test_empty_handoff(cuda):
    from paper_2502_09334_b200 import compress, decompress_into_paged
    kv = cuda.zeros((2, 2, 0, 8, 128), dtype=cuda.float16, device="cuda")
    p = compress(kv, 4)
    kc = cuda.zeros((2, 1, 16, 8, 128), dtype=cuda.float16, device="cuda")
    decompress_into_paged(p, kc, kc.clone(), cuda.zeros(0, dtype=cuda.int64, device="cuda"))
    cuda.cuda.synchronize()
    assert not kc.any()


def test_cfg1_full_bit_exact(cuda):
    """BASELINE config 1 (7B, 512 tokens x batch 1) end to end on one GPU."""
    from paper_2502_09334_b200 import compress, decompress_into_paged
    from oracle import kvq_oracle_c as C
    L, T, H, D = 32, 512, 32, 128
    kv = O.synthetic_kv(L, T, H, D, seed=0)
    p = compress(cuda.from_numpy(kv).cuda(), 4, 128)
    c, s, z = C.quant_pack(kv.reshape(-1, D), 4, 128)
    assert np.array_equal(p.codes().cpu().numpy().reshape(c.shape), c)
    assert np.array_equal(h16(p.scale().cpu().numpy().reshape(s.shape)), h16(s))
    assert np.array_equal(h16(p.zero().cpu().numpy().reshape(z.shape)), h16(z))
    slots = O.synthetic_slots(T, 16, 64, seed=0)
    kc = cuda.zeros((L, 64, 16, H, D), dtype=cuda.float16, device="cuda")
    vc = cuda.zeros_like(kc)
    decompress_into_paged(p, kc, vc, cuda.from_numpy(slots).cuda())
    okc = np.zeros((L, 64, 16, H, D), np.float16); ovc = okc.copy()
    C.dequant_scatter_paged(c, s, z, slots, L, T, H, D, 128, 4, okc, ovc)
    assert np.array_equal(h16(kc.cpu().numpy()), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy()), h16(ovc))


def test_invalid_args_raise(cuda):
    from paper_2502_09334_b200 import compress
    kv = cuda.zeros((1, 2, 4, 1, 128), dtype=cuda.float16, device="cuda")
    with pytest.raises(ValueError):
        compress(kv, 3)
    with pytest.raises(ValueError):
        compress(kv, 4, 96)
    with pytest.raises(ValueError):
        compress(kv.float(), 4)


@pytest.mark.parametrize("bulk", [False, True])
@pytest.mark.parametrize("bits", [4, 8])
def test_head_windows(cuda, bits, bulk):
    """TP head shards: pack heads [2, 5) of an 8-head source, scatter them to
    heads [1, 4) of a 6-head cache (SURVEY 8(e) head-range remap)."""
    from paper_2502_09334_b200.datapath import (KVPlanes, PackedLayout, alloc_packed,
                                                dequant_scatter_layers, quant_pack_layers)
    torch = cuda
    L, T, H, D, bs = 3, 70, 8, 128, 16
    kv = O.synthetic_kv(L, T, H, D, seed=11)
    src = KVPlanes.dense(torch.from_numpy(kv).cuda()).window(2, 3)
    lay = PackedLayout(L, T, 3, D, bits, 128)
    p = alloc_packed(lay, "cuda")
    quant_pack_layers(src, p, 0, L)
    nb = (T + bs - 1) // bs + 1
    slots = O.synthetic_slots(T, bs, nb, seed=11)
    kc = torch.full((L, nb, bs, 6, D), -2.0, dtype=torch.float16, device="cuda")
    vc = torch.full_like(kc, -2.0)
    dst = KVPlanes.paged(kc, vc, torch.from_numpy(slots).cuda()).window(1, 3)
    dequant_scatter_layers(p, dst, 0, L, bulk=bulk)
    torch.cuda.synchronize()
    sub = np.ascontiguousarray(kv[:, :, :, 2:5])
    c, s, z = O.quant_pack(sub.reshape(-1, D), bits, 128)
    assert np.array_equal(p.codes().cpu().numpy().reshape(c.shape), c)
    rows = O.unpack_dequant(c, s, z, bits, 128, D).reshape(L, 2, T, 3, D)
    okc = np.full((L, nb * bs, 6, D), -2.0, np.float16); ovc = okc.copy()
    okc[:, slots, 1:4] = rows[:, 0]; ovc[:, slots, 1:4] = rows[:, 1]
    assert np.array_equal(h16(kc.cpu().numpy().reshape(okc.shape)), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy().reshape(ovc.shape)), h16(ovc))
