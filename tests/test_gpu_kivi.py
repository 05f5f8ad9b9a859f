"""The "kivi" format on the GPU: per-channel K groups with a
residual fp16 window, V per token -- bit-exact vs oracle.quant_pack_kivi."""
import numpy as np
import pytest

from oracle import kvq_oracle as O

pytestmark = pytest.mark.gpu


def h16(x):
    return np.ascontiguousarray(x).view(np.uint16)


CASES = [  # (L, H, D, seqlens)
    (2, 4, 128, (70, 64, 66)),
    (3, 8, 128, (200,)),
    (1, 2, 64, (31,)),            # no full group: residual only
    (2, 32, 128, (96, 0, 33)),    # empty request in the batch
    (2, 40, 128, (128, 64)),      # 13B head count, no residual
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("group", [32, 64])
@pytest.mark.parametrize("bulk", [False, True])  # per-lane kernels / TMA bulk-staged (pull)
def test_kivi_bit_exact(cuda, case, bits, group, bulk):
    torch = cuda
    from paper_2502_09334_b200.kivi import compress_kivi, decompress_kivi_into_paged
    L, H, D, seq = case
    if D % group:
        pytest.skip("group must divide head_dim")
    T = sum(seq)
    kv = O.synthetic_kv(L, T, H, D, seed=T + bits)
    p = compress_kivi(torch.from_numpy(kv).cuda(), bits, group, seq)
    torch.cuda.synchronize()
    want = O.quant_pack_kivi(kv, bits, group, seq)
    names = ["Kc", "Ks", "Kz", "Kr", "Vc", "Vs", "Vz"]
    for i, n in enumerate(names):
        got = p.part(i).cpu().numpy().reshape(L, -1)
        w = np.ascontiguousarray(want[n]).view(np.uint8).reshape(L, -1)
        assert got.shape == w.shape, n
        assert np.array_equal(got, w), n
    bs = 16
    nb = (T + bs - 1) // bs + 2
    slots = O.synthetic_slots(T, bs, nb, seed=T)
    kc = torch.full((L, nb, bs, H, D), -5.0, dtype=torch.float16, device="cuda")
    vc = torch.full_like(kc, -5.0)
    sl = slots.copy()
    sl[::7] = -1  # padding tokens are skipped by every kernel
    decompress_kivi_into_paged(p, kc, vc, torch.from_numpy(sl).cuda(), bulk=bulk)
    torch.cuda.synchronize()
    K, V = O.unpack_dequant_kivi(want, bits, group, seq, H, D)
    keep = sl >= 0
    K, V, slots = K[:, keep], V[:, keep], slots[keep]
    okc = np.full((L, nb * bs, H, D), -5.0, np.float16); ovc = okc.copy()
    okc[:, slots] = K; ovc[:, slots] = V
    assert np.array_equal(h16(kc.cpu().numpy().reshape(okc.shape)), h16(okc))
    assert np.array_equal(h16(vc.cpu().numpy().reshape(ovc.shape)), h16(ovc))


def test_kivi_beats_per_token_on_outlier_keys(cuda):
    """The point of the variant: K with outlier channels reconstructs better."""
    torch = cuda
    from paper_2502_09334_b200 import compress, decompress_into_paged
    from paper_2502_09334_b200.kivi import compress_kivi, decompress_kivi_into_paged
    L, T, H, D = 2, 256, 8, 128
    kv = O.synthetic_kv(L, T, H, D, seed=5)
    x = torch.from_numpy(kv).cuda()
    slots = torch.arange(T, device="cuda")
    kc = torch.zeros((L, T // 16, 16, H, D), dtype=torch.float16, device="cuda")
    vc = torch.zeros_like(kc)
    decompress_kivi_into_paged(compress_kivi(x, 4, 32), kc, vc, slots)
    err_kivi = (kc.view(L, T, H, D).float() - x[:, 0].float()).abs().mean().item()
    decompress_into_paged(compress(x, 4, 32), kc, vc, slots)
    err_tok = (kc.view(L, T, H, D).float() - x[:, 0].float()).abs().mean().item()
    assert err_kivi < 0.75 * err_tok
