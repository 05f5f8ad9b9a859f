"""Property-based GPU parity (hypothesis): random geometry, bit-width, group,
paging and padding -- K1 -> K3 (both variants) must equal the oracle
bit-for-bit on every draw."""
import numpy as np
import pytest

from oracle import kvq_oracle as O

pytestmark = pytest.mark.gpu


def test_random_geometries_bit_exact(cuda):
    from hypothesis import given, settings, strategies as st
    from paper_2502_09334_b200 import compress, compress_paged, decompress_into_paged
    torch = cuda

    @settings(max_examples=60, deadline=None, derandomize=True)
    @given(L=st.integers(1, 4), T=st.integers(1, 300), H=st.sampled_from([1, 2, 5, 8, 12]),
           D=st.sampled_from([64, 128, 256]), bits=st.sampled_from([2, 4, 8, 16]),
           group=st.sampled_from([32, 64, 128]), paged_src=st.booleans(),
           bulk=st.booleans(), pad=st.integers(0, 3), seed=st.integers(0, 2**16))
    def check(L, T, H, D, bits, group, paged_src, bulk, pad, seed):
        if D % group:
            group = 32
        kv = O.synthetic_kv(L, T, H, D, seed=seed)
        bs = 16
        nb = (T + bs - 1) // bs + 2
        if paged_src:
            ss = O.synthetic_slots(T, bs, nb, seed=seed + 1)
            kc0 = np.zeros((L, nb * bs, H, D), np.float16); vc0 = kc0.copy()
            kc0[:, ss] = kv[:, 0]; vc0[:, ss] = kv[:, 1]
            p = compress_paged(torch.from_numpy(kc0.reshape(L, nb, bs, H, D)).cuda(),
                               torch.from_numpy(vc0.reshape(L, nb, bs, H, D)).cuda(),
                               torch.from_numpy(ss).cuda(), bits, group)
        else:
            p = compress(torch.from_numpy(kv).cuda(), bits, group)
        slots = O.synthetic_slots(T, bs, nb, seed=seed)
        rng = np.random.default_rng(seed)
        for i in rng.choice(T, size=min(pad, T), replace=False):
            slots[i] = -1
        kc = torch.full((L, nb, bs, H, D), 3.0, dtype=torch.float16, device="cuda")
        vc = torch.full_like(kc, 3.0)
        decompress_into_paged(p, kc, vc, torch.from_numpy(slots).cuda(), bulk=bulk)
        torch.cuda.synchronize()
        c, s, z = O.quant_pack(kv.reshape(-1, D), bits, group)
        rows = O.unpack_dequant(c, s, z, bits, group, D).reshape(L, 2, T, H, D)
        okc = np.full((L, nb, bs, H, D), 3.0, np.float16); ovc = okc.copy()
        O.scatter_paged(rows, slots, okc, ovc)
        assert np.array_equal(kc.cpu().numpy().view(np.uint16), okc.view(np.uint16))
        assert np.array_equal(vc.cpu().numpy().view(np.uint16), ovc.view(np.uint16))
        assert np.array_equal(p.codes().cpu().numpy().reshape(c.shape), c)

    check()
