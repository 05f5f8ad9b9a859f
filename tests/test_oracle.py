"""Oracle pinning (CPU): hand-computed groups, two independent restatements
(numpy, C) agreeing bit-for-bit, committed SHA-256 pins, and KIVI's own fp16
op chain as an accuracy cross-check.  SURVEY.md 8(c)."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import kvq_oracle as O
from oracle import kvq_oracle_c as C

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def h16(x):
    return np.asarray(x, np.float16).view(np.uint16)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class TestHandComputedGroups:
    """Values derived by hand from the format definition (kvx.h)."""

    def setup_method(self):
        self.g = np.load(os.path.join(GOLD, "groups.npz"))
        self.x = self.g["x"]

    def test_ramp_is_identity(self):
        c, s, z = O.quant_pack(self.x[:1], 4, 128)
        assert float(s[0, 0]) == 1.0 and float(z[0, 0]) == 0.0
        assert list(c[0, :8]) == [0x10, 0x32, 0x54, 0x76, 0x98, 0xBA, 0xDC, 0xFE]
        d = O.unpack_dequant(c, s, z, 4, 128, 128)
        assert np.array_equal(d, self.x[:1])

    def test_constant_group_has_zero_scale(self):
        c, s, z = O.quant_pack(self.x[1:2], 4, 128)
        assert h16(s)[0, 0] == 0 and float(z[0, 0]) == 3.5 and not c.any()
        assert np.all(O.unpack_dequant(c, s, z, 4, 128, 128) == 3.5)

    def test_signed_zeros_canonicalise(self):
        c, s, z = O.quant_pack(self.x[2:3], 4, 128)
        assert h16(s)[0, 0] == 0x0000 and h16(z)[0, 0] == 0x0000 and not c.any()

    def test_fp16_extremes_saturate(self):
        c, s, z = O.quant_pack(self.x[3:4], 4, 128)
        # (65504 - -65504)/15 = 8733.87 -> fp16 (ulp 8) = 8736
        assert float(s[0, 0]) == 8736.0 and float(z[0, 0]) == -65504.0
        q = O.unpack(c, 4, 128)[0]
        assert list(q[:4]) == [0, 15, 0, 15]
        d = O.unpack_dequant(c, s, z, 4, 128, 128)[0]
        # 15*8736 - 65504 = 65536 would round to +inf; saturates to 65504
        assert np.isfinite(d).all() and float(d[1]) == 65504.0 and float(d[0]) == -65504.0

    def test_subnormal_scale_clamps(self):
        c, s, z = O.quant_pack(self.x[4:5], 4, 128)
        # max = 127*2^-24; /15 = 8.47*2^-24 -> fp16 subnormal 8*2^-24
        assert h16(s)[0, 0] == 8
        q = O.unpack(c, 4, 128)[0]
        assert q[127] == 15 and q[8] == 1 and q[4] == 0 and q[12] == 2  # 12/8=1.5 -> even 2
        assert q.max() == 15

    def test_outlier(self):
        c, s, z = O.quant_pack(self.x[5:6], 4, 128)
        assert float(s[0, 0]) == 6.66796875  # f16(100/15)
        d = O.unpack_dequant(c, s, z, 4, 128, 128)[0]
        assert float(d[77]) == 100.0 and not d[:77].any()

    @pytest.mark.parametrize("bits", [2, 4, 8])
    def test_committed_group_outputs(self, bits):
        c, s, z = O.quant_pack(self.x, bits, 128)
        assert np.array_equal(c, self.g[f"codes{bits}"])
        assert np.array_equal(h16(s), h16(self.g[f"scale{bits}"]))
        assert np.array_equal(h16(z), h16(self.g[f"zero{bits}"]))
        d = O.unpack_dequant(c, s, z, bits, 128, 128)
        assert np.array_equal(h16(d), h16(self.g[f"deq{bits}"]))


def _random_rows(n, seed, patterns):
    rng = np.random.default_rng(seed)
    if patterns:
        x = rng.integers(0, 0x10000, size=(n, 128), dtype=np.uint16).view(np.float16)
        return np.where(np.isfinite(x), x, np.float16(0))
    return (rng.standard_normal((n, 128)) * rng.choice([1e-3, 1, 30], (n, 1))).astype(np.float16)


@pytest.mark.parametrize("patterns", [False, True])
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("group", [32, 64, 128])
def test_numpy_and_c_restatements_agree(bits, group, patterns):
    x = _random_rows(4000, bits * 1000 + group, patterns)
    a = O.quant_pack(x, bits, group)
    b = C.quant_pack(x, bits, group)
    for p, q in zip(a, b):
        assert np.array_equal(np.asarray(p).view(np.uint8), np.asarray(q).view(np.uint8))
    da = O.unpack_dequant(*a, bits, group, 128)
    db = C.unpack_dequant(*b, bits, group, 128)
    assert np.array_equal(h16(da), h16(db))
    assert np.isfinite(da).all()


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("group", [32, 64, 128])
def test_c_simd_and_scalar_statements_agree(bits, group):
    """The AVX2/F16C baseline path equals the scalar statement and numpy."""
    assert C.simd(), "oracle/Makefile should build the AVX2/F16C path on x86-64"
    x = _random_rows(3000, 77 + bits + group, True)
    a = C.quant_pack(x, bits, group)
    b = C.quant_pack_scalar(x, bits, group)
    for p, q in zip(a, b):
        assert np.array_equal(np.asarray(p).view(np.uint8), np.asarray(q).view(np.uint8))
    assert np.array_equal(h16(C.unpack_dequant(*a, bits, group, 128)),
                          h16(C.unpack_dequant_scalar(*b, bits, group, 128)))


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_dequant_arbitrary_scale_zero(bits):
    """Dequantisation of arbitrary codes under arbitrary finite scale/zero bit
    patterns (subnormals, ties, saturation): numpy == C SIMD == C scalar."""
    rng = np.random.default_rng(100 + bits)
    rows, group = 20000, 32
    codes = rng.integers(0, 256, size=(rows, 128 * bits // 8), dtype=np.uint8)
    def meta():
        m = rng.integers(0, 0x10000, size=(rows, 128 // group), dtype=np.uint16).view(np.float16)
        m = np.where(np.isfinite(m), m, np.float16(1))
        return m
    s, z = np.abs(meta()), meta()
    a = O.unpack_dequant(codes, s, z, bits, group, 128)
    b = C.unpack_dequant(codes, s, z, bits, group, 128)
    c = C.unpack_dequant_scalar(codes, s, z, bits, group, 128)
    assert np.array_equal(h16(a), h16(b))
    assert np.array_equal(h16(a), h16(c))


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(5)
    for bits in (2, 4, 8):
        q = rng.integers(0, 1 << bits, size=(37, 128)).astype(np.uint8)
        assert np.array_equal(O.unpack(O.pack(q, bits), bits, 128), q)


def test_error_bound():
    """|x_hat - x| <= s/2 + 15*s*2^-10 + ulp16(x)/2 for non-degenerate groups."""
    x = _random_rows(5000, 9, False)
    for bits in (2, 4, 8):
        c, s, z = O.quant_pack(x, bits, 128)
        d = O.unpack_dequant(c, s, z, bits, 128, 128).astype(np.float64)
        sf = s.astype(np.float64)
        ulp = np.spacing(np.abs(x).astype(np.float16)).astype(np.float64)
        bound = sf * (0.5 + ((1 << bits) - 1) * 2.0 ** -10) + ulp
        assert np.all(np.abs(d - x.astype(np.float64)) <= bound)


def test_kivi_crosscheck():
    """Our fp32 format vs KIVI's published fp16 op chain (jy-yuan/KIVI
    quant_and_pack_vcache): codes agree except at rounding ties/near-ties, and
    our reconstruction error is no worse."""
    x = _random_rows(4000, 11, False)
    q_ours = O.quantize(x, 4, 128)[0]
    q_kivi, y_kivi = O.kivi_quant_dequant(x, 4, 128)
    agree = np.mean(q_ours == q_kivi)
    assert agree > 0.99, agree
    assert np.abs(q_ours.astype(int) - q_kivi.astype(int)).max() <= 1
    c, s, z = O.quant_pack(x, 4, 128)
    y = O.unpack_dequant(c, s, z, 4, 128, 128)
    e_ours = np.abs(y.astype(np.float64) - x).mean()
    e_kivi = np.abs(y_kivi.astype(np.float64) - x).mean()
    assert e_ours <= e_kivi * 1.001


def test_sha256_pins():
    pins = json.load(open(os.path.join(GOLD, "oracle_sha256.json")))
    for key, want in pins.items():
        if "L32_T512" in key:
            continue  # cfg1 pin is checked by the slower test below
        L, T, H, seed, b, g = (int(p[1:]) for p in key.split("_"))
        kv = O.synthetic_kv(L, T, H, 128, seed=seed)
        assert sha(kv) == want["input"]
        c, s, z = O.quant_pack(kv.reshape(-1, 128), b, g)
        assert sha(c) == want["codes"] and sha(s) == want["scale"] and sha(z) == want["zero"]
        assert sha(O.unpack_dequant(c, s, z, b, g, 128)) == want["dequant"]


def test_cfg1_pin_with_c_oracle():
    """BASELINE config 1 (7B, 512 tokens, batch 1) through the C restatement."""
    pins = json.load(open(os.path.join(GOLD, "oracle_sha256.json")))
    want = pins["L32_T512_H32_s0_b4_g128"]
    kv = O.synthetic_kv(32, 512, 32, 128, seed=0)
    assert sha(kv) == want["input"]
    c, s, z = C.quant_pack(kv.reshape(-1, 128), 4, 128)
    assert sha(c) == want["codes"] and sha(s) == want["scale"] and sha(z) == want["zero"]
    assert sha(C.unpack_dequant(c, s, z, 4, 128, 128)) == want["dequant"]
    assert c.nbytes == 67_108_864  # codes = exactly 1/4 of the fp16 268,435,456 B


def test_scatter_paged_oracles_agree():
    L, T, H, D = 3, 37, 4, 128
    kv = O.synthetic_kv(L, T, H, D, seed=3)
    nb, bs = 8, 16
    slots = O.synthetic_slots(T, bs, nb, seed=3)
    slots[5] = -1  # padding token
    c, s, z = O.quant_pack(kv.reshape(-1, D), 4, 64)
    kc = np.zeros((L, nb, bs, H, D), np.float16); vc = np.zeros_like(kc)
    rows = O.unpack_dequant(c, s, z, 4, 64, D).reshape(L, 2, T, H, D)
    O.scatter_paged(rows, slots, kc, vc)
    kc2 = np.zeros_like(kc); vc2 = np.zeros_like(kc)
    C.dequant_scatter_paged(c, s, z, slots, L, T, H, D, 64, 4, kc2, vc2)
    assert np.array_equal(h16(kc), h16(kc2)) and np.array_equal(h16(vc), h16(vc2))
    flat = kc.reshape(L, nb * bs, H, D)
    assert np.array_equal(flat[:, slots[0]], rows[:, 0, 0])


def test_kivi_oracle_layout_and_accuracy():
    from paper_2502_09334_b200.kivi import KiviLayout, kivi_groups
    seq = (70, 64, 0, 66)
    gs, rt = O.kivi_groups(seq, 32)
    gs2, rt2 = kivi_groups(seq, 32)
    assert np.array_equal(gs, gs2) and np.array_equal(rt, rt2)
    assert list(gs) == [0, 32, 70, 102, 134, 166] and list(rt) == [64, 65, 66, 67, 68, 69, 198, 199]
    kv = O.synthetic_kv(2, 200, 4, 128, seed=1)
    p = O.quant_pack_kivi(kv, 4, 32, seq)
    lay = KiviLayout(2, 4, 128, 4, 32, seq)
    for name, size in zip(("Kc", "Ks", "Kz", "Kr", "Vc", "Vs", "Vz"), lay.sizes):
        assert p[name].nbytes == 2 * size, name
    K, V = O.unpack_dequant_kivi(p, 4, 32, seq, 4, 128)
    assert np.array_equal(K[:, rt], kv[:, 0][:, rt])  # residual window is exact
    e_kivi = np.abs(K.astype(np.float64) - kv[:, 0]).mean()
    c, s, z = O.quant_pack(kv[:, 0].reshape(-1, 128), 4, 32)
    e_tok = np.abs(O.unpack_dequant(c, s, z, 4, 32, 128).astype(np.float64) - kv[:, 0].reshape(-1, 128)).mean()
    assert e_kivi < 0.75 * e_tok  # per-channel K isolates the outlier channels


def test_oracle_volume_model_matches_reference_golden():
    """The oracle's restatement of the reference's volume/time model
    (kv_volume_bytes, kv_comm_time; costs.py:83-103) reproduces the
    reference's own outputs bit for bit (tests/golden/kv_volume.json), and its
    packed_layout byte counts equal the 4-bit code volume the reference charges."""
    import json
    import os
    from fractions import Fraction
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kv_volume.json")))
    for c in gold["cases"]:
        v = O.kv_volume_bytes(c["b"], c["s"], c["n_layers"], c["hidden_size"], c["bits"],
                              c["kv_layer_factor"])
        assert v == Fraction(c["volume"]), c["name"]
        assert float(O.kv_comm_time(v, c["alpha"], c["beta"])).hex() == c["ref_time_hex"]
        if c["bits"] in (8, 4, 2) and c["kv_layer_factor"] and c["hidden_size"] % 128 == 0:
            rows = c["n_layers"] * 2 * c["b"] * c["s"] * (c["hidden_size"] // 128)
            codes, scale, zero = O.packed_layout(rows, 128, 128, c["bits"])
            assert codes == v and scale == zero == rows * 2
    with pytest.raises(ValueError):
        O.kv_volume_bytes(1, 1, 1, 1, 3)
    with pytest.raises(ValueError):
        O.kv_volume_bytes(0, 1, 1, 1, 4)


# ---------------------------------------------------------------------------
# The torch-CPU variant of the CPU path equals the oracle
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("patterns", [False, True])
@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("group", [32, 64, 128])
def test_torch_cpu_variant_equals_oracle(bits, group, patterns):
    import torch
    from oracle import kvq_torch_cpu as TC
    x = _random_rows(3000, 500 + bits * 7 + group, patterns)
    a = O.quant_pack(x, bits, group)
    b = TC.quant_pack(torch.from_numpy(x), bits, group)
    for p, q in zip(a, b):
        assert np.array_equal(np.asarray(p).view(np.uint8), q.numpy().view(np.uint8))
    da = O.unpack_dequant(*a, bits, group, 128)
    db = TC.unpack_dequant(*b, bits, group, 128).numpy()
    assert np.array_equal(h16(da), h16(db))


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_torch_cpu_dequant_arbitrary_scale_zero(bits):
    """Arbitrary finite scale/zero bit patterns: the float64 -> float16 step
    (round-to-odd float32, then RN) rounds once, like numpy."""
    import torch
    from oracle import kvq_torch_cpu as TC
    rng = np.random.default_rng(300 + bits)
    rows, group = 20000, 32
    codes = rng.integers(0, 256, size=(rows, 128 * bits // 8), dtype=np.uint8)

    def meta():
        m = rng.integers(0, 0x10000, size=(rows, 128 // group), dtype=np.uint16).view(np.float16)
        return np.where(np.isfinite(m), m, np.float16(1))
    s, z = np.abs(meta()), meta()
    a = O.unpack_dequant(codes, s, z, bits, group, 128)
    b = TC.unpack_dequant(torch.from_numpy(codes), torch.from_numpy(s), torch.from_numpy(z),
                          bits, group, 128).numpy()
    assert np.array_equal(h16(a), h16(b))


def test_torch_cpu_golden_groups_and_scatter():
    import torch
    from oracle import kvq_torch_cpu as TC
    g = np.load(os.path.join(GOLD, "groups.npz"))
    for bits in (2, 4, 8):
        c, s, z = TC.quant_pack(torch.from_numpy(g["x"]), bits, 128)
        assert np.array_equal(c.numpy(), g[f"codes{bits}"])
        assert np.array_equal(h16(s.numpy()), h16(g[f"scale{bits}"]))
        d = TC.unpack_dequant(c, s, z, bits, 128, 128).numpy()
        assert np.array_equal(h16(d), h16(g[f"deq{bits}"]))
    T, H, D, nb, bs = 37, 4, 128, 8, 16
    kv = O.synthetic_kv(1, T, H, D, seed=4)
    slots = O.synthetic_slots(T, bs, nb, seed=4)
    slots[3] = -1
    c, s, z = O.quant_pack(kv.reshape(-1, D), 4, 64)
    kc = np.zeros((1, nb, bs, H, D), np.float16); vc = np.zeros_like(kc)
    C.dequant_scatter_paged(c, s, z, slots, 1, T, H, D, 64, 4, kc, vc)
    kt = torch.zeros((nb, bs, H, D), dtype=torch.float16); vt = torch.zeros_like(kt)
    TC.dequant_scatter_paged(torch.from_numpy(c), torch.from_numpy(s), torch.from_numpy(z),
                             torch.from_numpy(slots), T, H, D, 64, 4, kt, vt)
    assert np.array_equal(h16(kc[0]), h16(kt.numpy())) and np.array_equal(h16(vc[0]), h16(vt.numpy()))
