"""Regenerate the committed golden fixtures (run in the CPU container).

  python tests/golden/make_golden.py

1. kv_volume.json -- outputs of the REFERENCE itself (hetplan.costs.kv_comm_cost,
   /root/reference/pkg/src/hetplan/costs.py:83-103) on the BASELINE.json shapes
   and on randomized clusters, imported read-only from /root/reference.  Pins the
   volume/time model of our drop-in (paper_2502_09334_b200.costs) to the reference.
2. oracle_sha256.json -- SHA-256 of the oracle's codes/scale/zero/dequant on
   seeded LLaMA-shaped tensors (pins the oracle against silent drift; the GPU
   tests compare the kernels to the oracle directly).
3. groups.npz -- the hand-built edge-case groups (ramp, constant, +-0,
   +-65504, subnormals, outlier, random) with the oracle's outputs.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

from oracle import kvq_oracle as O  # noqa: E402

# BASELINE.json configs: name, L, hidden (=H_kv*D), b, s
SHAPES = [
    ("cfg1_7b_512x1", 32, 4096, 1, 512),
    ("cfg2_7b_2048x8", 32, 4096, 8, 2048),
    ("cfg3_13b_2048x8", 40, 5120, 8, 2048),
    ("cfg4_70b_gqa_4096x8", 80, 1024, 8, 4096),
    ("cfg4_70b_gqa_pair", 80, 1024, 2, 4096),
]


def make_volume():
    sys.path.append("/root/reference/pkg/src")
    from hetplan.core import ClusterSpec, Gpu, GpuType, ModelSpec
    from hetplan.costs import CostParams, KvPrecision, kv_comm_cost

    gt = GpuType("B200", mem_bandwidth=8e12, peak_flops=2.25e15, mem_capacity=180e9, price=1.0)

    def pair(beta, alpha=0.0):
        return ClusterSpec(gpus=(Gpu(0, gt, 0), Gpu(1, gt, 0)),
                           alpha=np.array([[0.0, alpha], [alpha, 0.0]]),
                           beta=np.array([[1e30, beta], [beta, 1e30]]))

    cases = []
    for name, L, h, b, s in SHAPES:
        model = ModelSpec(n_layers=L, hidden_size=h, n_params=7e9)
        for bits in (16, 8, 4, 2):
            for beta, alpha in ((5e9, 0.0), (900e9, 0.0), (770e9, 2e-6)):
                for lf in (True, False):
                    t = kv_comm_cost([0], [1], b, s, model, KvPrecision(bits), pair(beta, alpha),
                                     CostParams(kv_layer_factor=lf))
                    vol = 2 * b * s * h * Fraction(bits, 8) * (L if lf else 1)
                    cases.append(dict(name=name, n_layers=L, hidden_size=h, b=b, s=s, bits=bits,
                                      beta=beta, alpha=alpha, kv_layer_factor=lf,
                                      ref_time=float(t), ref_time_hex=float(t).hex(),
                                      volume=str(vol)))
    rng = np.random.default_rng(7)
    for i in range(20):  # mirrors test_acceptance.py:193-202 randomized clusters
        L = int(rng.integers(1, 100))
        h = int(rng.integers(1, 64)) * 128
        b = int(rng.integers(1, 9))
        s = int(rng.integers(16, 8193))
        beta = float(rng.uniform(1e8, 1e12))
        alpha = float(rng.choice([0.0, 1e-6, 1e-3]))
        bits = int(rng.choice([16, 8, 4, 2]))
        model = ModelSpec(n_layers=L, hidden_size=h, n_params=1e9)
        t = kv_comm_cost([0], [1], b, s, model, KvPrecision(bits), pair(beta, alpha))
        cases.append(dict(name=f"rand{i}", n_layers=L, hidden_size=h, b=b, s=s, bits=bits,
                          beta=beta, alpha=alpha, kv_layer_factor=True, ref_time=float(t),
                          ref_time_hex=float(t).hex(),
                          volume=str(2 * b * s * h * Fraction(bits, 8) * L)))
    with open(os.path.join(HERE, "kv_volume.json"), "w") as f:
        json.dump({"generator": "hetplan.costs.kv_comm_cost (reference, imported read-only)",
                   "cases": cases}, f, indent=1)
    print("kv_volume.json", len(cases))


def edge_groups() -> np.ndarray:
    """[8, 128] fp16 edge-case rows (one 128-element group each)."""
    rows = []
    rows.append(np.tile(np.arange(16, dtype=np.float16), 8))                       # ramp 0..15
    rows.append(np.full(128, 3.5, np.float16))                                     # constant
    z = np.zeros(128, np.float16); z[1::2] = -0.0                                  # +-0
    rows.append(z)
    rows.append(np.where(np.arange(128) % 2, 65504, -65504).astype(np.float16))    # +-max
    rows.append((np.arange(128) * np.float64(2.0 ** -24)).astype(np.float16))     # subnormals
    o = np.zeros(128, np.float16); o[77] = 100.0                                   # outlier
    rows.append(o)
    rng = np.random.default_rng(123)
    rows.append(rng.standard_normal(128).astype(np.float16))                       # random
    rows.append((-np.arange(128) / 64.0 - 1).astype(np.float16))                   # negative ramp
    return np.stack(rows)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_oracle_pins():
    pins = {}
    for (L, T, H, seed) in ((2, 64, 8, 0), (32, 512, 32, 0)):  # the latter = cfg1 (7B 512x1)
        kv = O.synthetic_kv(L, T, H, 128, seed=seed)
        rows = kv.reshape(-1, 128)
        for bits in (2, 4, 8):
            for g in (32, 64, 128):
                if (L, T) == (32, 512) and (bits, g) != (4, 128):
                    continue
                c, s, z = O.quant_pack(rows, bits, g)
                d = O.unpack_dequant(c, s, z, bits, g, 128)
                pins[f"L{L}_T{T}_H{H}_s{seed}_b{bits}_g{g}"] = dict(
                    codes=sha(c), scale=sha(s), zero=sha(z), dequant=sha(d),
                    input=sha(kv))
    with open(os.path.join(HERE, "oracle_sha256.json"), "w") as f:
        json.dump(pins, f, indent=1)
    x = edge_groups()
    out = {"x": x}
    for bits in (2, 4, 8):
        c, s, z = O.quant_pack(x, bits, 128)
        out[f"codes{bits}"], out[f"scale{bits}"], out[f"zero{bits}"] = c, s, z
        out[f"deq{bits}"] = O.unpack_dequant(c, s, z, bits, 128, 128)
    np.savez(os.path.join(HERE, "groups.npz"), **out)
    print("oracle pins", len(pins))


if __name__ == "__main__":
    make_volume()
    make_oracle_pins()
