"""The CPU hand-off in torch ops (TEST INFRASTRUCTURE ONLY: the "torch-CPU
variant" SURVEY.md section 8(d) asks to report next to the CPU baseline).

Same arithmetic as ``kvq_oracle.quantize / pack / unpack / dequantize`` (the
restatement of SURVEY.md 8(c); ``PAPER.md:490-493``), written as torch CPU
tensor ops so that torch's intra-op thread pool runs it on every host core
(``torch.set_num_threads``).  Only ``tests/`` and ``bench.py``'s cpu_baseline
leg import it; bit-identity with the numpy oracle is tested in
``tests/test_oracle.py``.

One detail differs in HOW, not WHAT: the dequantised value must be the single
correctly-rounded fp16 of the exact ``q*s + z``.  numpy converts float64 to
float16 directly; torch converts through float32, which could round twice, so
the float64 value is first narrowed to float32 with round-to-odd (exact for a
later rounding to the 11-bit fp16 significand) and then rounded to fp16.
"""
from __future__ import annotations

import torch

_MAG = 0x7FFFFFFF


def _check(head_dim: int, group: int, bits: int):
    if bits not in (8, 4, 2):
        raise ValueError("quantised bits must be one of 8, 4, 2")
    if group not in (32, 64, 128) or head_dim % group:
        raise ValueError("group must be 32, 64 or 128 and divide head_dim")


def quant_pack(x: torch.Tensor, bits: int = 4, group: int = 128):
    """fp16 [rows, D] (CPU) -> (codes u8 [rows, D*bits/8], scale f16 [rows, D/G],
    zero f16 [rows, D/G]); kvq_oracle.quant_pack in torch ops."""
    assert x.dtype == torch.float16 and x.dim() == 2 and not x.is_cuda
    rows, d = x.shape
    _check(d, group, bits)
    ng = d // group
    qmax = (1 << bits) - 1
    xf = x.float().view(rows, ng, group)
    mn = xf.amin(dim=-1)
    mx = xf.amax(dim=-1)
    zero16 = (mn + 0.0).half()                       # canonicalises -0
    scale16 = ((mx - mn) / float(qmax) + 0.0).half()  # IEEE fp32 division, RN to fp16
    s = scale16.float()
    z = zero16.float()
    ok = s != 0
    inv = torch.where(ok, 1.0 / torch.where(ok, s, torch.ones_like(s)), torch.zeros_like(s))
    t = (xf - z.unsqueeze(-1)).double()              # RN32(x - z), widened exactly
    q = torch.round(t * inv.double().unsqueeze(-1))  # exact product, ONE rounding (half-even)
    # s == 0: inv = 0 and the finite t gives q = 0, the oracle's explicit case
    q = q.clamp_(0, qmax).to(torch.uint8).view(rows, d)
    return pack(q, bits), scale16, zero16


def pack(q: torch.Tensor, bits: int) -> torch.Tensor:
    rows, d = q.shape
    if bits == 8:
        return q.clone()
    per = 8 // bits
    qq = q.view(rows, d // per, per).to(torch.int32)
    out = torch.zeros((rows, d // per), dtype=torch.int32)
    for k in range(per):
        out |= qq[:, :, k] << (k * bits)
    return out.to(torch.uint8)


def unpack(codes: torch.Tensor, bits: int, head_dim: int) -> torch.Tensor:
    rows = codes.shape[0]
    if bits == 8:
        return codes.clone()
    per = 8 // bits
    mask = (1 << bits) - 1
    c = codes.to(torch.int32)
    q = torch.empty((rows, head_dim // per, per), dtype=torch.int32)
    for k in range(per):
        q[:, :, k] = (c >> (k * bits)) & mask
    return q.view(rows, head_dim)


def _f64_to_f16(y: torch.Tensor) -> torch.Tensor:
    """Correctly rounded float64 -> float16: narrow to float32 with round-to-odd
    (the float32 neighbour with an odd significand when inexact), then RN."""
    f = y.float()
    inexact = f.double() != y
    bits = f.view(torch.int32)
    even = (bits & 1) == 0
    # |y| beyond |f|: step the magnitude up one ulp, else down (the odd neighbour)
    up = y.abs() > f.double().abs()
    mag = (bits & _MAG) + torch.where(up, 1, -1).to(torch.int32)
    fixed = (bits & ~_MAG) | mag
    bits = torch.where(inexact & even, fixed, bits)
    return bits.view(torch.float32).half()


def dequantize(q: torch.Tensor, scale16: torch.Tensor, zero16: torch.Tensor,
               group: int) -> torch.Tensor:
    rows, d = q.shape
    ng = d // group
    s = scale16.double().view(rows, ng, 1)
    z = zero16.double().view(rows, ng, 1)
    y = q.double().view(rows, ng, group) * s + z     # exact
    y = torch.clamp_max(y, 65504.0)
    return _f64_to_f16(y).view(rows, d)


def unpack_dequant(codes, scale16, zero16, bits: int, group: int, head_dim: int) -> torch.Tensor:
    return dequantize(unpack(codes, bits, head_dim), scale16, zero16, group)


def dequant_scatter_paged(codes, scale16, zero16, slots: torch.Tensor, n_tokens: int,
                          n_heads: int, head_dim: int, group: int, bits: int,
                          k_cache: torch.Tensor, v_cache: torch.Tensor) -> None:
    """One layer: payload rows [2, T, H] -> the paged caches [NB, BS, H, D] at
    ``slots`` (slot < 0: padding token, skipped), like kvq_oracle.scatter_paged."""
    rows = unpack_dequant(codes, scale16, zero16, bits, group, head_dim)
    rows = rows.view(2, n_tokens, n_heads, head_dim)
    keep = slots >= 0
    sl = slots[keep]
    k_cache.view(-1, n_heads, head_dim)[sl] = rows[0][keep]
    v_cache.view(-1, n_heads, head_dim)[sl] = rows[1][keep]
