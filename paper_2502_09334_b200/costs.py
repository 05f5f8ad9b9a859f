"""The reference's KV-transfer API, kept signature-compatible, plus the measured
drop-in.

Restated from ``/root/reference/pkg/src/hetplan/costs.py`` (the reference is a
planner; its hand-off exists only as this model):

* ``KvPrecision``      costs.py:18-30   bits in {16, 8, 4, 2}, exact bytes/elem
* ``CostParams``       costs.py:33-48   (``kv_layer_factor`` costs.py:41-42)
* ``bottleneck_link``  costs.py:51-65   min-beta pair, NoPath if none
* ``kv_comm_cost``     costs.py:83-103  alpha + 2*b*s*h*N_bytes*L / beta

All three accept the reference's own ``ModelSpec`` / ``ClusterSpec`` objects
(duck-typed: ``n_layers``, ``hidden_size``; ``index_of``, ``alpha``, ``beta``),
so ``measured_kv_comm_cost`` can be rebound into ``hetplan.simulate`` /
``hetplan.orchestrate`` (they import ``kv_comm_cost`` by name,
simulate.py:16-23, orchestrate.py:17-24).  See INTEGRATION.md.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Callable

from .errors import NoPath

ALLOWED_BITS = (16, 8, 4, 2)
DEFAULT_GROUP = 128
DEFAULT_BLOCK = 16


@dataclass(frozen=True)
class KvPrecision:
    """Element bitwidth used for KV-cache transfer between phases (costs.py:18-30)."""

    bits: int = 16

    def __post_init__(self):
        if self.bits not in ALLOWED_BITS:
            raise ValueError("bits must be one of 16, 8, 4, 2")

    @property
    def bytes_per_element(self) -> Fraction:
        """Code bytes only, as the reference charges (costs.py:28-30)."""
        return Fraction(self.bits, 8)

    def wire_bytes_per_element(self, group: int = DEFAULT_GROUP) -> Fraction:
        """Code bytes + the fp16 scale and zero of every group of ``group``
        elements: what actually crosses the link (0.53125 at 4-bit, G=128).
        The reference's model omits this metadata."""
        if self.bits == 16:
            return Fraction(2)
        return Fraction(self.bits, 8) + Fraction(4, group)


@dataclass(frozen=True)
class CostParams:
    """Calibration constants (costs.py:33-48); only ``kv_layer_factor`` is used here."""

    flops_efficiency: float = 0.6
    mem_efficiency: float = 0.8
    tp_allreduce_latency: float = 0.0
    batch_token_plateau: int = 1024
    kv_layer_factor: bool = True

    def __post_init__(self):
        for f in ("flops_efficiency", "mem_efficiency"):
            v = getattr(self, f)
            if not 0 < v <= 1:
                raise ValueError(f"{f} must be in (0,1]")


def _bits(prec) -> int:
    b = getattr(prec, "bits", prec)
    if b not in ALLOWED_BITS:
        raise ValueError("bits must be one of 16, 8, 4, 2")
    return int(b)


def bottleneck_link(src_gpu_ids, dst_gpu_ids, cluster) -> tuple[float, float]:
    """(alpha, beta) of the minimum positive-bandwidth pair (costs.py:51-65)."""
    found = None
    for a in src_gpu_ids:
        ia = cluster.index_of(a)
        for b in dst_gpu_ids:
            ib = cluster.index_of(b)
            bw = cluster.beta[ia, ib]
            if bw <= 0:
                continue
            if found is None or bw < found[1]:
                found = (cluster.alpha[ia, ib], bw)
    if found is None:
        raise NoPath(f"no positive-bandwidth link between {src_gpu_ids} and {dst_gpu_ids}")
    return found


def kv_volume(b: int, s: int, model, prec, params: CostParams = CostParams()) -> Fraction:
    """Exact modelled transfer volume ``2*b*s*h*N_bytes*L`` (costs.py:101-102)."""
    if b < 1 or s < 1:
        raise ValueError("batch size and sequence length must be >= 1")
    layers = model.n_layers if params.kv_layer_factor else 1
    return 2 * b * s * model.hidden_size * Fraction(_bits(prec), 8) * layers


def kv_comm_cost(prefill_gpu_ids, decode_gpu_ids, b: int, s: int, model, prec, cluster,
                 params: CostParams = CostParams()) -> float:
    """alpha + 2*b*s*h*N_bytes*L / beta over the bottleneck link (costs.py:83-103)."""
    if b < 1 or s < 1:
        raise ValueError("batch size and sequence length must be >= 1")
    alpha, beta = bottleneck_link(prefill_gpu_ids, decode_gpu_ids, cluster)
    return alpha + float(kv_volume(b, s, model, prec, params)) / beta


def measured_kv_comm_cost(table: Callable[[int, int, int], float] | dict,
                          fallback: Callable | None = kv_comm_cost) -> Callable:
    """A ``kv_comm_cost``-signature function backed by measured hand-off times.

    ``table`` maps (bits, fp16_bytes) -> seconds (a callable, or a dict of
    bits -> (alpha_s, bytes_per_s) fitted from ``bench.py`` / ``tools``
    measurements).  The returned function keeps the reference's argument
    checks and NoPath behaviour (it still resolves the bottleneck link), and
    can be installed as ``hetplan.simulate.kv_comm_cost``.
    """

    def _cost(prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster,
              params: CostParams = CostParams()) -> float:
        if b < 1 or s < 1:
            raise ValueError("batch size and sequence length must be >= 1")
        bottleneck_link(prefill_gpu_ids, decode_gpu_ids, cluster)  # NoPath semantics
        bits = _bits(prec)
        fp16_bytes = int(kv_volume(b, s, model, KvPrecision(16), params))
        if callable(table):
            return float(table(bits, fp16_bytes, len(tuple(prefill_gpu_ids))))
        if bits in table:
            alpha, rate = table[bits]
            return float(alpha) + fp16_bytes / float(rate)
        if fallback is None:
            raise ValueError(f"no measurement for {bits}-bit hand-off")
        return fallback(prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster, params)

    return _cost
