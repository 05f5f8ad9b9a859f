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


class HandoffTable:
    """Measured hand-off times of this data path on one link class.

    ``entries`` maps bits -> (alpha_s, fp16_bytes_per_s): one hand-off of V
    fp16-equivalent bytes takes ``alpha + V / rate`` (the bench's per-pair
    two-point calibration, ``bench.py`` N>1 ``calibration``; one entry per
    bit-width the reference plans with, ``cli.py:278``).  ``link_beta`` is the
    cluster beta (bytes/s) of the link the table was measured on, kept as
    provenance.  The table prices the kernels + transfer; the link the planner
    resolves still bounds the result (``measured_kv_comm_cost``)."""

    def __init__(self, entries: dict, link_beta: float | None = None, source: str = ""):
        self.entries = {}
        for bits, (alpha, rate) in entries.items():
            bits = _bits(int(bits))
            if not (alpha >= 0 and rate > 0):
                raise ValueError(f"bad measurement for {bits}-bit: alpha={alpha}, rate={rate}")
            self.entries[bits] = (float(alpha), float(rate))
        self.link_beta = link_beta
        self.source = source

    def time(self, bits: int, fp16_bytes: int) -> float | None:
        e = self.entries.get(bits)
        return None if e is None else e[0] + fp16_bytes / e[1]

    @classmethod
    def from_json(cls, path: str) -> "HandoffTable":
        """``{"entries": {"4": {"alpha_s": .., "fp16_bytes_per_s": ..}, ..},
        "link_beta": .., "source": ..}`` (tools/handoff_table.py writes it)."""
        import json
        with open(path) as f:
            d = json.load(f)
        ent = {int(k): (v["alpha_s"], v["fp16_bytes_per_s"]) for k, v in d["entries"].items()}
        return cls(ent, d.get("link_beta"), d.get("source", path))


_ACTIVE_TABLE: HandoffTable | None = None


def install_measurements(table) -> HandoffTable | None:
    """Make ``table`` (a HandoffTable, a dict bits -> (alpha_s, rate) or a
    path to its JSON; None to clear) the one ``measured_kv_comm_cost`` reads.
    Returns the previous table."""
    global _ACTIVE_TABLE
    prev = _ACTIVE_TABLE
    if table is None or isinstance(table, HandoffTable):
        _ACTIVE_TABLE = table
    elif isinstance(table, str):
        _ACTIVE_TABLE = HandoffTable.from_json(table)
    else:
        _ACTIVE_TABLE = HandoffTable(table)
    return prev


def _measured(table, prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster, params,
              fallback):
    analytic = kv_comm_cost(prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster, params)
    bits = _bits(prec)
    t = table.time(bits, int(kv_volume(b, s, model, KvPrecision(16), params))) if table else None
    if t is None:
        if fallback is None:
            raise ValueError(f"no measurement for {bits}-bit hand-off")
        return fallback(prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster, params)
    # the measured kernels + NVLink path, but never faster than the link the
    # planner resolved: a slower (e.g. cross-node) bottleneck keeps its model
    return max(t, analytic)


def measured_kv_comm_cost(prefill_gpu_ids, decode_gpu_ids, b: int, s: int, model, prec, cluster,
                          params: CostParams = CostParams()) -> float:
    """``kv_comm_cost``'s signature and contract (costs.py:83-103), priced by
    the installed measured table (``install_measurements``):

        max(alpha_m + V16 / rate_m[bits],  alpha + V(bits) / beta)

    where the second term is the reference's own model over the bottleneck
    link: the measured hand-off (quantise + NVLink + dequantise into the paged
    cache, metadata included) where it is the slower one -- the NVLink class
    it was measured on -- and the link model where the planner's link is
    slower than the measured path (a cross-node pair).  ``ValueError`` for
    bad bits / b / s and ``NoPath`` as the reference; a bit-width the table
    lacks (or no table) falls back to the analytic model.  Install it with
    ``hetplan.simulate.kv_comm_cost = hetplan.orchestrate.kv_comm_cost =
    measured_kv_comm_cost``."""
    return _measured(_ACTIVE_TABLE, prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster,
                     params, kv_comm_cost)


def measured_cost_fn(table, fallback: Callable | None = kv_comm_cost) -> Callable:
    """A ``kv_comm_cost``-signature closure over its own ``table`` (a
    HandoffTable or dict bits -> (alpha_s, fp16_bytes_per_s)); same pricing as
    ``measured_kv_comm_cost`` without touching the installed table.
    ``fallback=None`` raises ValueError for an unmeasured bit-width."""
    tab = table if isinstance(table, HandoffTable) else HandoffTable(table)

    def _cost(prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster,
              params: CostParams = CostParams()) -> float:
        return _measured(tab, prefill_gpu_ids, decode_gpu_ids, b, s, model, prec, cluster, params,
                         fallback)

    return _cost
