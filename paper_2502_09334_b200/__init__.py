"""B200-native prefill->decode KV hand-off for ThunderServe (arXiv 2502.09334).

Drop-in for the reference's KV-transfer path (``hetplan.costs.KvPrecision`` /
``kv_comm_cost``, ``/root/reference/pkg/src/hetplan/costs.py:18-103``): the
same model API, plus the data path it models -- sm_100a quantise+pack (K1),
NVLink transfer, dequantise+scatter into the decode paged cache (K3) -- behind
the C-ABI in ``include/kvx.h``.
"""
from .costs import (  # noqa: F401
    CostParams,
    KvPrecision,
    bottleneck_link,
    kv_comm_cost,
    HandoffTable,
    install_measurements,
    kv_volume,
    measured_cost_fn,
    measured_kv_comm_cost,
)
from .errors import NoPath, PlanningError  # noqa: F401

__version__ = "0.1.0"

_HANDOFF_NAMES = (
    "PackedKV", "PackedLayout", "KVPlanes", "HandoffPlan", "alloc_packed", "compress",
    "compress_paged", "decompress_into_paged", "transfer", "handoff", "enable_peer",
    "layer_chunks", "quant_pack_layers", "dequant_scatter_layers",
)


def __getattr__(name):  # lazy: the data path needs torch; the model API does not
    if name in _HANDOFF_NAMES:
        import importlib
        return getattr(importlib.import_module(__name__ + ".datapath"), name)
    raise AttributeError(name)
