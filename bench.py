#!/usr/bin/env python
"""Benchmark of the prefill->decode KV hand-off (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric: "KV hand-off GB/s (fp16-equiv)" = the reference's 16-bit KV volume
(2*b*s*h*2*L, costs.py:102) moved per second, whole job, with the % of the
HBM / NVLink roofline.

* N = 1: BASELINE config 2 (LLaMA-2-7B KV, 2048 tokens x batch 8): one step =
  K1 quantise+pack of the whole [32, 2, 16384, 32, 128] fp16 KV, then K3
  dequantise + scatter into a paged decode cache (block 16, random block
  table).  Inputs (8.6 GB) are far larger than L2 (126 MB), so no flush.
* N > 1 (torchrun, one process per GPU): ranks [0, N/2) are prefill, [N/2, N)
  decode, pair i -> i + N/2 (1P1D / 2P2D / 4P4D); see transport.py.
* --impl reference: the CPU reference path (the C restatement of the oracle,
  oracle/kvq_oracle.c, all host threads) on a bounded sample of the same
  workload; rank 0 only.

One JSON line on rank 0.  Timing: CUDA events on the launching streams, a
barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV hand-off GB/s (fp16-equiv)"
UNIT = "GB/s"

# name -> (n_layers, n_kv_heads, head_dim, batch, seq)
WORKLOADS = {
    "cfg1_7b_512x1": (32, 32, 128, 1, 512),
    "cfg2_7b_2048x8": (32, 32, 128, 8, 2048),
    "cfg3_13b_2048x8": (40, 40, 128, 8, 2048),
    "cfg4_70b_gqa_pair": (80, 8, 128, 2, 4096),  # one 4P4D pair: 8x4096 tokens / 4 pairs
    "small_70b_gqa_128x1": (80, 8, 128, 1, 128),  # shortest trace request: latency-bound
}
BLOCK = 16

# Config 5: mixed prompt-length trace: batches of 1-16
# requests, lengths log-uniform in [128, 8192], np.random.default_rng(0),
# a batch closes at 16,384 tokens (a prefill batch's worth of KV).
TRACE_MODELS = {"trace_7b": (32, 32, 128), "trace_70b_gqa": (80, 8, 128)}
TRACE_CAP = 16384


def make_trace(n_batches: int, seed: int = 0, cap: int = TRACE_CAP):
    import numpy as np
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_batches):
        lens = []
        for _ in range(int(rng.integers(1, 17))):
            n = int(round(float(np.exp(rng.uniform(np.log(128), np.log(8192))))))
            if sum(lens) + n > cap:
                break
            lens.append(n)
        out.append(lens or [128])
    return out


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


# NVLink roofline per direction: the fastest peer copy measured on this pool's
# B200s -- a TMA bulk pull into shared memory (tools/nvlink_bench.cu,
# profiles/r01_nvlink/nvlink_bench.jsonl: 782-783 GB/s; copy engines 777,
# B200_PROFILING.md's peer copy 770; 900 nominal)
NVLINK_GBS = 783.0
L2_BYTES = 126 * 2**20  # B200 L2


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        time.sleep(0.1)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), util=float(parts[4]),
                                 reasons=[n for n, v in zip(
                                     ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                      "sw_power_cap"), parts[5:9]) if v.lower() == "active"]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [r for r in rows if r["util"] > 0] or rows
        reasons = sorted({x for r in busy for x in r["reasons"]})
        return {"sm_mhz": statistics.median(r["sm"] for r in busy),
                "sm_max_mhz": max(r["smax"] for r in rows), "reasons": reasons,
                "samples": len(busy)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle/kvq_oracle.c) on a bounded sample
# ---------------------------------------------------------------------------
_CPU_LAYERS: dict = {}


def _cpu_layer(workload, i, T, H, D):
    """Synthetic layer i of the workload (generated once, outside timing)."""
    from oracle import kvq_oracle as O
    key = (workload, i % 4)
    if key not in _CPU_LAYERS:
        _CPU_LAYERS[key] = O.synthetic_kv(1, T, H, D, seed=i % 4)  # [1, 2, T, H, D]
    return _CPU_LAYERS[key]


def cpu_reference(workload: str, bits: int, group: int, budget_s: float | None = 12.0,
                  max_layers: int | None = None):
    """Time the C oracle (quant+pack, then dequant+scatter into a paged cache)
    layer by layer over the workload until ``budget_s`` or ``max_layers``."""
    import numpy as np
    from oracle import kvq_oracle as O
    from oracle import kvq_oracle_c as C
    C.lib()
    L, H, D, b, s = WORKLOADS[workload]
    T = b * s
    nb = (T + BLOCK - 1) // BLOCK
    key = ("dst", workload)
    if key not in _CPU_LAYERS:  # destination cache, allocated and touched once
        kc0 = np.zeros((1, nb, BLOCK, H, D), np.float16)
        vc0 = np.zeros_like(kc0)
        kc0.fill(0)
        vc0.fill(0)  # fault the pages in outside the timed region
        _CPU_LAYERS[key] = (O.synthetic_slots(T, BLOCK, nb, seed=0), kc0, vc0)
    slots, kc, vc = _CPU_LAYERS[key]
    okey = ("out", workload, bits, group)
    if okey not in _CPU_LAYERS and bits != 16:  # payload buffers, touched once
        rows = 2 * T * H
        outs = (np.zeros((rows, D * bits // 8), np.uint8), np.zeros((rows, D // group), np.float16),
                np.zeros((rows, D // group), np.float16))
        _CPU_LAYERS[okey] = outs
    outs = _CPU_LAYERS.get(okey)
    layers = 0
    elapsed = 0.0
    # cycle over the workload's layers until the time budget (a bounded sample
    # of about 10-30 s of CPU work), or exactly max_layers layers
    limit = max_layers or (L if budget_s is None else 1 << 30)
    while layers < limit:
        kv = _cpu_layer(workload, layers % L, T, H, D)
        t0 = time.perf_counter()
        c, sc, z = C.quant_pack(kv.reshape(-1, D), bits, group, out=outs)
        C.dequant_scatter_paged(c, sc, z, slots, 1, T, H, D, group, bits, kc, vc)
        elapsed += time.perf_counter() - t0
        layers += 1
        if budget_s is not None and elapsed >= budget_s:
            break
    fp16_bytes = layers * 2 * T * H * D * 2
    return dict(value=fp16_bytes / elapsed / 1e9, unit=UNIT, cores=C.threads(), kind="port",
                cpu_model=cpu_model(), affinity=len(os.sched_getaffinity(0)),
                simd="avx2+f16c+fma" if C.simd() else "scalar",
                sample=f"{layers} layers ({layers / L:.2f} passes over the {L}) of {workload} "
                       f"({fp16_bytes / 1e9:.2f} GB fp16), "
                       f"oracle/kvq_oracle.c quant+pack+dequant+paged-scatter "
                       f"({'AVX2/F16C' if C.simd() else 'scalar'}), "
                       f"{C.threads()} OpenMP threads on {cpu_model()}, {elapsed:.2f} s")


def cpu_torch_variant(workload: str, bits: int, group: int, budget_s: float = 5.0):
    """The torch-CPU variant SURVEY.md 8(d) asks for next to the C baseline:
    oracle/kvq_torch_cpu.py (the same arithmetic in torch ops, bit-identical
    to the oracle) with torch's intra-op pool on every usable core, layer by
    layer over the workload until ``budget_s``."""
    import torch
    from oracle import kvq_torch_cpu as TC
    L, H, D, b, s = WORKLOADS[workload]
    T = b * s
    nb = (T + BLOCK - 1) // BLOCK
    threads = len(os.sched_getaffinity(0))
    prev = torch.get_num_threads()
    torch.set_num_threads(threads)
    try:
        slots = torch.from_numpy(_CPU_LAYERS[("dst", workload)][0]) if ("dst", workload) in \
            _CPU_LAYERS else torch.randperm(nb * BLOCK)[:T]
        kc = torch.zeros((nb, BLOCK, H, D), dtype=torch.float16)
        vc = torch.zeros_like(kc)
        layers, elapsed = 0, 0.0
        while elapsed < budget_s and layers < 4 * L:
            kv = torch.from_numpy(_cpu_layer(workload, layers % L, T, H, D)).reshape(-1, D)
            t0 = time.perf_counter()
            c, sc, z = TC.quant_pack(kv, bits, group)
            TC.dequant_scatter_paged(c, sc, z, slots, T, H, D, group, bits, kc, vc)
            elapsed += time.perf_counter() - t0
            layers += 1
    finally:
        torch.set_num_threads(prev)
    fp16_bytes = layers * 2 * T * H * D * 2
    return {"value": round(fp16_bytes / elapsed / 1e9, 4), "unit": UNIT, "threads": threads,
            "sample": f"{layers} layers of {workload} ({fp16_bytes / 1e9:.2f} GB fp16), "
                      f"oracle/kvq_torch_cpu.py (torch {torch.__version__} CPU ops, "
                      f"{threads} intra-op threads), {elapsed:.2f} s"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    bits, group = args.bits, args.group
    wl = args.workload or ("cfg2_7b_2048x8" if world == 1 else default_pair_workload(world))
    L, H, D, b, s = WORKLOADS[wl]
    if not args.ref_layers:
        # the whole workload per step when it is at most 16 GB of fp16 KV
        # (~0.4-0.8 s of AVX2 work on 16 cores), else an 8 GB layer sample
        per_layer = 2 * b * s * H * D * 2
        args.ref_layers = L if L * per_layer <= 16e9 else max(1, min(L, round(8e9 / per_layer)))
    for _ in range(args.warmup):  # generates the sampled layers and the cache once
        cpu_reference(wl, bits, group, budget_s=None, max_layers=min(L, 4))
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_reference(wl, bits, group, budget_s=None, max_layers=args.ref_layers)
        vals.append(r["value"])
        secs.append(args.ref_layers * 2 * b * s * H * D * 2 / 1e9 / r["value"])
    value = statistics.median(vals)
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(secs), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp16->u4", "data": "synthetic",
        "config": base_config(wl, bits, group, args.format, fp16_bytes_of(wl)),
        "run": {"sample_layers_per_step": args.ref_layers},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": r["cores"],
                         "kind": "port", "cpu_model": r["cpu_model"], "affinity": r["affinity"],
                         "simd": r["simd"],
                         "sample": (f"each step: the whole workload ({L} layers); "
                                    if args.ref_layers >= L else
                                    f"each step: {args.ref_layers} of the workload's {L} layers "
                                    f"(bounded sample; GB/s is per fp16 byte processed); ")
                                   + r["sample"]},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


def fp16_bytes_of(wl: str):
    """fp16 KV bytes of one step of a fixed workload (None for traces)."""
    if wl not in WORKLOADS:
        return None
    L, H, D, b, s = WORKLOADS[wl]
    return L * 2 * b * s * H * D * 2


def base_config(wl, bits, group, fmt, fp16_bytes):
    """The workload identity both arms print (the same dict for the same run)."""
    l2 = ("inputs larger than L2 (no flush)" if fp16_bytes and fp16_bytes > L2_BYTES else
          "inputs fit in L2 (126 MB): a latency-bound workload, no bandwidth claim")
    return {"workload": wl, "bits": bits, "group": group, "block_size": BLOCK,
            "format": fmt, "l2": l2}


def _pair_roofline(fp16: float, wire: float, hbm_gbs: float, ms: float) -> dict:
    """Per pair and step: the link, prefill-HBM and decode-HBM times at the
    measured peaks, the bound among them and the step's fraction of it."""
    t = {"link": wire / (NVLINK_GBS * 1e9) * 1e3,
         "prefill_hbm": (fp16 + 2 * wire) / (hbm_gbs * 1e9) * 1e3,
         "decode_hbm": fp16 / (hbm_gbs * 1e9) * 1e3}
    bound = max(t, key=t.get)
    return {"step_roofline_ms": round(t[bound], 4), "step_bound": bound,
            "step_frac": round(t[bound] / ms, 4),
            "link_ms": round(t["link"], 4), "prefill_hbm_ms": round(t["prefill_hbm"], 4),
            "decode_hbm_ms": round(t["decode_hbm"], 4)}


def default_pair_workload(world: int) -> str:
    return "cfg3_13b_2048x8" if world == 2 else "cfg4_70b_gqa_pair"


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def synthetic_kv_device(torch, L, T, H, D, device, seed=0):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    kv = torch.empty((L, 2, T, H, D), dtype=torch.float16, device=device)
    for l in range(L):  # per layer keeps the fp32 temporary small
        kv[l].copy_(torch.randn((2, T, H, D), generator=g, device=device, dtype=torch.float32))
    ch = torch.randperm(D, generator=torch.Generator().manual_seed(seed))[:4].to(device)
    kv[:, 0, :, :, ch] *= 8  # K outlier channels
    return kv


def paged_slots(torch, T, device, slack_blocks=64, seed=0):
    need = (T + BLOCK - 1) // BLOCK
    nb = need + slack_blocks
    perm = torch.randperm(nb, generator=torch.Generator().manual_seed(seed + 1))[:need]
    t = torch.arange(T)
    return (perm[t // BLOCK] * BLOCK + t % BLOCK).to(device), nb


def run_local(args, torch):
    from paper_2502_09334_b200 import KvPrecision
    from paper_2502_09334_b200.datapath import HandoffPlan, HostHandoff, KVPlanes
    wl = args.workload or "cfg2_7b_2048x8"
    L, H, D, b, s = WORKLOADS[wl]
    T = b * s
    dev = torch.device("cuda", torch.cuda.current_device())
    kv = synthetic_kv_device(torch, L, T, H, D, dev)
    slots, nb = paged_slots(torch, T, dev)
    kc = torch.zeros((L, nb, BLOCK, H, D), dtype=torch.float16, device=dev)
    vc = torch.zeros_like(kc)
    if args.format == "kivi":
        from paper_2502_09334_b200.kivi import KiviHandoff
        plan = KiviHandoff(kv, kc, vc, slots, KvPrecision(args.bits), args.group, (s,) * b)
    else:
        plan = HandoffPlan(KVPlanes.dense(kv), KVPlanes.paged(kc, vc, slots), T,
                           KvPrecision(args.bits), args.group, mode="local", n_chunks=args.chunks,
                           bulk=None if args.k3 == "auto" else args.k3 == "bulk")
    lay = plan.layout
    fp16_bytes = lay.fp16_bytes
    for _ in range(args.warmup):
        plan.run()
    torch.cuda.synchronize()
    timing = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            plan.run(timing)
        end.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.steps
    launches_per_step = 6 if args.format == "kivi" else 2 * len(plan.chunks)
    k1 = sum(e["k1"][0].elapsed_time(e["k1"][1]) for e in timing) / args.steps
    k3 = sum(e["k3"][0].elapsed_time(e["k3"][1]) for e in timing) / args.steps
    kernel_bytes = fp16_bytes + lay.wire_bytes  # K1 reads fp16, writes payload; K3 the reverse
    hbm, peak_kind = peaks()
    k3_bulk = getattr(plan, "bulk", args.k3 == "bulk")
    k3_name = "pull_dequant_scatter_paged" if k3_bulk else "dequant_scatter_paged"
    dom, dom_ms = ("quant_pack", k1) if k1 >= k3 else (k3_name, k3)
    achieved = kernel_bytes / (dom_ms * 1e-3) / 1e9
    step_bytes = 2 * kernel_bytes  # algorithmic HBM bytes of the round trip
    roof_ms = step_bytes / (hbm * 1e9) * 1e3
    value = fp16_bytes / (ms * 1e-3) / 1e9

    # e2e: the same hand-off from pinned host KV to a host paged cache
    e2e = None
    if not args.no_e2e and args.format == "default":
        kv_h = torch.empty(kv.shape, dtype=torch.float16, pin_memory=True)
        kv_h.copy_(kv)
        # the host cache holds exactly the blocks this hand-off fills (a random
        # permutation of them): the D2H moves the hand-off's result, no slack
        e_slots, e_nb = paged_slots(torch, T, dev, slack_blocks=0)
        kc_h = torch.empty((L, e_nb, BLOCK, H, D), dtype=torch.float16, pin_memory=True)
        vc_h = torch.empty((L, e_nb, BLOCK, H, D), dtype=torch.float16, pin_memory=True)
        del plan
        host = HostHandoff(kv_h, kc_h, vc_h, e_slots, dev, KvPrecision(args.bits), args.group,
                           n_chunks=args.e2e_chunks)
        for _ in range(max(1, min(args.warmup, 3))):
            host.run()
        torch.cuda.synchronize()
        n_e2e = max(1, min(args.steps, args.e2e_steps or args.steps))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_e2e):
            host.run()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / n_e2e
        e2e = {"value": round(fp16_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": host.h2d_bytes, "d2h_bytes_per_step": host.d2h_bytes,
               "ms_per_step": round(e2e_ms, 3), "steps": n_e2e,
               "path": "pinned host KV -> H2D -> K1 -> K3 -> D2H of the paged cache (exactly "
                       f"the blocks the hand-off fills), {len(host.chunks)} layer chunks on 3 "
                       "streams"}
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_reference(wl, args.bits, args.group, budget_s=args.cpu_budget)
        if args.bits != 16 and args.format == "default":
            cpu["torch_cpu"] = cpu_torch_variant(wl, args.bits, args.group)
    traffic = ncu_traffic(wl, args, dom)
    return dict(
        value=value, ms=ms, workload=wl, fp16_bytes=fp16_bytes, wire_bytes=lay.wire_bytes,
        launches=launches_per_step * args.steps, clocks=clk.summary(), e2e=e2e, cpu=cpu,
        roofline={"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                  "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                  "frac": round(achieved / hbm, 4), "traffic": traffic,
                  "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram read+write "
                                    "per launch)" if traffic else None,
                  "algorithmic_bytes_per_launch": kernel_bytes // len(plan_chunks(args, L)),
                  "k1_ms": round(k1, 4), "k3_ms": round(k3, 4),
                  "step_roofline_ms": round(roof_ms, 4), "step_frac": round(roof_ms / ms, 4)},
        extra={"n_chunks": args.chunks, "mode": "local",
               "k3": "bulk" if k3_bulk else "ldg", "format": args.format},
    )


def ncu_traffic(workload, args, kernel):
    """DRAM traffic per launch of ``kernel`` from the committed ncu capture of
    this exact configuration (bench.py cannot run ncu itself), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            doc = json.load(f)
        key = f"{workload}/bits{args.bits}/g{args.group}/chunks{args.chunks}"
        if kernel == "pull_dequant_scatter_paged":  # K3-bulk on the local payload
            key += "/k3bulk"
        return int(doc["configs"][key][kernel]["traffic_bytes"])
    except Exception:  # noqa: BLE001
        return None


def ncu_link_traffic(workload, args):
    """NVLink bytes per K3-bulk launch of this configuration from the committed
    ncu capture (nvlrx user bytes = the payload exactly when nothing is
    re-read; raw bytes include the link protocol), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            doc = json.load(f)
        key = f"{workload}/bits{args.bits}/g{args.group}/nvlink_pull"
        return dict(doc["configs"][key]["pull_dequant_scatter_paged"], source=doc["source_" + key])
    except Exception:  # noqa: BLE001
        return None


def plan_chunks(args, L):
    from paper_2502_09334_b200.datapath import layer_chunks
    return layer_chunks(L, args.chunks)


def _calibration(spec, T, ms_large, ms_small, t_small=16, host_us=None):
    """(alpha, beta) of t = alpha + V/beta with V the reference's modelled
    volume 2*b*s*h*bits/8*L (costs.py:102) -- what calibrate.cluster_dict and
    measured_kv_comm_cost consume."""
    from paper_2502_09334_b200.calibrate import fit_alpha_beta
    v_large = spec.layout(T).fp16_bytes * spec.bits / 16
    v_small = spec.layout(t_small).fp16_bytes * spec.bits / 16
    try:
        alpha, beta = fit_alpha_beta(ms_small * 1e-3, v_small, ms_large * 1e-3, v_large)
    except ValueError:
        return None
    return {"alpha_us": round(alpha * 1e6, 2), "beta_GBps_of_modelled_volume": round(beta / 1e9, 1),
            "small_handoff_us": round(ms_small * 1e3, 2), "small_tokens": t_small,
            "host_enqueue_us_per_handoff": round(host_us, 2) if host_us is not None else None,
            "note": "t = alpha + (2*b*s*h*bits/8*L)/beta, per pair, back-to-back native "
                    "launches on the caller's stream"}


def run_pairs(args, torch, rank: int, world: int) -> None:
    """N > 1: weak-scaling pair benchmark -- every prefill -> decode pair
    (transport.pairing) hands off the same workload over its own NVLink."""
    import torch.distributed as dist

    from paper_2502_09334_b200.datapath import KVPlanes
    from paper_2502_09334_b200.transport import ChannelSpec, PairChannel, exchange, pairing
    B = sys.modules[__name__]

    local = int(os.environ.get("LOCAL_RANK", rank))
    # more ranks than GPUs (a dry run of the N=8 rank logic on a smaller box:
    # pairs i -> i+N/2 then share a GPU over same-device IPC; the numbers mean
    # nothing): gloo as the default group, since NCCL refuses duplicate GPUs
    oversub = world > torch.cuda.device_count()
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    wl = args.workload or B.default_pair_workload(world)
    trace = None
    if wl in B.TRACE_MODELS:
        L, H, D = B.TRACE_MODELS[wl]
        trace = B.make_trace(args.warmup + args.steps + 2, seed=0)
        T = B.TRACE_CAP
    else:
        L, H, D, b, s = B.WORKLOADS[wl]
        T = b * s
    mode = args.mode
    n_chunks = args.chunks or 8
    spec = ChannelSpec(L, T, H, D, args.bits, args.group, n_chunks, mode,
                       format=getattr(args, "format", "default"),
                       queue_depth=getattr(args, "queue_depth", 2),
                       pdl=not args.no_pdl, gate_recv=args.gate_recv,
                       gate_send=args.gate_send and not args.no_gate_send)
    ch = PairChannel(spec, rank, world, control_group=ctrl)
    lay = spec.layout(T)
    # per step token counts (fixed workload, or the trace's batches)
    tok = [T] * ((args.warmup + args.steps + 2) * args.batch) if trace is None else [
        sum(x) for x in trace]
    seqs = ([(s,) * b] * len(tok)) if trace is None else [tuple(x) for x in trace]
    it = {"i": 0}
    kivi = spec.format == "kivi"

    def next_t():
        t = tok[it["i"] % len(tok)]
        it["i"] += 1
        return t

    if ch.role == "prefill":
        kv = B.synthetic_kv_device(torch, L, T, H, D, dev, seed=ch.pair)
        planes = KVPlanes.dense(kv)
        def step(timing=None):
            for _ in range(args.batch if trace is None else 1):
                i = it["i"] % len(tok)
                t = next_t()
                if kivi:
                    ch.send(planes, t, timing, seqlens=seqs[i])
                else:
                    ch.send(planes, t, timing)
    else:
        # fixed workloads: a random permutation of exactly the blocks the
        # hand-off fills (the e2e download then moves only the result);
        # traces keep slack blocks for their per-request block rounding
        slots, nb = B.paged_slots(torch, T, dev, seed=ch.pair,
                                  slack_blocks=0 if trace is None else 64)
        kc = torch.zeros((L, nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
        vc = torch.zeros_like(kc)
        if trace is None and args.batch > 1:
            # decode rounds: each step drains `batch` queued hand-offs with
            # one pull launch (recv_many), each into its own blocks
            need = (T + B.BLOCK - 1) // B.BLOCK
            nbb = args.batch * need + 64
            kc = torch.zeros((L, nbb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
            vc = torch.zeros_like(kc)
            perm = torch.randperm(nbb, generator=torch.Generator().manual_seed(ch.pair + 1))
            tt = torch.arange(T)
            planes_k = [KVPlanes.paged(kc, vc, (perm[j * need + tt // B.BLOCK] * B.BLOCK +
                                                tt % B.BLOCK).to(dev))
                        for j in range(args.batch)]
            planes = planes_k[0]

            def step(timing=None):
                ch.recv_many([(pl, next_t()) for pl in planes_k], timing)
        elif trace is None and args.chained and not kivi:
            # chained pulls (kvx.h KVX_PAIR_CHAINED): every hand-off of a chain
            # lands in its own block set (a ring of up to 8 GB of sets); the
            # chain restarts with an unchained recv whenever the ring wraps,
            # so no two hand-offs that may be in flight together share blocks
            set_bytes = L * nb * B.BLOCK * H * D * 2 * 2
            n_sets = max(2, min(args.warmup + args.steps + 2, int(8e9 // set_bytes)))
            kc = torch.zeros((L, n_sets * nb, B.BLOCK, H, D), dtype=torch.float16, device=dev)
            vc = torch.zeros_like(kc)
            planes_ring = [KVPlanes.paged(kc, vc, slots + j * nb * B.BLOCK) for j in range(n_sets)]
            planes = planes_ring[0]
            torch.cuda.synchronize()  # the caches and slot mappings are ready

            def step(timing=None):
                j = it["i"] % n_sets
                ch.recv(planes_ring[j], next_t(), timing, chained=j > 0 and timing is None)
        elif trace is None:
            planes = KVPlanes.paged(kc, vc, slots)

            def step(timing=None):
                i = it["i"] % len(tok)
                t = next_t()
                if kivi:
                    ch.recv(planes, t, timing, seqlens=seqs[i])
                else:
                    ch.recv(planes, t, timing)
        else:
            # each batch gets its own random block placement (requests start on
            # a block boundary, as a paged allocator hands them out)
            import numpy as np
            rng = np.random.default_rng(ch.pair + 7)
            per_batch = []
            for lens in trace:
                nblk = sum((n + B.BLOCK - 1) // B.BLOCK for n in lens)
                blocks = rng.permutation(nb)[:nblk]
                sl, bi = [], 0
                for n in lens:
                    t = np.arange(n)
                    sl.append(blocks[bi + t // B.BLOCK] * B.BLOCK + t % B.BLOCK)
                    bi += (n + B.BLOCK - 1) // B.BLOCK
                per_batch.append(torch.from_numpy(np.concatenate(sl).astype(np.int64)).to(dev))
            planes_b = [KVPlanes.paged(kc, vc, sl) for sl in per_batch]

            def step(timing=None):
                i = it["i"] % len(tok)
                if kivi:
                    ch.recv(planes_b[i], next_t(), timing, seqlens=seqs[i])
                else:
                    ch.recv(planes_b[i], next_t(), timing)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with B.ClockSampler(local) as clk:
        t0.record()
        for _ in range(args.steps):
            step()  # one native kernel launch per end and hand-off (fused pull)
        t1.record()
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    # per-kernel durations: a separate eager pass with CUDA events on the
    # launching streams (events between launches break the PDL chaining)
    timing = []
    n_kt = max(1, min(args.steps, 5))
    for _ in range(n_kt):
        step(timing)
    torch.cuda.synchronize()
    dist.barrier()
    kern = {}
    for name, a, b_ in timing:
        kern[name] = kern.get(name, 0.0) + a.elapsed_time(b_) / n_kt
    launches = len(timing) / n_kt * args.steps
    # alpha-beta calibration of this very channel (native pull): a
    # 16-token hand-off against the main one -> kv_comm_cost's (alpha, beta)
    # for the reference's volume at this bit-width
    cal_small_ms, host_us = 0.0, 0.0
    if trace is None and not kivi:
        t_small = 16
        if ch.role == "prefill":
            small = lambda: ch.send(planes, t_small)  # noqa: E731
        else:
            sl_small = KVPlanes.paged(kc, vc, planes.slots[:t_small])
            small = lambda: ch.recv(sl_small, t_small)  # noqa: E731
        for _ in range(3):
            small()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_cal = 50
        h0 = time.perf_counter()
        c0.record()
        for _ in range(n_cal):
            small()
        c1.record()
        host_us = (time.perf_counter() - h0) / n_cal * 1e6  # enqueue cost per hand-off
        torch.cuda.synchronize()
        cal_small_ms = c0.elapsed_time(c1) / n_cal
        dist.barrier()
    # e2e through the same public API with host buffers: pinned host KV on the
    # prefill side (H2D inside the step), pinned host paged cache on the decode
    # side (D2H inside the step)
    e2e_ms, h2d, d2h = 0.0, 0, 0
    if not args.no_e2e and not kivi:
        if ch.role == "prefill":
            host = torch.empty(kv.shape, dtype=torch.float16, pin_memory=True)
            host.copy_(kv)
            stage = dict(stage_in=(host, kv))
            h2d = host.numel() * 2
            e2e_step = lambda: ch.send(planes, next_t(), None, **stage)  # noqa: E731
        else:
            hk = torch.empty(kc.shape, dtype=torch.float16, pin_memory=True)
            hv = torch.empty(vc.shape, dtype=torch.float16, pin_memory=True)
            stage = dict(stage_out=((kc, vc), (hk, hv)))
            d2h = (hk.numel() + hv.numel()) * 2
            e2e_step = (lambda: ch.recv(planes, next_t(), None, **stage)) if trace is None else (
                lambda: ch.recv(planes_b[it["i"] % len(tok)], next_t(), None, **stage))
        n_e2e = max(1, min(args.steps, args.e2e_steps or args.steps))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_e2e):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / n_e2e
        dist.barrier()
    stats = torch.tensor([ms, kern.get("k1", 0.0), kern.get("k3", 0.0), e2e_ms, h2d, d2h,
                          launches, cal_small_ms, host_us], dtype=torch.float64,
                         device="cpu" if oversub else dev)
    gathered = [torch.zeros_like(stats) for _ in range(world)]
    dist.all_gather(gathered, stats)
    clocks = exchange(clk.summary(), ctrl)
    if rank == 0:
        g = torch.stack(gathered).cpu()
        ms_max = float(g[:, 0].max())
        k1 = float(g[:, 1].max())
        k3 = float(g[:, 2].max())
        pairs = world // 2
        if kivi:
            timed = range(args.warmup, args.warmup + args.steps)
            fp16 = sum(spec.kivi_layout(seqs[i % len(tok)]).fp16_bytes for i in timed) / len(timed)
            wire_mean = sum(spec.kivi_layout(seqs[i % len(tok)]).wire_bytes
                            for i in timed) / len(timed)
        elif trace is None:
            fp16 = lay.fp16_bytes
        else:  # mean fp16 bytes of the timed batches
            timed = tok[args.warmup:args.warmup + args.steps]
            fp16 = sum(spec.layout(t).fp16_bytes for t in timed) / len(timed)
            wire_mean = sum(spec.layout(t).wire_bytes for t in timed) / len(timed)
        per_step = args.batch if trace is None else 1  # hand-offs per pair and step
        value = pairs * per_step * fp16 / (ms_max * 1e-3) / 1e9
        wire = lay.wire_bytes if (trace is None and not kivi) else wire_mean
        link_gbs = per_step * wire / (ms_max * 1e-3) / 1e9  # per pair
        hbm, peak_kind = B.peaks()
        k3_link = per_step * wire / (k3 * 1e-3) / 1e9 if k3 > 0 else None
        sm = [c["sm_mhz"] for c in clocks if c.get("sm_mhz")]
        reasons = sorted({r for c in clocks for r in c.get("reasons", [])})
        r = dict(
            value=value, ms=ms_max, workload=wl, fp16_bytes=fp16 * pairs * per_step,
            wire_bytes=wire * pairs * per_step,
            launches=int(g[:, 6].sum()),  # kvx kernels launched in the timed region
            clocks={"sm_mhz": min(sm) if sm else None,
                    "sm_max_mhz": max((c.get("sm_max_mhz") or 0) for c in clocks) or None,
                    "reasons": reasons, "per_rank_median_sm_mhz": sm},
            e2e=None if (args.no_e2e or kivi) else {
                "value": round(pairs * fp16 / (float(g[:, 3].max()) * 1e-3) / 1e9, 3),
                "unit": "GB/s", "h2d_bytes_per_step": int(g[:, 4].sum()),
                "d2h_bytes_per_step": int(g[:, 5].sum()),
                "ms_per_step": round(float(g[:, 3].max()), 3),
                "path": "pinned host KV -(H2D)-> K1 on P -(NVLink)-> K3 on D -(D2H)-> pinned "
                        "host paged cache, per layer chunk"},
            cpu=None,
            roofline={"bound": "nvlink", "kernel": "pull_dequant_scatter_paged (TMA bulk pull "
                      "over NVLink)" if mode == "pull" else f"hand-off ({mode})",
                      "achieved": round(link_gbs, 1), "peak": B.NVLINK_GBS,
                      "peak_kind": "measured TMA bulk-pull peer copy, tools/nvlink_bench.cu "
                                   "(770 in B200_PROFILING.md, 900 nominal)",
                      "unit": "GB/s", "frac": round(link_gbs / B.NVLINK_GBS, 4),
                      "traffic": None,  # DRAM traffic is not the bound here; see link_traffic
                      "link_traffic": B.ncu_link_traffic(wl, args),
                      "k1_ms": round(k1, 4), "k3_ms": round(k3, 4),
                      "k3_link_gbs": round(k3_link, 1) if k3_link else None,
                      "frac_of_nominal_900": round(link_gbs / 900.0, 4),
                      "hbm_peak": hbm,
                      # the pair's roofline is max(NVLink time,
                      # busiest-GPU HBM time).  P's HBM: K1 reads fp16 and
                      # writes the payload, the pull reads it; D's: fp16 writes
                      **_pair_roofline(per_step * fp16, per_step * wire, hbm, ms_max)},
            calibration=_calibration(spec, T, ms_max, float(g[:, 7].max()),
                                     host_us=float(g[:, 8].max())) if (
                trace is None and not kivi) else None,
            extra={"mode": mode,
                   "n_chunks": (len(ch._pull_chunks(lay)[0]) if mode in ("pull", "pull_ldg")
                                and not kivi else len(spec.chunks())),
                   "pairs": pairs,
                   "format": spec.format,
                   "native_pair": ch._pair is not None,
                   "pdl": spec.pdl, "gate_recv": spec.gate_recv, "gate_send": spec.gate_send,
                   "queue_depth": ch.Q,
                   **({"trace_batches_timed": tok[args.warmup:args.warmup + args.steps],
                       "trace": "lengths log-uniform [128, 8192], 1-16 req/batch, <=16384 "
                                "tokens/batch, rng(0)"} if trace is not None else {}),
                   "pairing": pairing(world), "parallelism": f"{pairs}P{pairs}D",
                   "handoffs_per_step": per_step,
                   **({"chained": "recv(chained=True), each hand-off of a chain into its own "
                                  "block set (the chain restarts when the set ring wraps)"}
                      if args.chained and trace is None and not kivi and args.batch == 1 else {}),
                   **({"oversubscribed_dry_run": f"{world} ranks on "
                       f"{torch.cuda.device_count()} GPUs (pairs share a GPU): not a measurement"}
                      if oversub else {}),
                   **({"decode_pull": f"recv_many: {per_step} queued hand-offs per pull launch"}
                      if per_step > 1 else {})},
        )
        emit(args, r, world)
    dist.barrier()
    ch.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS) + sorted(TRACE_MODELS))
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--format", default="default", choices=["default", "kivi"],
                    help="payload format: per-token groups, or KIVI per-channel K + residual")
    ap.add_argument("--group", type=int, default=128)
    ap.add_argument("--chunks", type=int, default=None,
                    help="layer chunks per hand-off (default: 1 at N=1; 8 per pair at N>1 for "
                    "the non-fused paths -- the fused pull picks layer-granular chunks itself)")
    ap.add_argument("--mode", default="pull", choices=["pull", "pull_ldg", "push", "copy", "nccl"])
    ap.add_argument("--k3", default="auto", choices=["auto", "ldg", "bulk"],
                    help="N=1: K3 variant (per-lane loads or TMA bulk staging; auto: "
                    "datapath.local_bulk_preferred, by row length)")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="host-buffer e2e steps (default: --steps; consecutive steps "
                    "pipeline, so few steps under-report the streaming rate)")
    ap.add_argument("--e2e-chunks", type=int, default=32,
                    help="N=1 e2e: layer chunks for H2D/compute/D2H overlap")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-layers", type=int, default=None,
                    help="reference arm: layers per step (default: the whole workload up to 16 GB of fp16 KV)")
    ap.add_argument("--chained", action="store_true",
                    help="N>1 fixed workloads: chained pulls (recv(chained=True)), each "
                         "hand-off of a chain into its own block set")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--queue-depth", type=int, default=4,
                    help="pull: queue slots per pair in the prefill GPU's HBM")
    ap.add_argument("--no-pdl", action="store_true",
                    help="N>1: no programmatic dependent launch between consecutive pulls")
    ap.add_argument("--tokens", type=int, default=None,
                    help="override the workload's token count (batch 1 x TOKENS) for sweeps")
    ap.add_argument("--batch", type=int, default=1,
                    help="N>1: hand-offs per step; the decode side drains them with ONE pull "
                         "launch (recv_many, a decode round's pull) -- needs --queue-depth >= it")
    ap.add_argument("--gate-send", action="store_true",
                    help="N>1: hold each K1 in the GPU front-end until its queue slot is free "
                         "(ChannelSpec.gate_send; default here: latency mode -- K1s chained with "
                         "PDL, waiting for the slot in-kernel)")
    ap.add_argument("--no-gate-send", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--gate-recv", action="store_true",
                    help="N>1: hold each pull in the GPU front-end until chunk 0 is published")
    args = ap.parse_args()
    if args.chained:
        args.no_e2e = True  # the ring of block sets would inflate the e2e download
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.tokens:
        base = args.workload or ("cfg2_7b_2048x8" if world == 1 else default_pair_workload(world))
        L, H, D, _, _ = WORKLOADS[base]
        args.workload = f"{base}@{args.tokens}x1"
        WORKLOADS[args.workload] = (L, H, D, 1, args.tokens)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    from paper_2502_09334_b200 import _lib
    _lib.load()
    if world > 1:
        run_pairs(args, torch, rank, world)
        return
    torch.cuda.set_device(0)
    args.chunks = args.chunks or 1
    r = run_local(args, torch)
    emit(args, r, world)


def emit(args, r, world):
    out = {
        "metric": METRIC, "value": round(r["value"], 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms"], 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp16" if args.bits == 16 else f"fp16->u{args.bits}",
        "data": "synthetic",
        "config": base_config(r["workload"], args.bits, args.group, args.format,
                              r["fp16_bytes"]),
        "run": {"fp16_bytes_per_step": r["fp16_bytes"], "wire_bytes_per_step": r["wire_bytes"],
                **r.get("extra", {})},
        "roofline": r["roofline"],
        "cpu_baseline": r["cpu"],
        "e2e": r["e2e"],
        "clocks": r["clocks"],
        "gpu_launches": r["launches"],
    }
    if r.get("calibration"):
        out["calibration"] = r["calibration"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
