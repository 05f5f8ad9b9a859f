"""Close the loop of SURVEY.md 8(f)1 on the CPU: run the reference's UNCHANGED
tabu-search planner and simulator (hetplan, imported read-only from
/root/reference) on a nominal 8x B200 NVSwitch node -- the datasheet link
model a planner would be given (beta = 900 GB/s per direction, alpha = 0) --
once with the reference's analytic kv_comm_cost and once with
``measured_kv_comm_cost`` rebound into hetplan.simulate / hetplan.orchestrate
(orchestrate.py:369-372, simulate.py:228-233), priced by the measured
hand-off table (tools/handoff_table.py, every bit-width 16/8/4/2).

Two workloads: LLaMA-2-70B-GQA at 4096-token prompts (bandwidth term
dominates) and at 128-token prompts (the measured per-hand-off alpha
dominates, which the datasheet model does not have).

  python tools/plan_with_measured.py --table profiles/r02_handoff_table.json \
      --out profiles/r02_plan_with_measured.json      (needs /root/reference)
"""
import argparse
import importlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True
sys.path.append("/root/reference/pkg/src")


def nominal_cluster(n=8):
    from paper_2502_09334_b200.calibrate import cluster_dict
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, flops = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    except Exception:  # noqa: BLE001
        hbm, flops = 6.65e12, 1.4e15
    return cluster_dict([[0.0] * n for _ in range(n)], [[900e9] * n for _ in range(n)],
                        local_beta=hbm, mem_bandwidth=hbm, peak_flops=flops)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--table", default=os.path.join(ROOT, "profiles", "r02_handoff_table.json"))
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=15)
    a = ap.parse_args()

    from hetplan.core import ModelSpec, SloSpec, WorkloadProfile
    from hetplan.costs import CostParams, KvPrecision
    from hetplan.fixtures import trace_from_profile
    from hetplan.io import cluster_from_dict
    from hetplan.search import TabuParams, tabu_search

    from paper_2502_09334_b200 import HandoffTable, install_measurements, measured_kv_comm_cost

    table = HandoffTable.from_json(a.table)
    cluster = cluster_from_dict(nominal_cluster())
    # LLaMA-2-70B with GQA: KV hidden = 8 heads x 128
    model = ModelSpec(n_layers=80, hidden_size=1024, n_params=70e9)
    slo = SloSpec(ttft_ref=1.0, tpot_ref=0.05, slo_scale=2.0)
    workloads = {"prompt4096": WorkloadProfile(arrival_rate=8.0, mean_input_len=4096,
                                               mean_output_len=128),
                 "prompt128": WorkloadProfile(arrival_rate=64.0, mean_input_len=128,
                                              mean_output_len=32)}
    sim = importlib.import_module("hetplan.simulate")
    orch = importlib.import_module("hetplan.orchestrate")
    prev = install_measurements(table)
    out = {"cluster": "nominal 8x B200 NVSwitch (beta 900 GB/s, alpha 0: the datasheet model)",
           "table": {k: list(v) for k, v in table.entries.items()}, "table_source": table.source,
           "model": "LLaMA-2-70B GQA (80 L, KV hidden 1024)"}
    try:
        for wname, workload in workloads.items():
            trace = trace_from_profile(workload, n_requests=200, seed=0)
            for bits in (16, 8, 4, 2):
                for label in ("analytic", "measured"):
                    orig = (sim.kv_comm_cost, orch.kv_comm_cost)
                    if label == "measured":
                        sim.kv_comm_cost = orch.kv_comm_cost = measured_kv_comm_cost
                    try:
                        res = tabu_search(cluster, model, workload, slo, prec=KvPrecision(bits),
                                          params=CostParams(),
                                          tp=TabuParams(n_step=a.steps, n_nghb=8, rng_seed=0))
                        s = sim.simulate(res.plan, trace, slo, CostParams(), seed=0, model=model,
                                         cluster=cluster)
                    finally:
                        sim.kv_comm_cost, orch.kv_comm_cost = orig
                    kv = [r.kv_delay for r in s.records if r.completed]
                    out[f"{wname}/kv{bits}_{label}"] = {
                        "best_score": round(res.best_score, 4),
                        "n_prefill": len(res.plan.prefills), "n_decode": len(res.plan.decodes),
                        "simulated_attainment_e2e": round(s.attainment_e2e, 4),
                        "mean_kv_delay_us": round(1e6 * sum(kv) / max(1, len(kv)), 2),
                    }
    finally:
        install_measurements(prev)
    txt = json.dumps(out, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")


if __name__ == "__main__":
    main()
