"""Close the loop of SURVEY.md 8(f)1 on the CPU: run the reference's UNCHANGED
tabu-search planner (hetplan.search.tabu_search, imported read-only from
/root/reference) on the measured 8x B200 cluster (profiles/r01_b200x8_measured
.cluster.json, alpha/beta of our hand-off) with 16-bit and 4-bit KV, and with
the simulator's kv_comm_cost rebound to measured_kv_comm_cost.

  python tools/plan_with_measured.py      (needs /root/reference; CPU only)
"""
import importlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True
sys.path.append("/root/reference/pkg/src")


def main():
    from hetplan.core import ModelSpec, SloSpec, WorkloadProfile
    from hetplan.costs import CostParams, KvPrecision
    from hetplan.fixtures import trace_from_profile
    from hetplan.io import cluster_from_dict
    from hetplan.search import TabuParams, tabu_search

    from paper_2502_09334_b200 import measured_kv_comm_cost

    d = json.load(open(os.path.join(ROOT, "profiles", "r01_b200x8_measured.cluster.json")))
    cluster = cluster_from_dict(d)
    alpha, beta4 = d["alpha"][0][1], d["beta"][0][1]
    # LLaMA-2-70B with GQA: KV hidden = 8 heads x 128
    model = ModelSpec(n_layers=80, hidden_size=1024, n_params=70e9)
    workload = WorkloadProfile(arrival_rate=8.0, mean_input_len=4096, mean_output_len=128)
    slo = SloSpec(ttft_ref=1.0, tpot_ref=0.05, slo_scale=2.0)
    sim = importlib.import_module("hetplan.simulate")
    orch = importlib.import_module("hetplan.orchestrate")
    # fp16-equivalent measured rate: the 4-bit modelled volume is 1/4 of fp16
    measured = measured_kv_comm_cost({4: (alpha, beta4 * 4)})
    out = {}
    for bits in (16, 4):
        for label, fn in (("analytic", None), ("measured", measured)):
            if fn is not None and bits != 4:
                continue
            orig = (sim.kv_comm_cost, orch.kv_comm_cost)
            if fn is not None:
                sim.kv_comm_cost = orch.kv_comm_cost = fn
            try:
                res = tabu_search(cluster, model, workload, slo, prec=KvPrecision(bits),
                                  params=CostParams(),
                                  tp=TabuParams(n_step=15, n_nghb=8, rng_seed=0))
                trace = trace_from_profile(workload, n_requests=200, seed=0)
                s = sim.simulate(res.plan, trace, slo, CostParams(), seed=0, model=model,
                                 cluster=cluster)
            finally:
                sim.kv_comm_cost, orch.kv_comm_cost = orig
            kv = [r.kv_delay for r in s.records if r.completed]
            out[f"kv{bits}_{label}"] = {
                "best_score": round(res.best_score, 4),
                "n_prefill": len(res.plan.prefills), "n_decode": len(res.plan.decodes),
                "simulated_attainment_e2e": round(s.attainment_e2e, 4),
                "mean_kv_delay_us": round(1e6 * sum(kv) / max(1, len(kv)), 2),
            }
    print(json.dumps({"cluster": "8x B200, measured alpha/beta (r01)", "alpha_us": alpha * 1e6,
                      "beta_GBps_4bit_volume": beta4 / 1e9, **out}, indent=1))


if __name__ == "__main__":
    main()
