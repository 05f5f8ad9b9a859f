"""bench.py's JSON contract on CPU (reference arm) and its workload tables."""
import json
import subprocess
import sys

import bench


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--workload", "cfg1_7b_512x1", "--ref-layers", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_workloads_match_baseline_configs():
    # BASELINE.json configs 1-4: fp16 bytes per hand-off
    def fp16(name):
        L, H, D, b, s = bench.WORKLOADS[name]
        return L * 2 * b * s * H * D * 2
    assert fp16("cfg1_7b_512x1") == 268_435_456
    assert fp16("cfg2_7b_2048x8") == 8_589_934_592
    assert fp16("cfg3_13b_2048x8") == 13_421_772_800
    assert 4 * fp16("cfg4_70b_gqa_pair") == 10_737_418_240


def test_trace_is_deterministic_and_bounded():
    a, b = bench.make_trace(50, seed=0), bench.make_trace(50, seed=0)
    assert a == b
    for lens in a:
        assert 1 <= len(lens) <= 16 and sum(lens) <= bench.TRACE_CAP
        assert all(128 <= n <= 8192 for n in lens)


def test_pair_roofline_is_max_of_link_and_hbm():
    """a pair's roofline is max(NVLink time, busiest-GPU HBM time)."""
    fp16 = 13_421_772_800  # config 3
    r4 = bench._pair_roofline(fp16, 3_565_158_400, 6538.3, 4.6117)  # 4-bit G=128
    assert r4["step_bound"] == "link"
    assert abs(r4["link_ms"] - 3_565_158_400 / 783e9 * 1e3) < 1e-3
    assert r4["step_frac"] == round(r4["link_ms"] / 4.6117, 4)
    r2 = bench._pair_roofline(fp16, 2_097_152_000, 6538.3, 3.1243)  # 2-bit G=64
    assert r2["step_bound"] == "prefill_hbm"
    assert abs(r2["prefill_hbm_ms"] - (fp16 + 2 * 2_097_152_000) / 6538.3e9 * 1e3) < 1e-3
    assert r2["step_roofline_ms"] >= max(r2["link_ms"], r2["decode_hbm_ms"])
