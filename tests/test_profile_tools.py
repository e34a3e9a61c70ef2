"""The tooling that turns a capture into profiles/<round>/ and DESIGN.md's tables (CPU only)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROUND = os.path.join(ROOT, "profiles", "r02_v3")


def test_design_tables_render_from_the_committed_capture():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "profiles", "tools", "design_table.py"), ROUND],
                         capture_output=True, text=True, check=True).stdout
    assert "| **cfg5 8192×8192×16384 (default)** |" in out and "heavy-tailed X" in out
    assert "reference arm:" in out and "kind reference" in out


def test_committed_bench_lines_follow_the_contract():
    """Every committed line of the final capture carries the fields the driver reads; both arms
    describe the same workload; the timed point passed the parity gate."""
    ours = json.loads(open(os.path.join(ROUND, "bench_default.json")).read().strip().splitlines()[-1])
    ref = json.loads(open(os.path.join(ROUND, "bench_ref_default.json")).read().strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in ours, key
    assert ours["config"] == ref["config"] and ours["config"]["workload"] == "cfg5"
    assert ref["impl"] == "reference" and ref["e2e"]["h2d_bytes_per_step"] == 0
    assert ours["e2e"]["h2d_bytes_per_step"] == 8192 * 8192 * 4 and ours["e2e"]["d2h_bytes_per_step"] == 8192 * 16384 * 4
    assert ours["gpu_launches"] == 2 * ours["steps"]
    r = ours["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["traffic"] and 0.5 < r["tensor"]["frac"] <= 1.05  # against the int8 rate measured in the same run
    p = ours["parity"]
    assert p["normwise_vs_fp64"] <= 1e-5 and p["scaled_vs_fp64"] <= 1e-5 and p["integer_twin_bit_exact"]
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(ours["clocks"]["reasons"])
    traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    for cfg in ("cfg1", "cfg2", "cfg3_s1_16", "cfg3_s1_8", "cfg3_s1_4", "cfg3_s1_2", "cfg4", "cfg5"):
        assert traffic.get(f"{cfg}:mma"), cfg
