"""The bench JSON contract (task statement) on the committed bench line of this
round (profiles/r2h_bench_line.json, produced on a B200 by `python bench.py`): every key the
driver and the judge read is present and self-consistent. CPU-only: reads the file."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(ROOT, "profiles", "r2h_bench_line.json")


@pytest.fixture(scope="module")
def line():
    if not os.path.exists(LINE):
        pytest.skip("no committed bench line")
    with open(LINE) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_base_keys(line):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["warmup"] >= 3 and line["steps"] >= 1
    assert line["higher_is_better"] is True and line["scaling"] == "weak"
    assert line["dtype"] == "f64" and "workload" in line["config"]
    # value is the metric: evaluations per second = 1000 / ms_per_step at N = 1
    assert abs(line["value"] * line["ms_per_step"] / 1e3 * line["n_gpus"] - line["n_gpus"]) < 1e-6


def test_roofline_object(line):
    r = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # achieved = algorithmic bytes per launch / launch time
    assert abs(r["achieved"] - r["alg_bytes_per_launch"] / (r["launch_ms"] * 1e-3) / 1e9) < 1e-6 * r["achieved"]
    assert 0.0 < r["frac"] < 1.2


def test_cpu_baseline_and_e2e(line):
    c, e = line["cpu_baseline"], line["e2e"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(line["clocks"]["reasons"])


def test_cpu_baseline_is_measured_not_extrapolated_from_few(line):
    """>= 100 timed oracle iterations, phases timed separately, CPU model and
    threads stated; the projection's iteration count is named."""
    c = line["cpu_baseline"]
    assert c["pcg_iterations_timed"] >= 100
    for k in ("setup", "pcg_iteration", "sensitivity", "filter_build_and_transpose"):
        assert c["phases_s"][k] > 0
    assert c["cpu_model"] and c["threads"]["scipy_sparse"] == 1
    assert c["pcg_iterations_projected"] > 0 and "projected to" in c["sample"]
