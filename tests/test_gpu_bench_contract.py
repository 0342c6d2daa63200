"""bench.py's JSON line keeps the driver contract on the GPU: one line with
the headline keys, the roofline / e2e / clocks objects, the launch count, the
same `config` object as the reference arm, and (float64 lines) the
float32-within-tolerance leg."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config", ["C1", "C3"])
def test_bench_line_contract(config):
    d = _line("--config", config, "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["metric"] == "events/s" and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["steps"] == 5 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "fp64" and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    assert d["clocks"]["sm_mhz"] > 0
    alt = d["float32_within_tolerance"]
    assert alt["dtype"] == "f32" and alt["value"] > 0 and alt["e2e"]["value"] > 0
    # the reference arm prints the same config object (the driver compares them)
    from bench import workload_config

    assert d["config"] == workload_config(config, "f64")


def test_bench_bands_line():
    """`--bands N` (the C5 row-band split) prints one strong-scaling line."""
    d = _line("--config", "C5", "--bands", "2", "--steps", "3", "--warmup", "3")
    assert d["scaling"] == "strong" and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["sensor"] == "2048x2048"


@pytest.mark.parametrize("variant", ["rof", "l1", "tgv"])
def test_bench_variant_line(variant):
    """`--variant` (the operator-level solves of configs[1]) prints one line
    with its C-port baseline."""
    d = _line("--config", "C2", "--variant", variant, "--steps", "3", "--warmup", "3")
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0
