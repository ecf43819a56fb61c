"""GPU: bench.py's contract line (the driver parses it): the keys and their internal consistency,
on short C4 (decode: one fused launch per linear per step) and C3 (prefill: two) runs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,launches_per_linear", [("C4", 1), ("C3", 2)])
def test_bench_line(config, launches_per_linear):
    steps = 4
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--steps", str(steps),
                        "--warmup", "3", "--no-cpu", "--no-kv", "--no-fig6", "--no-fp16"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert d["unit"] == "tokens/s" and d["value"] > 0
    T = d["config"]["tokens_total"]
    assert abs(d["value"] - T / (d["ms_per_step"] * 1e-3)) / d["value"] < 0.01
    assert d["config"]["workload"].startswith(config)
    roof = d["roofline"]
    assert roof["bound"] in ("hbm", "tensor") and roof["unit"] in ("GB/s", "TOPS")
    assert roof["achieved"] > 0 and roof["peak"] > 0 and abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] < d["value"]                     # host copies make it slower than the device line
    # four linears per timed step: one fused launch each at decode sizes, transform + GEMM otherwise
    assert d["gpu_launches"] == 4 * launches_per_linear * steps
    assert d["clocks"]["sm_mhz"] > 0
