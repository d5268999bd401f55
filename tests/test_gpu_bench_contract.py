"""GPU: bench.py's JSON line keeps the driver's contract (one line, the keys and types the round-end
bench, the scaling run and the reference-arm comparison read), on the small C1 config."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*extra):
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "2", "--warmup", "3", *extra],
                       capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # exactly ONE JSON line on stdout
    return json.loads(lines[0])


def test_bench_line_contract(gpu):
    d = _line("--ref-seconds", "3")
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int), ("warmup", int),
                 ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str), ("dtype", str), ("data", str),
                 ("config", dict), ("roofline", dict), ("cpu_baseline", dict), ("e2e", dict), ("gpu_launches", int),
                 ("clocks", dict)):
        assert isinstance(d[k], t), (k, d[k])
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["vs_baseline"] is None
    assert d["unit"] == "transitions/s" and d["dtype"] == "f64" and d["data"] == "synthetic" and d["value"] > 0
    assert "workload" in d["config"] and "model" not in d["config"]
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and rf["unit"] in ("GB/s", "TFLOP/s")
    assert rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"]) and rf["peak"] > 0
    for k in ("traffic", "dram_frac", "l2_frac", "issue_frac", "modelled_gbs", "binding_resource"):
        assert k in rf
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] != d["value"]  # measured on its own, not a copy of the device-timed figure
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] >= c["sm_mhz"] and isinstance(c["reasons"], list)


def test_reference_arm_line_contract(gpu):
    ours = _line("--no-cpu-baseline", "--no-e2e")
    d = _line("--impl", "reference", "--ref-rows-per-step", "8")
    assert d["impl"] == "reference" and d["config"] == ours["config"]
    assert d["metric"] == ours["metric"] and d["unit"] == ours["unit"] and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
