"""Seed-to-seed variability of the MLMC estimates at the configured sizes (TEST INFRASTRUCTURE).

On a GPU box: run the MLMC driver on a scale fixture's components with both samplers and with
shifted row seeds and dump per-component results (estimate, SE, l0, L, per-level samples) to
gpurun_out/diag_<name>.json:

    python scripts/scale_diag.py c3 [sampler:shift ...]     (default: both samplers, shifts 0, 7e6, 13e6)

Here (no GPU): turn that dump into the committed fixture tests/golden/scale_<name>_reseed.json,
which tests/test_gpu_scale_parity.py uses as the null distribution of the statistical rule -- the
reference-order sampler is the reference draw for draw (its shift-0 run reproduces the CPU
reference's fixture, asserted by the same test), so its shifted-seed runs are the reference's own
seed-to-seed spread:

    python scripts/scale_diag.py c3 --to-fixture
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12754_b200 as P  # noqa: E402
from paper_1904_12754_b200 import configs  # noqa: E402

name = sys.argv[1]
if "--to-fixture" in sys.argv:
    d = json.load(open(f"gpurun_out/diag_{name}.json"))
    out = {"generator": "scripts/scale_diag.py (GPU run) + --to-fixture", "config": name, "rows": d["rows"], "runs": {}}
    for key, r in d.items():
        if key == "rows":
            continue
        out["runs"][key] = {"estimate": [float(x).hex() for x in r["estimate"]],
                            "statistical_error": [float(x).hex() for x in r["se"]], "L": r["L"], "l0": r["l0"]}
    path = os.path.join("tests", "golden", f"scale_{name}_reseed.json")
    json.dump(out, open(path, "w"), indent=0)
    print("wrote", path, list(out["runs"]))
    sys.exit(0)
fx = json.load(open(os.path.join("tests", "golden", f"scale_{name}.json")))
done = [r for r in fx["rows"] if not r.get("timed_out")]
rows = np.array([r["row"] for r in done], np.int64)
cfg = configs.make_config(name)
out = {"rows": rows.tolist()}
runs = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[2:] if ":" in a] or [
    ("event", 0), ("event", 7_000_000), ("event", 13_000_000), ("reference", 0), ("reference", 7_000_000),
    ("reference", 13_000_000)]
for sampler, shift in runs:
    t0 = time.perf_counter()
    with P.Context(cfg.a, cfg.u, sampler=sampler) as ctx:
        res, lv = P.mlmc_driver_rows(ctx, cfg.beta, rows, configs.row_seeds(rows) + np.uint64(shift),
                                     P.MlmcOptions(epsilon=fx["epsilon"]))
    key = f"{sampler}_{shift}"
    out[key] = {"estimate": res["estimate"].tolist(), "se": res["statistical_error"].tolist(),
                "l0": res["l0"].tolist(), "L": res["L"].tolist(), "cost": res["total_cost"].astype(float).tolist(),
                "samples": [[int(x["samples"]) for x in lv[k][:int(res["nlevels"][k])]] for k in range(len(rows))]}
    print(key, f"{time.perf_counter() - t0:.1f}s", flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open(f"gpurun_out/diag_{name}.json", "w"))  # after every run: a cut-off call keeps the finished ones
