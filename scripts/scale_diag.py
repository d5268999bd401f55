"""Diagnostic for the configured-size parity tests: run the MLMC driver on a scale fixture's
components with both samplers and with shifted row seeds, dump per-component results (estimate,
SE, l0, L, per-level samples) to gpurun_out/diag_<name>.json for offline analysis.

    python scripts/scale_diag.py c3
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
fx = json.load(open(os.path.join("tests", "golden", f"scale_{name}.json")))
done = [r for r in fx["rows"] if not r.get("timed_out")]
rows = np.array([r["row"] for r in done], np.int64)
cfg = configs.make_config(name)
out = {"rows": rows.tolist()}
for sampler, shift in (("event", 0), ("event", 7_000_000), ("event", 13_000_000), ("reference", 0),
                       ("reference", 7_000_000), ("reference", 13_000_000)):
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
json.dump(out, open(f"gpurun_out/diag_{name}.json", "w"))
