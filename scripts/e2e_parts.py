"""Where the end-to-end C2 step spends its time beyond the device-timed solve."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1904_12754_b200 as P  # noqa: E402
from paper_1904_12754_b200 import configs  # noqa: E402

cfg = configs.make_config("c2")
rows = np.arange(cfg.a.n)
seeds = configs.row_seeds(rows)
opts = P.MlmcOptions(epsilon=cfg.epsilon)
for it in range(3):
    t0 = time.perf_counter()
    ctx = P.Context(cfg.a, cfg.u)
    t1 = time.perf_counter()
    P.mlmc_driver_rows(ctx, cfg.beta, rows, seeds, opts, want_levels=False)
    t2 = time.perf_counter()
    k = ctx.counters()
    ctx.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms (sampler {k['sampler_ms']:.1f})  destroy {1e3*(t3-t2):.1f} ms")
