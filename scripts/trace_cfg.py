"""Driver timeline of one config solve (EXPMC_TRACE=1 prints per-round build / wait / advance)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1904_12754_b200 as P  # noqa: E402
from paper_1904_12754_b200 import configs  # noqa: E402

name, nrows = sys.argv[1], int(sys.argv[2])
cfg = configs.make_config(name)
universe = cfg.rows if cfg.rows is not None else np.arange(cfg.a.n, dtype=np.int64)
rows = np.sort(np.random.default_rng(3).choice(universe, size=min(nrows, len(universe)), replace=False))
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 1e10
opts = P.MlmcOptions(epsilon=cfg.epsilon, max_levels_above_l0=cfg.max_levels_above_l0, max_cost=budget)
ctx = P.Context(cfg.a, cfg.u, sampler=cfg.sampler)
for i in range(2):
    k0 = ctx.counters()["sampler_ms"]
    t = time.perf_counter()
    P.mlmc_driver_rows(ctx, cfg.beta, rows, configs.row_seeds(rows), opts, want_levels=False)
    print(f"solve {1e3 * (time.perf_counter() - t):.1f} ms sampler {ctx.counters()['sampler_ms'] - k0:.1f} ms",
          file=sys.stderr)
