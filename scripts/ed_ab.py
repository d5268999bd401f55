"""Event-sampler kernel experiment: run_level batches (base level l0 and coupled l0+1, l0+2) over
seeded C3 components with the library in EXPMC_LIB; writes a SHA-256 of the results
(scripts/ed_ab.py OUT.sha) -- kernel variants that draw the same words must agree bit for bit."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs

cfg = configs.make_config("c3")
rng = np.random.default_rng(11)
rows = np.sort(rng.choice(cfg.a.n, size=16384, replace=False)).astype(np.int64)
with P.Context(cfg.a, cfg.u, sampler="event") as ctx:
    l0 = P.initial_level(cfg.beta, ctx.d_max)
    h = hashlib.sha256()
    for rep in range(2):
        for level, base in ((l0, 1), (l0 + 1, 0), (l0 + 2, 0)):
            ctx.reset_counters()
            r = ctx.run_level_batch(cfg.beta, rows, level, base, 0, 8192, 1000 + rows)
            k = ctx.counters()
            print(f"rep {rep} level {level}: sampler {k['sampler_ms']:.1f} ms, jumps {k['jumps']}", flush=True)
            if rep == 0:
                for key in ("sum", "sum_sq", "cost", "jumps"):
                    h.update(np.ascontiguousarray(r[key]).tobytes())
    with open(sys.argv[1], "w") as f:
        f.write(h.hexdigest() + "\n")
