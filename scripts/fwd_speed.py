"""Forward vs entry sampling throughput on C2 (the grid is symmetric, so A^T = A): samples/s of
one big run_level batch per lane, CUDA-event timed by the library's sampler_ms counter."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs

cfg = configs.make_config("c2")
u = np.abs(cfg.u) + 0.1
with P.Context(cfg.a, u) as ctx:
    for lane, name in ((P.LANE_ENTRY, "entry"), (P.LANE_FORWARD, "forward")):
        for level in (0, 2):
            ctx.run_level_batch(cfg.beta, 12345, level, int(level == 0), 0, 1 << 20, 7, lane=lane)  # warm
            ctx.reset_counters()
            nreq = 256
            st = ctx.run_level_batch(cfg.beta, np.arange(nreq) * 4099 % cfg.a.n, level, int(level == 0), 0,
                                     1 << 22, np.arange(nreq), lane=lane)
            c = ctx.counters()
            print(f"{name:8s} level {level}: {c['samples'] / (c['sampler_ms'] * 1e-3):.3e} samples/s, "
                  f"{c['jumps'] / (c['sampler_ms'] * 1e-3):.3e} jumps/s, kernel {c['sampler_ms']:.1f} ms")
