import numpy as np, time, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs
cfg = configs.make_config("c2"); rows = np.arange(cfg.a.n); seeds = configs.row_seeds(rows)
ctx = P.Context(cfg.a, cfg.u)
for i in range(3):
    k0 = ctx.counters()["sampler_ms"]
    t = time.perf_counter(); P.mlmc_driver_rows(ctx, cfg.beta, rows, seeds, P.MlmcOptions(epsilon=cfg.epsilon), want_levels=False); t1 = time.perf_counter()
    print("solve %.1f ms sampler %.1f ms" % (1e3 * (t1 - t), ctx.counters()["sampler_ms"] - k0), file=sys.stderr)
