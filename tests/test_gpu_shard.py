"""GPU: sample sharding over GPUs (include/expmc_b200.h, expmc_ctx_shard_samples).

Only one GPU is available here, so the N-rank exchange is emulated on one device: rank r of N
runs the same batch with the chunk filter (expmc_ctx_set_shard) and its window of chunk
partials is read back; the elementwise sum over the emulated ranks must equal the unsharded
window bit for bit (every chunk non-zero on exactly one rank), which is what the NCCL
all-reduce computes.  The NCCL path itself runs with a communicator of size 1.
"""
import numpy as np
import pytest

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs

pytestmark = pytest.mark.gpu


def _batch(ctx, cfg):
    entries = np.array([0, 17, 100, 2080, 4095, 3000])
    levels = np.array([0, 1, 2, 3, 0, 4])
    return ctx.run_level_batch(cfg.beta, entries, levels, (levels == 0).astype(np.int32),
                               [0, 512, 7, 100000, 3, 0], [40000, 9000, 12345, 2048, 777, 5000], 1000 + entries)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_emulated_ranks_sum_exactly(gpu, world):
    cfg = configs.make_config("c1")
    with P.Context(cfg.a, cfg.u) as ctx:
        full = _batch(ctx, cfg)
        ref = ctx.last_partials()
        parts = []
        for r in range(world):
            ctx.set_shard(r, world)
            _batch(ctx, cfg)
            parts.append(ctx.last_partials())
        ctx.set_shard(0, 1)
    nz = np.zeros(len(ref["sum"]), int)
    for p in parts:
        nz += (p["cost"] != 0).astype(int)
    assert np.all(nz == 1)  # every chunk sampled on exactly one rank
    for k in ("sum", "sum_sq"):
        tot = np.zeros_like(ref[k])
        for p in parts:
            tot = tot + p[k]
        assert tot.tobytes() == ref[k].tobytes(), k
    for k in ("cost", "jumps"):
        assert np.array_equal(sum(p[k] for p in parts), ref[k])
    assert full["cost"].sum() == ref["cost"].sum()


def test_nccl_world_one_is_identity(gpu):
    cfg = configs.make_config("c1")
    with P.Context(cfg.a, cfg.u) as ctx:
        a = _batch(ctx, cfg)
        ctx.shard_samples(P.nccl_unique_id(), 0, 1)
        b = _batch(ctx, cfg)
        rows = np.array([3, 700, 2222])
        r1, _ = P.mlmc_driver_rows(ctx, cfg.beta, rows, configs.row_seeds(rows), P.MlmcOptions(epsilon=1e-2))
    with P.Context(cfg.a, cfg.u) as ctx2:
        r2, _ = P.mlmc_driver_rows(ctx2, cfg.beta, rows, configs.row_seeds(rows), P.MlmcOptions(epsilon=1e-2))
    assert a.tobytes() == b.tobytes()
    assert r1.tobytes() == r2.tobytes()


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_ranks_event_sampler_groups(gpu, world):
    # k_sample_grouped deals aligned chunk groups to ranks whole, so each rank's window holds
    # exactly the one-GPU partials of its groups (zeros elsewhere): the elementwise sum over the
    # emulated ranks is the unsharded window bit for bit, and the item totals follow.
    cfg = configs.make_config("c3-20000")
    with P.Context(cfg.a, cfg.u, sampler="event") as ctx:
        entries = np.array([0, 5, 77, 1234, 19999])
        levels = np.array([7, 8, 9, 7, 10])
        args = (cfg.beta, entries, levels, (levels == 7).astype(np.int32), [0, 100, 3, 512, 9],
                [300000, 70000, 20000, 4096, 9000], 1000 + entries)
        full = ctx.run_level_batch(*args)
        ref = ctx.last_partials()
        parts, outs = [], []
        for r in range(world):
            ctx.set_shard(r, world)
            outs.append(ctx.run_level_batch(*args))
            parts.append(ctx.last_partials())
        ctx.set_shard(0, 1)
    for k in ("sum", "sum_sq"):
        tot = np.zeros_like(ref[k])
        for p in parts:
            tot = tot + p[k]
        assert tot.tobytes() == ref[k].tobytes(), k
    for k in ("cost", "jumps"):
        assert np.array_equal(sum(p[k] for p in parts), ref[k])
    assert full["cost"].sum() == ref["cost"].sum()
