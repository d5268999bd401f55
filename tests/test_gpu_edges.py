"""Edge cases of the CUDA path (through the C-ABI): empty and degenerate inputs, extreme seeds
and sample indices, isolated / absorbing rows, the multi-launch sampler window, and batches
mixing every lane-independent request shape.  Each is checked against the oracle (bit-exact
integer work, <= 4 ulp values, 1e-12 sums) or against a closed form."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1904_12754_b200 as P
from oracle import CSR

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ulp_diff(a, b):
    ia = np.asarray(a, np.float64).view(np.int64)
    ib = np.asarray(b, np.float64).view(np.int64)
    ia = np.where(ia < 0, np.int64(-(2 ** 63)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2 ** 63)) - ib, ib)
    return np.abs(ia - ib)


def test_empty_matrix_and_empty_batches(gpu):
    e = P.SparseMatrix.from_triplets(0, [], [], [])
    with P.Context(e, np.zeros(0)) as ctx:
        assert ctx.n == 0 and ctx.n_edges == 0
        assert ctx.run_level_batch(1.0, [], [], [], [], [], []).size == 0
        with pytest.raises(P.OutOfRange):
            P.run_level(P.MlmcProblem(ctx, 0, 1.0), 0, True, 0, 10, 1)
    z = P.SparseMatrix.from_triplets(3, [], [], [])  # zero matrix: every row absorbing, e^{0} = I
    with P.Context(z, [1.0, -2.0, 3.0]) as ctx:
        st = P.run_level(P.MlmcProblem(ctx, 1, 1.0), 3, True, 0, 1000, 5)
        assert st.sum == -2000.0 and st.sum_sq == 4000.0 and st.cost == 1000 * 8 and st.jumps == 0
        # count = 0 requests (any level, even 62) do nothing and raise nothing
        out = ctx.run_level_batch(1.0, [0, 1, 2], [62, 0, 5], [0, 1, 0], [0, 0, 0], [0, 0, 0], [1, 2, 3])
        assert np.all(out["samples"] == 0) and np.all(out["sum"] == 0.0)


def test_extreme_seeds_and_indices(gpu, oracle_lib):
    a = P.SparseMatrix.from_dense([[0.1, -1.0, 0.5], [0.7, -0.2, -0.2], [-0.4, 0.0, 0.3]])
    u = np.array([0.3, -1.1, 2.0])
    och = oracle_lib.chain(CSR(a.n, a.row_ptr, a.col, a.val))
    idx = np.array([0, 2 ** 32 - 1, 2 ** 32, 2 ** 63, 2 ** 64 - 2, 2 ** 64 - 1], np.uint64)
    with P.Context(a, u) as ctx:
        for seed in (0, 1, 2 ** 32 - 1, 2 ** 63 + 11, 2 ** 64 - 1):
            for level, base in ((0, 1), (4, 0), (9, 0)):
                got = ctx.sample_debug(0.9, 2, level, base, seed, idx)
                exp = och.samples(u, 2, 0.9, level, base, seed, idx)
                assert np.array_equal(got["cost"], exp["cost"]) and np.array_equal(got["end_state"], exp["end_state"])
                assert ulp_diff(got["fine"], exp["fine"]).max() <= 4
                assert ulp_diff(got["coarse"], exp["coarse"]).max() <= 4
        # run_level ranges near the top of the index space.  The reference's chunk bound
        # (chunk + 1) * 512 wraps to 0 for the last chunk before 2^64 and that chunk draws no
        # samples (parallel.hpp:46-49); the GPU path reproduces it, sample count included.
        for first, count in ((2 ** 64 - 1 - 700, 700), (2 ** 64 - 2 ** 20, 1000), (2 ** 64 - 600, 100)):
            st = P.run_level(P.MlmcProblem(ctx, 0, 0.9), 3, False, first, count, 2 ** 64 - 1)
            o = och.run_level(u, 0, 0.9, 3, 0, first, count, 2 ** 64 - 1)
            assert (st.samples, st.cost, st.jumps) == (o["samples"], o["cost"], o["jumps"])
            assert st.sum == pytest.approx(o["sum"], rel=1e-12, abs=1e-13)


def test_isolated_and_absorbing_rows(gpu, oracle_lib):
    # row 1 isolated (no entries), row 3 with only a diagonal, row 0 pointing into both
    a = P.SparseMatrix.from_triplets(4, [0, 0, 0, 2, 2, 3], [1, 3, 2, 0, 2, 3], [0.5, -0.25, 1.0, 0.3, -1.0, -0.7])
    u = np.array([1.0, 2.0, -3.0, 0.5])
    och = oracle_lib.chain(CSR(a.n, a.row_ptr, a.col, a.val))
    with P.Context(a, u) as ctx:
        dec = ctx.decomposition()
        assert dec["rate"][1] == 0.0 and dec["rate"][3] == 0.0
        for entry in range(4):
            for level, base in ((0, 1), (3, 0), (6, 0)):
                idx = np.arange(300, dtype=np.uint64)
                got = ctx.sample_debug(1.3, entry, level, base, 77 + entry, idx)
                exp = och.samples(u, entry, 1.3, level, base, 77 + entry, idx)
                assert np.array_equal(got["cost"], exp["cost"]) and np.array_equal(got["jumps"], exp["jumps"])
                assert ulp_diff(got["fine"], exp["fine"]).max() <= 4


def test_multi_window_launches_are_bitwise_identical(gpu, tmp_path):
    """The sampler's chunk-partial window (4M chunks per launch by default) set to 7 chunks in a
    child process: every request spans windows, the per-item combine continues across launches
    -- the results must equal the single-window run bit for bit."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs
cfg = configs.make_config("c1")
with P.Context(cfg.a, cfg.u) as ctx:
    e = np.arange(40) * 97 % cfg.a.n
    out = ctx.run_level_batch(cfg.beta, e, np.arange(40) % 5, (np.arange(40) % 5 == 0).astype(np.int32),
                              np.arange(40) * 311, 3000 + np.arange(40) * 17, 1000 + e)
    fw = ctx.run_level_batch(cfg.beta, 0, 2, 0, 0, 50000, 9, lane=P.LANE_FORWARD)
    np.save(sys.argv[2], np.concatenate([out, fw]))
'''
    res = {}
    for w in ("", "7"):
        env = dict(os.environ)
        if w:
            env["EXPMC_WINDOW_CHUNKS"] = w
        path = str(tmp_path / f"w{w or 'default'}.npy")
        subprocess.run([sys.executable, "-c", code, ROOT, path], check=True, env=env)
        res[w] = np.load(path)
    assert res[""].tobytes() == res["7"].tobytes()


def test_long_paths_and_mixed_batch(gpu, oracle_lib):
    """Levels up to 12 (4096 fine steps per sample) next to level-0 requests in one batch."""
    from paper_1904_12754_b200 import configs

    cfg = configs.make_config("c1")
    och = oracle_lib.chain(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val))
    with P.Context(cfg.a, cfg.u) as ctx:
        reqs = [(5, 12, 0, 0, 40), (9, 0, 1, 3, 5000), (4095, 7, 0, 600, 513), (2048, 1, 0, 0, 1)]
        out = ctx.run_level_batch(cfg.beta, [r[0] for r in reqs], [r[1] for r in reqs], [r[2] for r in reqs],
                                  [r[3] for r in reqs], [r[4] for r in reqs], [1000 + r[0] for r in reqs])
        for k, (e, l, b, f, c) in enumerate(reqs):
            o = och.run_level(cfg.u, e, cfg.beta, l, b, f, c, 1000 + e)
            assert int(out[k]["cost"]) == o["cost"] and int(out[k]["jumps"]) == o["jumps"]
            assert float(out[k]["sum"]) == pytest.approx(o["sum"], rel=1e-12, abs=1e-13)


def test_event_sampler_multi_window_groups(gpu, monkeypatch):
    """k_sample_grouped with windows that are not a multiple of the 4-chunk group (groups
    straddle launches): same sample counts and costs as one window, sums to 1e-12."""
    from paper_1904_12754_b200 import configs

    cfg = configs.make_config("c3-20000")
    entries = np.array([0, 5, 77, 1234, 19999])
    levels = np.array([7, 8, 9, 7, 10])
    args = (cfg.beta, entries, levels, (levels == 7).astype(np.int32), [0, 100, 3, 512, 9],
            [300000, 70000, 20000, 4096, 9000], 1000 + entries)
    out = {}
    for w in ("", "7"):
        if w:
            monkeypatch.setenv("EXPMC_WINDOW_CHUNKS", w)
        with P.Context(cfg.a, cfg.u, sampler="event") as ctx:
            out[w] = ctx.run_level_batch(*args)
    for k in ("samples", "cost", "jumps"):
        assert np.array_equal(out[""][k], out["7"][k]), k
    for k in ("sum", "sum_sq"):
        assert np.allclose(out[""][k], out["7"][k], rtol=1e-12, atol=1e-12 * np.abs(out[""][k]).max()), k


def test_driver_too_few_levels_is_invalid_argument(gpu):
    """max_levels_above_l0 < 2 leaves fewer than two coupled levels: the reference's first driver
    iteration throws std::invalid_argument from bias_estimate (mlmc.cpp:45-47); here the same
    error, raised before any per-row state is sized from it (a negative value used to wrap)."""
    from paper_1904_12754_b200 import configs

    cfg = configs.make_config("c1")
    with P.Context(cfg.a, cfg.u) as ctx:
        for mla in (1, 0, -2, -100):
            with pytest.raises(P.InvalidArgument, match="two coupled levels"):
                P.mlmc_driver_rows(ctx, cfg.beta, [3, 4], [1003, 1004], P.MlmcOptions(max_levels_above_l0=mla))
        res, _ = P.mlmc_driver_rows(ctx, cfg.beta, [3], [1003], P.MlmcOptions(max_levels_above_l0=2))
        assert res["L"][0] <= 2


def test_level0_items_split_launch_bitwise(gpu):
    """Reference-order batches sample their level-0 items (base level, one fine step) with the
    step-free walker in a launch of their own (context.cu sample_launch, RefPolicy0): a batch
    mixing level-0 and coupled items of several levels, with empty requests and partial first
    chunks, returns bitwise what each request returns alone -- in one window and across many."""
    import subprocess
    import sys
    code = r'''
import numpy as np, paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs
cfg = configs.make_config("c1")
rng = np.random.default_rng(4)
k = 40
entry = rng.integers(0, cfg.a.n, k)
level = rng.integers(0, 4, k)
base = np.where(level == 0, 1, rng.integers(0, 2, k))
base[level > 0] = 0
base[::7] = 1  # base levels above 0 too (nsteps > 1: the general walker)
first = rng.integers(0, 3000, k).astype(np.uint64)
count = rng.integers(0, 5000, k).astype(np.uint64)
count[::9] = 0
seed = 1000 + entry
with P.Context(cfg.a, cfg.u) as c:
    both = c.run_level_batch(cfg.beta, entry, level, base, first, count, seed)
    for i in range(k):
        one = c.run_level_batch(cfg.beta, entry[i], level[i], base[i], first[i], count[i], seed[i])
        for f in ("sum", "sum_sq", "samples", "cost", "jumps"):
            assert both[f][i] == one[f][0], (i, f)
print("ok")
'''
    import os
    for window in (None, "7"):
        env = dict(os.environ)
        if window:
            env["EXPMC_WINDOW_CHUNKS"] = window
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("beta", [0.7, 900.0])
def test_level0_walker_matches_oracle_on_every_row_kind(gpu, oracle_lib, beta):
    """The level-0 walker (RefPolicy0 / walker0_event: level 0, base, one fine step) against the
    oracle's run_level on a matrix with every kind of row its fast paths distinguish: uniform rows
    of degree 1, 2, 4, 8 (one-shift pick), uniform rows of degree 3, 5, 6, 7 (exact-floor pick),
    non-uniform rows of degree <= 4 and > 4 (CDF count / binary search), mixed signs, absorbing
    rows, and rates spread over five decades (S-mode -> T-mode on a rate change).  beta = 900 puts
    rate * dt past the S-mode range on the fast rows (T-mode from the first event).  Draw chains
    are exact: cost and jump counts equal the oracle's; sums to 1e-12."""
    rng = np.random.default_rng(29)
    n = 72
    dense = np.zeros((n, n))
    for i in range(n):
        kind = i % 6
        if kind == 5:
            continue  # absorbing: no off-diagonal entries
        if kind in (0, 1):  # uniform rows: equal magnitudes, degree 1..8
            deg = [1, 2, 4, 8, 3, 5, 6, 7][(i // 6) % 8]
            cols = rng.choice([j for j in range(n) if j != i], size=deg, replace=False)
            dense[i, cols] = rng.choice([-1.0, 1.0], size=deg) * (2.0 if kind == 0 else 0.37)
        else:  # non-uniform rows, narrow and wide
            deg = int(rng.integers(2, 5)) if kind == 2 else int(rng.integers(5, 13))
            cols = rng.choice([j for j in range(n) if j != i], size=deg, replace=False)
            dense[i, cols] = rng.uniform(-1.5, 1.5, deg)
        dense[i] *= 10.0 ** rng.integers(-3, 2)  # rates over five decades
    # d = a_ii + rate in (-0.5, 0.3): e^{beta d} and its square stay finite at beta = 900
    np.fill_diagonal(dense, -np.abs(dense).sum(axis=1) + rng.uniform(-0.5, 0.3, n))
    a = P.SparseMatrix.from_dense(dense)
    u = rng.uniform(-1.0, 1.0, n)
    och = oracle_lib.chain(CSR(a.n, a.row_ptr, a.col, a.val))
    entries = np.arange(n)
    count = 3000 if beta < 10 else 400  # beta = 900: hundreds of jumps per path on the fast rows
    with P.Context(a, u) as ctx:
        got = ctx.run_level_batch(beta, entries, 0, 1, 0, count, 77 + entries)
    for e in entries:
        o = och.run_level(u, int(e), beta, 0, 1, 0, count, 77 + int(e))
        assert int(got["cost"][e]) == o["cost"] and int(got["jumps"][e]) == o["jumps"], (e, e % 6)
        # signed terms cancel: the summation-order rounding scales with sum |x| <= sqrt(count sum x^2)
        assert abs(float(got["sum"][e]) - o["sum"]) <= 1e-12 * max(1.0, math.sqrt(count * o["sum_sq"])), (e, e % 6)
        assert abs(float(got["sum_sq"][e]) - o["sum_sq"]) <= 1e-12 * max(1.0, abs(o["sum_sq"])), (e, e % 6)
