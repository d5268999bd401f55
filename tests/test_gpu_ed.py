"""GPU: the event-driven sampler (csrc/ed_walker.cuh) -- same path law, different draws.

Exact checks where the law leaves no randomness (the reference unit tests' known answers:
diagonal, K2 = e, coupled difference 0 on constant d, sign parity), the cost identity
(cost = jumps + #non-absorbing boundaries + 2^l), and statistical agreement with the
reference-order sampler (which is bit-for-bit the reference) at 4 standard errors.
"""
import math

import numpy as np
import pytest

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs
from oracle import CSR

pytestmark = pytest.mark.gpu


def test_ed_known_answers(gpu):
    # diagonal: never moves, cost = steps (absorbing rows draw nothing), value exact (test_paths.cpp:84-99)
    with P.Context(P.SparseMatrix.from_dense([[0.75, 0.0], [0.0, -0.5]]), np.array([3.0, 5.0]), sampler="event") as c:
        s = c.sample_debug(2.0, 0, 3, 1, 2, np.arange(50))
        assert np.all(s["cost"] == 8) and np.all(s["jumps"] == 0)
        assert np.all(s["fine"] == s["fine"][0])
        assert s["fine"][0] == pytest.approx(3.0 * math.exp(1.5), rel=1e-14)
        s = c.sample_debug(2.0, 0, 3, 0, 4, np.arange(50))  # coupled on constant d: difference exactly 0
        assert np.all(s["fine"] - s["coarse"] == 0.0)
    # K2: d constant = 1 -> every path is exactly e (test_paths.cpp:101-111)
    with P.Context(P.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 0.0]]), np.ones(2), sampler="event") as c:
        s = c.sample_debug(1.0, 0, 4, 1, 3, np.arange(1000))
        assert np.all(s["fine"] == math.exp(1.0))
        assert np.all(s["cost"] == s["jumps"] + 2 * 16)  # no absorbing rows: cost = jumps + 2 N
        r = c.run_level_batch(1.0, 0, 4, 0, 0, 5000, 7)
        assert r["sum"][0] == 0.0 and r["sum_sq"][0] == 0.0


def test_ed_sign_parity(gpu):  # test_paths.cpp:226-249
    pos = P.SparseMatrix.from_dense([[0, 1.0, 0], [1.0, 0, 0.5], [0, 0.5, 0]])
    neg = P.SparseMatrix.from_dense([[0, -1.0, 0], [-1.0, 0, -0.5], [0, -0.5, 0]])
    u = np.array([1.0, 2.0, 3.0])
    with P.Context(pos, u, sampler="event") as cp, P.Context(neg, u, sampler="event") as cn:
        a = cp.sample_debug(2.0, 0, 2, 1, 8, np.arange(300))
        b = cn.sample_debug(2.0, 0, 2, 1, 8, np.arange(300))
    assert np.array_equal(a["end_state"], b["end_state"]) and np.array_equal(a["jumps"], b["jumps"])
    assert np.array_equal(b["fine"], a["fine"] * np.where(a["jumps"] % 2 == 0, 1.0, -1.0))


def test_ed_absorbing_cost_identity(gpu):
    # row 1 absorbing: cost = jumps + #{k >= 1 : rate(s_k) > 0} + N; check the bound and the mean
    a = P.SparseMatrix.from_dense([[0.0, 1.0, 0.5], [0.0, -1.0, 0.0], [0.25, 0.25, 0.0]])
    u = np.array([1.0, 2.0, 3.0])
    with P.Context(a, u, sampler="event") as ce, P.Context(a, u) as cr:
        e = ce.sample_debug(1.3, 0, 3, 0, 11, np.arange(20000))
        r = cr.sample_debug(1.3, 0, 3, 0, 11, np.arange(20000))
    n = 8
    assert np.all(e["cost"] <= e["jumps"] + 2 * n) and np.all(e["cost"] >= e["jumps"] + n)
    for key in ("cost", "jumps"):
        me, mr = e[key].mean(), r[key].mean()
        se = math.sqrt(e[key].var() / len(e[key]) + r[key].var() / len(r[key]))
        assert abs(me - mr) < 4 * se + 1e-12, key


@pytest.mark.parametrize("level,base", [(0, 1), (2, 1), (1, 0), (3, 0), (5, 0)])
def test_ed_matches_reference_order_statistically(gpu, level, base):
    cfg = configs.make_config("c1")
    rows = np.array([0, 63, 130, 2080, 4095])
    n = 400_000
    with P.Context(cfg.a, cfg.u) as cr, P.Context(cfg.a, cfg.u, sampler="event") as ce:
        r = cr.run_level_batch(cfg.beta, rows, level, base, 0, n, 1000 + rows)
        e = ce.run_level_batch(cfg.beta, rows, level, base, 0, n, 77 + rows)
    for k in range(len(rows)):
        mr, me = r["sum"][k] / n, e["sum"][k] / n
        vr = max(r["sum_sq"][k] / n - mr * mr, 0.0)
        ve = max(e["sum_sq"][k] / n - me * me, 0.0)
        se = math.sqrt((vr + ve) / n)
        assert abs(mr - me) <= 4 * se + 1e-15, (level, base, rows[k], mr, me, se)
        cr_, ce_ = r["cost"][k] / n, e["cost"][k] / n  # same unit cost in expectation
        assert abs(cr_ - ce_) <= 0.02 * cr_ + 0.05, (cr_, ce_)


def test_ed_driver_c1_rows_vs_exact(gpu, oracle_lib):
    cfg = configs.make_config("c1")
    rows = np.arange(0, cfg.a.n, 16)
    with P.Context(cfg.a, cfg.u, sampler="event") as c:
        res, _ = P.mlmc_driver_rows(c, cfg.beta, rows, configs.row_seeds(rows), P.MlmcOptions(epsilon=cfg.epsilon))
    exact = oracle_lib.dense_expmv(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val), cfg.u, cfg.beta)[rows]
    err = res["estimate"] - exact
    assert res["converged"].all()
    assert math.sqrt(float(np.mean(err ** 2))) <= cfg.epsilon
    assert float(np.mean(np.abs(err) > 3 * res["statistical_error"] + res["bias_estimate"])) <= 0.02


@pytest.mark.parametrize("level,base", [(0, 1), (3, 1), (1, 0), (4, 0)])
def test_ed_closed_form_first_hold_is_exact(gpu, level, base):
    # The closed-form first hold (ed_walker.cuh) must reproduce the full first event bit for
    # bit: per-sample values, costs, jumps and end states, and the run_level counts (sums to
    # 1e-12: the screened chunk loop changes the summation order), with the shortcut on and off.  Small rates so that most samples never leave the entry, plus a row
    # with d != 0 (non-trivial exponent), a negative off-diagonal and an absorbing row.
    rng = np.random.default_rng(5)
    n = 40
    dense = np.where(rng.random((n, n)) < 0.1, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    np.fill_diagonal(dense, rng.uniform(-2.0, 1.0, n))
    dense[7, :] = 0.0
    dense[7, 7] = -0.5  # absorbing
    a = P.SparseMatrix.from_dense(dense)
    u = rng.uniform(-1.0, 1.0, n)
    rows = np.array([0, 3, 7, 11, 39])
    with P.Context(a, u, sampler="event") as c:
        c.set_screen_each(True)  # per-sample screen: the same draws as the full first event
        for beta in (0.05, 0.7):
            c.set_full_hold(False)
            fast = c.sample_debug(beta, rows[:, None].repeat(400, 1).ravel(), level, base,
                                  (1000 + rows)[:, None].repeat(400, 1).ravel(), np.tile(np.arange(400), len(rows)))
            rf = c.run_level_batch(beta, rows, level, base, 3, 40_000, 1000 + rows)
            c.set_full_hold(True)
            full = c.sample_debug(beta, rows[:, None].repeat(400, 1).ravel(), level, base,
                                  (1000 + rows)[:, None].repeat(400, 1).ravel(), np.tile(np.arange(400), len(rows)))
            rr = c.run_level_batch(beta, rows, level, base, 3, 40_000, 1000 + rows)
            for k in ("fine", "coarse", "cost", "jumps", "end_state"):
                assert np.array_equal(fast[k], full[k]), (beta, k)
            for k in ("cost", "jumps"):
                assert np.array_equal(rf[k], rr[k]), (beta, k)
            # the screened chunk loop adds the closed-form samples first: same terms, other order
            for k in ("sum", "sum_sq"):
                assert np.allclose(rf[k], rr[k], rtol=1e-12, atol=1e-12 * np.abs(rr[k]).max()), (beta, k)
            if beta == 0.05:
                assert np.mean(fast["jumps"] == 0) > 0.5  # the shortcut was exercised
        if level == 0:  # classical MC (Welford in sample order): bitwise equal with and without
            mc = {}
            for full_hold in (False, True):
                c.set_full_hold(full_hold)
                mc[full_hold] = [P.mc_single_entry(c, int(e), 0.05, 0.05 / 8, 30_000, 9 + int(e)) for e in rows]
            for x, y in zip(mc[False], mc[True]):
                assert (x.estimate, x.std_error, x.wall_cost, x.jumps) == (y.estimate, y.std_error, y.wall_cost, y.jumps)


@pytest.mark.parametrize("level,base", [(0, 1), (3, 1), (1, 0), (4, 0)])
def test_ed_geometric_screen_matches_per_sample_screen(gpu, level, base):
    """The chunk kernel's geometric screen (jumpers located by Geometric gaps, their first draw
    conditioned on leaving the entry; ed_walker.cuh) has the per-sample screen's law: level
    means, mean unit cost and mean jumps agree at 4 combined SE on rows where most samples are
    held (the screen is on), and the held count is exact in expectation."""
    rng = np.random.default_rng(11)
    n = 60
    dense = np.where(rng.random((n, n)) < 0.08, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    np.fill_diagonal(dense, rng.uniform(-1.5, 0.5, n))
    a = P.SparseMatrix.from_dense(dense)
    u = rng.uniform(-1.0, 1.0, n)
    rows = np.array([0, 5, 17, 31, 44, 59])
    m = 400_000
    out = {}
    for each in (False, True):
        with P.Context(a, u, sampler="event") as c:
            c.set_screen_each(each)
            # first index not chunk-aligned: the first chunk is partial
            out[each] = c.run_level_batch(0.08, rows, level, base, 100, m, 300 + rows)
    g, e = out[False], out[True]
    for k in range(len(rows)):
        mg, me = g["sum"][k] / m, e["sum"][k] / m
        vg = max(g["sum_sq"][k] / m - mg * mg, 0.0)
        ve = max(e["sum_sq"][k] / m - me * me, 0.0)
        se = math.sqrt((vg + ve) / m)
        assert abs(mg - me) <= 4 * se + 1e-15, (rows[k], mg, me, se)
        for key in ("jumps", "cost"):
            # per-sample counts: Poisson-like, variance <= mean * (max per-sample count) -- a loose SE
            a_, b_ = float(g[key][k]), float(e[key][k])
            assert abs(a_ - b_) <= 4 * math.sqrt(2 * max(a_, b_) * (1 << (level + 2))) + 1, (key, rows[k], a_, b_)


def test_ed_edge_records_equal_row_gathers(gpu):
    """The per-edge records carrying the target row's payload (EdgeRec) change where a jump reads
    the landing row from, not what it reads: per-sample outputs and run_level results are
    bitwise those of the separate row gather, on uniform rows (grid), alias rows and absorbing
    rows alike."""
    rng = np.random.default_rng(17)
    n = 50
    dense = np.where(rng.random((n, n)) < 0.1, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    np.fill_diagonal(dense, rng.uniform(-2.0, 0.5, n))
    dense[9, :] = 0.0
    dense[9, 9] = -1.0  # absorbing
    for a, beta, rows in ((P.SparseMatrix.from_dense(dense), 0.9, np.array([0, 9, 21, 49])),
                          (configs.make_config("c1").a, 1.0, np.array([0, 130, 2080]))):
        u = rng.uniform(-1.0, 1.0, a.n)
        out = {}
        for sep in (False, True):
            with P.Context(a, u, sampler="event") as c:
                c.set_row_gather(sep)
                e = np.repeat(rows, 300)
                s = c.sample_debug(beta, e, 3, 0, 100 + e, np.tile(np.arange(300), len(rows)))
                r = c.run_level_batch(beta, rows, 2, 0, 0, 50_000, 7 + rows)
                out[sep] = (s, r)
        for k in ("fine", "coarse", "cost", "jumps", "end_state"):
            assert np.array_equal(out[False][0][k], out[True][0][k]), k
        for k in ("sum", "sum_sq", "cost", "jumps"):
            assert np.array_equal(out[False][1][k], out[True][1][k]), k


@pytest.mark.parametrize("level,base", [(0, 1), (2, 0)])
def test_ed_geometric_screen_is_split_invariant(gpu, level, base):
    """The driver extends a level in pieces (run_level(first, additional), mlmc.cpp:188-199), so a
    chunk can be sampled partly in one call and partly in the next.  The geometric screen lays its
    gaps from the chunk's first sample in every call, so the jumper set -- and with it every
    sample's path -- does not depend on where the calls split: jumps and costs are exactly those
    of one call over the same samples, sums equal up to summation order.  (Before this rule a split
    chunk re-used its first gaps for the second piece: correlated samples across extensions.)"""
    rng = np.random.default_rng(23)
    n = 60
    dense = np.where(rng.random((n, n)) < 0.08, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    np.fill_diagonal(dense, rng.uniform(-1.5, 0.5, n))
    a = P.SparseMatrix.from_dense(dense)
    u = rng.uniform(-1.0, 1.0, n)
    rows = np.array([0, 5, 17, 31, 44, 59])
    total = 100_000
    with P.Context(a, u, sampler="event") as c:
        one = c.run_level_batch(0.08, rows, level, base, 0, total, 300 + rows)
        parts = [c.run_level_batch(0.08, rows, level, base, f, k, 300 + rows)
                 for f, k in ((0, 1000), (1000, 37), (1037, 50_000 - 1037), (50_000, total - 50_000))]
    for key in ("cost", "jumps"):
        assert np.array_equal(one[key], sum(p[key] for p in parts)), key
    for key in ("sum", "sum_sq"):
        np.testing.assert_allclose(sum(p[key] for p in parts), one[key], rtol=1e-11, atol=1e-13)
