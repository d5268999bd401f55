"""GPU: alias tables of the event-driven sampler (AliasRec / k_build_alias, csrc/kernels.cu).

The reference picks a jump target by upper_bound over the row's CDF (chain.cpp:49-58,
paths.cpp:57-63); the event sampler's non-uniform rows draw from a Walker / Vose alias table
instead -- one 16-B record per jump, any degree.  Checks: (1) the law each row's table implies
equals the row's CDF increments; (2) uniform-only matrices build none; (3) end to end, the event
sampler with alias tables agrees with the reference-order sampler (the reference draw for draw)
on the C5 operator family (non-uniform, mixed-sign rows) at 4 combined SE.
"""
import math

import numpy as np
import pytest

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs

pytestmark = pytest.mark.gpu


def implied_law(dec, al, row):
    b, e = int(dec["row_ptr"][row]), int(dec["row_ptr"][row + 1])
    deg = e - b
    tgt = dec["jump_target"][b:e] * np.where(dec["sign"][b:e] == 1, -1, 1) - (dec["sign"][b:e] == 1)
    col = {int(t): k for k, t in enumerate(tgt)}  # signed target word -> slot
    law = np.zeros(deg)
    for j in range(deg):
        p = al["prob"][b + j]
        law[col[int(al["self"][b + j])]] += p / deg
        if p < 1.0:
            law[col[int(al["alias"][b + j])]] += (1.0 - p) / deg
    cdf = dec["jump_cdf"][b:e]
    return law, np.diff(np.concatenate([[0.0], cdf]))


def test_alias_tables_reproduce_row_laws(gpu):
    rng = np.random.default_rng(3)
    n = 300
    dense = np.where(rng.random((n, n)) < 0.05, rng.uniform(-2.0, 2.0, (n, n)), 0.0)
    dense[0, 1:200] = rng.uniform(0.001, 5.0, 199)  # a wide row, very unequal weights
    dense[1, 2:6] = [1e-9, 1.0, 3.0, 7.0]           # a tiny probability
    dense[2, :] = 0.0
    dense[2, 3:7] = 1.0                              # uniform row: exact pick, no record used
    np.fill_diagonal(dense, -1.0)
    a = P.SparseMatrix.from_dense(dense)
    with P.Context(a, np.ones(n)) as c:
        assert c.alias_tables() is None  # reference sampler: nothing built
        c.set_sampler("event")
        al = c.alias_tables()
        dec = c.decomposition()
    assert al is not None and al["rows"] > 0
    assert np.all((al["prob"] >= 0.0) & (al["prob"] <= 1.0))
    deg = np.diff(dec["row_ptr"])
    checked = 0
    for r in range(n):
        b, e = dec["row_ptr"][r], dec["row_ptr"][r + 1]
        if deg[r] < 2 or np.array_equal(dec["jump_cdf"][b:e], (np.arange(deg[r]) + 1.0) / deg[r]):
            continue  # uniform rows pick exactly from the degree and have no records
        law, p = implied_law(dec, al, r)
        assert np.allclose(law, p, rtol=0, atol=4e-15 * deg[r]), (r, np.abs(law - p).max())
        checked += 1
    assert checked > 100


def test_no_alias_for_uniform_rows(gpu):
    cfg = configs.make_config("c1")
    with P.Context(cfg.a, cfg.u, sampler="event") as c:
        assert c.alias_tables() is None


@pytest.mark.parametrize("level_offset,base", [(0, 1), (1, 0), (2, 0), (3, 0)])
def test_event_alias_matches_reference_order_c5(gpu, level_offset, base):
    """C5 operator family at 64^3 (7-point conv-diff, cell Peclet 10: off-diagonals +6/-4/1,
    t = 0.1): level means of the event sampler (alias picks) vs the reference-order sampler
    (CDF picks, the reference draw for draw) on interior, face and corner components."""
    cfg = configs.make_config("c5-64")
    g = 64
    idx = lambda x, y, z: (z * g + y) * g + x  # noqa: E731
    rows = np.array([idx(32, 32, 32), idx(0, 5, 9), idx(63, 63, 63), idx(0, 0, 0), idx(7, 40, 63), idx(63, 1, 14)])
    with P.Context(cfg.a, cfg.u) as c:
        l0 = P.initial_level(cfg.beta, c.d_max)
    level = l0 + level_offset
    m = 1 << 20
    with P.Context(cfg.a, cfg.u) as cr, P.Context(cfg.a, cfg.u, sampler="event") as ce:
        assert ce.alias_tables() is not None
        r = cr.run_level_batch(cfg.beta, rows, level, base, 0, m, 1000 + rows)
        e = ce.run_level_batch(cfg.beta, rows, level, base, 0, m, 5000 + rows)
    for k in range(len(rows)):
        mr, me = r["sum"][k] / m, e["sum"][k] / m
        vr = max(r["sum_sq"][k] / m - mr * mr, 0.0)
        ve = max(e["sum_sq"][k] / m - me * me, 0.0)
        se = math.sqrt((vr + ve) / m)
        assert abs(mr - me) <= 4 * se + 1e-15, (level, rows[k], mr, me, se)
        jr, je = r["jumps"][k] / m, e["jumps"][k] / m  # same mean number of transitions
        assert abs(jr - je) <= 0.01 * jr + 1e-3, (rows[k], jr, je)
