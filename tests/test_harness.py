"""Paper-figure harness (harness.cpp:41-177): fits against the reference's (bit for bit on the
same inputs) and, on the GPU, bench_levels / bench_l0 / bench_complexity against the
reference's own harness run on the same problem: costs and sample counts exact, level means
1e-12 and variances 1e-9 relative, slopes 1e-9."""
import numpy as np
import pytest

from oracle import CSR, have_reference

needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")


def grid(g):
    trips = []
    for y in range(g):
        for x in range(g):
            r = y * g + x
            trips.append((r, r, -4.0))
            for (dx, dy) in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                if 0 <= x + dx < g and 0 <= y + dy < g:
                    trips.append((r, r + dx + g * dy, 1.0))
    return CSR.from_triplets(g * g, trips)


@needs_ref
def test_fits_bitwise():
    from oracle import Reference

    from paper_1904_12754_b200 import harness as H

    ref = Reference()
    rng = np.random.default_rng(0)
    for _ in range(20):
        k = int(rng.integers(2, 12))
        x = rng.uniform(-3, 3, k)
        y = np.abs(rng.standard_normal(k)) * 10.0 ** rng.integers(-5, 5, k)
        y[rng.integers(0, k)] = 0.0 if k > 2 else y[0]
        assert H.fit_log2_slope(x, y) == ref.fit_slope(x, y, loglog=False)
        xp = np.abs(x) + 0.1
        assert H.fit_loglog_slope(xp, y) == ref.fit_slope(xp, y, loglog=True)


def test_fit_errors_and_csv(tmp_path):
    from paper_1904_12754_b200 import harness as H
    import paper_1904_12754_b200 as P

    with pytest.raises(P.InvalidArgument):
        H.fit_log2_slope([1.0, 2.0], [1.0, 0.0])
    assert H.fit_log2_slope([1, 2, 3], [2, 4, 8]) == pytest.approx(1.0)
    rep = H.LevelDecayReport([H.LevelDecayRow(1, 0.5, 1e-3, 2e-6, 12.0)], -2.0, -4.0, 1.0)
    H.write_level_decay_csv(rep, tmp_path / "l.csv")
    assert (tmp_path / "l.csv").read_text().splitlines() == [
        "level,dt,mean,variance,cost_per_sample", "1,0.5,0.001,2e-06,12",
        "# slope_mean=-2 slope_variance=-4 slope_cost_tail=1"]
    H.write_l0_csv(H.L0Report([H.L0Point(2, 1234567.0)], 2, 3), tmp_path / "z.csv")
    assert (tmp_path / "z.csv").read_text().splitlines()[1:] == ["2,1.23457e+06", "# best_l0=2 heuristic_l0=3"]


@pytest.mark.gpu
@needs_ref
def test_gpu_harness_matches_reference(gpu):
    from oracle import Reference

    import paper_1904_12754_b200 as P
    from paper_1904_12754_b200 import harness as H

    a = grid(16)
    u = np.linspace(0.2, 1.7, a.n)
    ref = Reference().chain(a)
    with P.Context(P.SparseMatrix(a.n, a.row_ptr, a.col, a.val), u) as ctx:
        prob = P.MlmcProblem(ctx, 37, 1.0)
        rep = H.bench_levels(prob, 0, 6, 20000, 5)
        rows, slopes = ref.bench_levels(u, 37, 1.0, 0, 6, 20000, 5)
        for r, e in zip(rep.rows, rows):
            assert r.level == int(e[0]) and r.dt == e[1] and r.cost_per_sample == e[4]
            assert r.mean == pytest.approx(e[2], rel=1e-12, abs=1e-16)
            assert r.variance == pytest.approx(e[3], rel=1e-9, abs=1e-18)
        assert [rep.slope_mean, rep.slope_variance, rep.slope_cost_tail] == pytest.approx(list(slopes), rel=1e-9)

        l0 = H.bench_l0(prob, 0, 3, 1e-2, 9)
        costs, best, heur = ref.bench_l0(u, 37, 1.0, 0, 3, 1e-2, 9)
        assert [p.cost for p in l0.points] == list(costs)
        assert (l0.best_l0, l0.heuristic_l0) == (best, heur)

        eps = [4e-2, 2e-2, 1e-2]
        cx = H.bench_complexity(prob, eps, 3)
        ml, mc, sl = ref.bench_complexity(u, 37, 1.0, eps, 3)
        assert [p.cost for p in cx.mlmc] == list(ml) and [p.cost for p in cx.mc] == list(mc)
        assert [cx.slope_mlmc, cx.slope_mc] == pytest.approx(list(sl), rel=1e-12)
