"""Paper-figure harness (harness.hpp / harness.cpp:41-177) over the GPU estimator.

Same names, arguments, report fields, fits and CSV layout as the reference:

    fit_log2_slope / fit_loglog_slope   harness.cpp:41-59   least-squares slopes
    bench_levels                        harness.cpp:61-94   level decay of m_l, V_l, cost (Fig. 1)
    bench_complexity                    harness.cpp:96-125  MLMC vs MC cost against epsilon (Fig. 2)
    bench_l0                            harness.cpp:127-144 total cost against the base level
    write_*_csv                         harness.cpp:146-177

The statistics come from the GPU path; bench_levels runs all its levels in ONE batched pass
(run_level_batch) with the same per-level results as the reference's level-by-level loop.
The fits are the reference's arithmetic in the same order, so equal inputs give equal slopes.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import api as A


def _ls_slope(x, y) -> float:  # harness.cpp:16-32
    n = len(x)
    if n < 2:
        raise A.InvalidArgument("slope fit needs at least two points")
    mx = 0.0
    my = 0.0
    for i in range(n):
        mx += x[i]
        my += y[i]
    mx /= n
    my /= n
    num = 0.0
    den = 0.0
    for i in range(n):
        num += (x[i] - mx) * (y[i] - my)
        den += (x[i] - mx) * (x[i] - mx)
    return num / den


def fit_log2_slope(x, y) -> float:
    """Slope of log2(y) against x over the points with y > 0 (harness.cpp:41-49)."""
    xs, ys = [], []
    for a, b in zip(x, y):
        if b > 0.0:
            xs.append(float(a))
            ys.append(math.log2(b))
    return _ls_slope(xs, ys)


def fit_loglog_slope(x, y) -> float:
    """Slope of log(y) against log(x) over the points with x, y > 0 (harness.cpp:51-59)."""
    xs, ys = [], []
    for a, b in zip(x, y):
        if a > 0.0 and b > 0.0:
            xs.append(math.log(a))
            ys.append(math.log(b))
    return _ls_slope(xs, ys)


@dataclass
class LevelDecayRow:
    level: int = 0
    dt: float = 0.0
    mean: float = 0.0
    variance: float = 0.0
    cost_per_sample: float = 0.0


@dataclass
class LevelDecayReport:
    rows: list = field(default_factory=list)
    slope_mean: float = 0.0
    slope_variance: float = 0.0
    slope_cost_tail: float = 0.0


def bench_levels(problem: A.MlmcProblem, l0: int, count: int, samples: int, seed: int,
                 threads: int = 0) -> LevelDecayReport:
    """Coupled levels l0+1 .. l0+count, `samples` each from index 0 (harness.cpp:61-94)."""
    if count < 2:
        raise A.InvalidArgument("need at least two coupled levels")
    levels = np.arange(l0 + 1, l0 + count + 1)
    mode = A.SampleMode(problem.mode)
    lane = {A.SampleMode.entry: A.LANE_ENTRY, A.SampleMode.forward: A.LANE_FORWARD,
            A.SampleMode.fem: A.LANE_FEM}[mode]
    st = problem.ctx.run_level_batch(problem.beta, problem.entry, levels, 0, 0, samples, seed, lane=lane)
    rep = LevelDecayReport()
    for k, lv in enumerate(levels):
        s = A.LevelStats(int(lv), float(st[k]["sum"]), float(st[k]["sum_sq"]), int(st[k]["samples"]),
                         int(st[k]["cost"]))
        rep.rows.append(LevelDecayRow(int(lv), problem.beta / float(1 << int(lv)), s.mean(), s.variance(),
                                      s.unit_cost()))
    ls = [float(r.level) for r in rep.rows]
    rep.slope_mean = fit_log2_slope(ls, [abs(r.mean) for r in rep.rows])
    rep.slope_variance = fit_log2_slope(ls, [r.variance for r in rep.rows])
    half = len(rep.rows) // 2
    rep.slope_cost_tail = fit_log2_slope(ls[half:], [r.cost_per_sample for r in rep.rows][half:])
    return rep


@dataclass
class ComplexityPoint:
    epsilon: float = 0.0
    cost: float = 0.0
    wall_seconds: float = 0.0


@dataclass
class ComplexityReport:
    mlmc: list = field(default_factory=list)
    mc: list = field(default_factory=list)
    slope_mlmc: float = 0.0
    slope_mc: float = 0.0


def bench_complexity(problem: A.MlmcProblem, epsilons, seed: int, threads: int = 0) -> ComplexityReport:
    """mlmc_driver and mc_auto at each epsilon; log-log cost slopes (harness.cpp:96-125)."""
    if A.SampleMode(problem.mode) != A.SampleMode.entry:
        raise A.InvalidArgument("complexity sweep runs on single-entry problems")
    rep = ComplexityReport()
    for eps in epsilons:
        t0 = time.perf_counter()
        ml = A.mlmc_driver(problem, A.MlmcOptions(epsilon=eps, seed=seed, threads=threads))
        rep.mlmc.append(ComplexityPoint(eps, float(ml.total_cost), time.perf_counter() - t0))
        t0 = time.perf_counter()
        mc = A.mc_auto(problem.ctx, problem.entry, problem.beta, eps, seed, threads)
        rep.mc.append(ComplexityPoint(eps, float(mc.wall_cost), time.perf_counter() - t0))
    eps = [p.epsilon for p in rep.mlmc]
    rep.slope_mlmc = fit_loglog_slope(eps, [p.cost for p in rep.mlmc])
    rep.slope_mc = fit_loglog_slope(eps, [p.cost for p in rep.mc])
    return rep


@dataclass
class L0Point:
    l0: int = 0
    cost: float = 0.0


@dataclass
class L0Report:
    points: list = field(default_factory=list)
    best_l0: int = 0
    heuristic_l0: int = 0


def bench_l0(problem: A.MlmcProblem, l0_min: int, l0_max: int, epsilon: float, seed: int,
             threads: int = 0) -> L0Report:
    """mlmc_driver total cost for each forced base level (harness.cpp:127-144)."""
    if l0_min < 0 or l0_max < l0_min:
        raise A.InvalidArgument("bad l0 range")
    rep = L0Report(heuristic_l0=A.initial_level(problem.beta, problem.ctx.d_max))
    best = math.inf
    for l0 in range(l0_min, l0_max + 1):
        r = A.mlmc_driver(problem, A.MlmcOptions(epsilon=epsilon, seed=seed, threads=threads, l0_override=l0))
        rep.points.append(L0Point(l0, float(r.total_cost)))
        if r.total_cost < best:
            best = r.total_cost
            rep.best_l0 = l0
    return rep


def _g(x) -> str:  # std::ostream's default formatting of a double (%g, 6 significant digits)
    return f"{x:g}"


def write_level_decay_csv(report: LevelDecayReport, path) -> None:
    with open(path, "w") as f:
        f.write("level,dt,mean,variance,cost_per_sample\n")
        for r in report.rows:
            f.write(f"{r.level},{_g(r.dt)},{_g(r.mean)},{_g(r.variance)},{_g(r.cost_per_sample)}\n")
        f.write(f"# slope_mean={_g(report.slope_mean)} slope_variance={_g(report.slope_variance)} "
                f"slope_cost_tail={_g(report.slope_cost_tail)}\n")


def write_complexity_csv(report: ComplexityReport, path) -> None:
    with open(path, "w") as f:
        f.write("method,epsilon,cost,wall_seconds\n")
        for p in report.mlmc:
            f.write(f"mlmc,{_g(p.epsilon)},{_g(p.cost)},{_g(p.wall_seconds)}\n")
        for p in report.mc:
            f.write(f"mc,{_g(p.epsilon)},{_g(p.cost)},{_g(p.wall_seconds)}\n")
        f.write(f"# slope_mlmc={_g(report.slope_mlmc)} slope_mc={_g(report.slope_mc)}\n")


def write_l0_csv(report: L0Report, path) -> None:
    with open(path, "w") as f:
        f.write("l0,total_cost\n")
        for p in report.points:
            f.write(f"{p.l0},{_g(p.cost)}\n")
        f.write(f"# best_l0={report.best_l0} heuristic_l0={report.heuristic_l0}\n")
