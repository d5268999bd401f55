"""fem mode (SampleMode::fem, lane 2): the inhomogeneous lumped-mass system M u' = -K u + F
solved at one node by MLMC on the chain of -M^{-1}K, with the Duhamel integral of the load
g = M^{-1}F carried along every path by composite-Simpson weights (fem_single / fem_coupled,
paths.cpp:183-245; run_level_ex mlmc.cpp:66-148; the driver's quadrature bound mlmc.cpp:177,
226-241; solve_convdiff_point fem.cpp:51-73).

CPU tests pin the oracle restatement to golden_fem.json (made by the reference,
tests/golden/make_golden.py fem()); GPU tests hold the CUDA path to the parity rule of
DESIGN.md §5 and re-check the reference's own fem KATs (test_paths.cpp:325-392,
test_apps.cpp:154-240).

Tolerances: draws, jumps, costs, terminal states and the driver's decision sequence are exact;
exponentials are CUDA's (<= 1 ulp from glibc), so the per-node terms carry ~1 ulp each and the
load integrals are compared to 1e-14 relative of their magnitude, the sample value
u[end](eta_f - eta_c) + (integ_f - integ_c) to 1e-14 of |u eta| + |integ| (it is a difference
of nearly equal quantities).
"""
import math

import numpy as np
import pytest

from oracle import CSR

SYSTEMS = ["toy3", "scalar", "smallw60"]


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


def system(m):
    c = m["csr"]
    a = CSR(c["n"], np.array(c["row_ptr"], np.int64), np.array(c["col"], np.int64), unhex(c["val"]))
    md = unhex(m["mass_diag"])
    return a, md, unhex(m["load"]), unhex(m["u0"]), float.fromhex(m["t"])


def scaled(a: CSR, md):
    """decompose_scaled's per-entry product scale_i * a_ij (chain.cpp:37) applied to the CSR."""
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    return CSR(a.n, a.row_ptr, a.col, (-1.0 / md)[rows] * a.val)


def ulp_diff(a, b):
    ia = np.asarray(a, np.float64).view(np.int64)
    ib = np.asarray(b, np.float64).view(np.int64)
    ia = np.where(ia < 0, np.int64(-(2 ** 63)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2 ** 63)) - ib, ib)
    return np.abs(ia - ib)


# ------------------------------------------------------------------ CPU: oracle vs reference
@pytest.mark.parametrize("name", SYSTEMS)
def test_oracle_fem_matches_reference(golden_fem, oracle_lib, name):
    m = golden_fem["systems"][name]
    a, md, load, u0, t = system(m)
    g = load / md
    ch = oracle_lib.chain(scaled(a, md))
    assert np.array_equal(ch.decomposition()["d"], unhex(m["d"]))
    for s in m["samples"]:
        got = ch.fem_samples(u0, g, s["entry"], t, s["level"], s["base"], s["seed"], np.array(s["idx"], np.uint64))
        for k in ("value", "eta_f", "eta_c", "integ_f", "integ_c"):
            assert np.array_equal(got[k], unhex(s[k])), (name, k, s["level"], s["base"])
        assert np.array_equal(got["cost"], np.array(s["cost"], np.uint64))
        assert np.array_equal(got["end_state"], np.array(s["end_state"]))
    for r in m["run_level"]:
        got = ch.fem_run_level(u0, g, r["entry"], t, r["level"], r["base"], r["first"], r["count"], r["seed"],
                               threads=3)
        assert got["sum"] == float.fromhex(r["sum"]) and got["sum_sq"] == float.fromhex(r["sum_sq"])
        assert got["samples"] == r["samples"] and got["cost"] == r["cost"]
    rows = [d["node"] for d in m["drivers"]]
    res = ch.fem_driver_rows(u0, g, t, rows, [d["seed"] for d in m["drivers"]], epsilon=m["drivers"][0]["epsilon"],
                             threads=4)
    for got, exp in zip(res, m["drivers"]):
        assert got["estimate"] == float.fromhex(exp["estimate"])
        assert got["quadrature_bound"] == float.fromhex(exp["quadrature_bound"])
        assert (got["l0"], got["L"], got["total_cost"], got["converged"]) == (exp["l0"], exp["L"], exp["total_cost"],
                                                                            exp["converged"])


def test_oracle_fem_errors(oracle_lib):
    from oracle import InvalidArgument

    ch = oracle_lib.chain(CSR.from_dense([[-1.0, 0.5], [0.5, -1.0]]))
    u, g = np.ones(2), np.ones(2)
    with pytest.raises(InvalidArgument, match="divisible by 4"):
        ch.fem_samples(u, g, 0, 1.0, 1, 0, 1, np.arange(2, dtype=np.uint64))
    with pytest.raises(InvalidArgument, match="divisible by 4"):
        ch.fem_run_level(u, g, 0, 1.0, 1, 0, 0, 10, 1)
    assert ch.fem_run_level(u, g, 0, 1.0, 1, 0, 0, 0, 1)["samples"] == 0  # no samples, no error


# ------------------------------------------------------------------ GPU
def _ctx(P, m, zero_load=False):
    a, md, load, u0, t = system(m)
    sysm = P.FemSystem(md, P.SparseMatrix(a.n, a.row_ptr, a.col, a.val), np.zeros(a.n) if zero_load else load, u0)
    return P.fem_context(sysm), t


def _close(got, exp, scale, rel=1e-14):
    return np.all(np.abs(got - exp) <= rel * scale + 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SYSTEMS)
def test_gpu_fem_tables_and_per_sample_golden(gpu, golden_fem, name):
    import paper_1904_12754_b200 as P

    m = golden_fem["systems"][name]
    ctx, t = _ctx(P, m)
    with ctx:
        assert np.array_equal(ctx.decomposition()["d"], unhex(m["d"]))
        u0 = unhex(m["u0"])
        gmax = np.abs(unhex(m["load"]) / unhex(m["mass_diag"])).max()
        for s in m["samples"]:
            idx = np.array(s["idx"], np.uint64)
            got = ctx.sample_records(t, s["entry"], s["level"], s["base"], s["seed"], idx, lane=P.LANE_FEM)
            assert np.array_equal(got["cost"], np.array(s["cost"], np.uint64)), (name, s["level"], s["base"])
            ef, ec, i_f, i_c = (unhex(s[k]) for k in ("eta_f", "eta_c", "integ_f", "integ_c"))
            # the size of the quadrature sums' terms: t max|g| e^{expo}
            iscale = t * gmax * np.maximum(np.maximum(np.abs(ef), np.abs(ec)), 1.0)
            if not s["base"]:
                assert np.array_equal(got["end_state"], np.array(s["end_state"]))
                assert ulp_diff(got["eta_fine"], ef).max() <= 4 and ulp_diff(got["eta_coarse"], ec).max() <= 4
                assert _close(got["integ_fine"], i_f, iscale) and _close(got["integ_coarse"], i_c, iscale)
                scale = np.abs(u0[got["end_state"]] * ef) + iscale
            else:  # fem_single reports the value only
                scale = np.abs(unhex(s["value"])) + t * gmax * np.maximum(np.abs(got["eta_fine"]), 1.0)
            assert _close(got["value"], unhex(s["value"]), scale), (name, s["level"], s["base"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", SYSTEMS)
def test_gpu_fem_run_level_golden(gpu, golden_fem, name):
    import paper_1904_12754_b200 as P

    m = golden_fem["systems"][name]
    ctx, t = _ctx(P, m)
    with ctx:
        for r in m["run_level"]:
            got = P.run_level(P.MlmcProblem(ctx, r["entry"], t, P.SampleMode.fem), r["level"], bool(r["base"]),
                              r["first"], r["count"], r["seed"])
            assert got.samples == r["samples"] and got.cost == r["cost"]
            assert got.sum == pytest.approx(float.fromhex(r["sum"]), rel=1e-11, abs=1e-12)
            assert got.sum_sq == pytest.approx(float.fromhex(r["sum_sq"]), rel=1e-11, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SYSTEMS)
def test_gpu_solve_convdiff_point_golden(gpu, golden_fem, name):
    """solve_convdiff_point through the GPU: the reference's decision sequence (l0 >= 1, L,
    samples per level, cost) and its estimate / quadrature bound."""
    import paper_1904_12754_b200 as P

    m = golden_fem["systems"][name]
    a, md, load, u0, t = system(m)
    sysm = P.FemSystem(md, P.SparseMatrix(a.n, a.row_ptr, a.col, a.val), load, u0)
    for d in m["drivers"]:
        r = P.solve_convdiff_point(sysm, d["node"], t, P.MlmcOptions(epsilon=d["epsilon"], seed=d["seed"]))
        assert (r.l0, r.L, r.total_cost, r.converged) == (d["l0"], d["L"], d["total_cost"], d["converged"])
        assert [lv.samples for lv in r.levels] == [x["samples"] for x in d["levels"]]
        assert r.estimate == pytest.approx(float.fromhex(d["estimate"]), rel=1e-11, abs=1e-13)
        assert r.quadrature_bound == pytest.approx(float.fromhex(d["quadrature_bound"]), rel=1e-8, abs=1e-15)
    # the batched fem driver takes the same sequences
    with P.fem_context(sysm) as ctx:
        rows = [d["node"] for d in m["drivers"]]
        res, _ = P.mlmc_driver_fem(ctx, t, rows, [d["seed"] for d in m["drivers"]],
                                   P.MlmcOptions(epsilon=m["drivers"][0]["epsilon"]))
        for k, d in enumerate(m["drivers"]):
            assert int(res[k]["total_cost"]) == d["total_cost"] and int(res[k]["L"]) == d["L"]


@pytest.mark.gpu
def test_gpu_fem_zero_load_is_the_coupled_sampler(gpu, oracle_lib):
    """test_paths.cpp:325-358: with zero load the fem coupled sample is the coupled sample on
    the same stream (integrals exactly 0, eta * u[end] equal, same cost: quadrature consumes no
    draws).  The reference test feeds both samplers one stream; here the fem lane's stream
    (lane 2) drives the oracle's plain coupled sampler."""
    import paper_1904_12754_b200 as P

    m_rng = np.random.default_rng(0)
    n = 60
    # a signed random sparse matrix with unit mass
    trips = [(i, i, -2.0) for i in range(n)] + [(i, (i + k) % n, float(m_rng.choice([-0.5, 0.7])))
                                                 for i in range(n) for k in (1, 7)]
    a = P.SparseMatrix.from_triplets(n, *zip(*trips))
    u = 1.0 + 0.01 * np.arange(n)
    with P.Context(a, u, load=np.zeros(n)) as ctx:
        beta = 1.0 / ctx.d_max if ctx.d_max > 0 else 0.3
        idx = np.arange(300, dtype=np.uint64)
        fem = ctx.sample_records(beta, 0, 3, 0, 15, idx, lane=P.LANE_FEM)
    ref = oracle_lib.chain(CSR(a.n, a.row_ptr, a.col, a.val)).samples(u, 0, beta, 3, 0, 15, idx, lane=2)
    assert np.all(fem["integ_fine"] == 0.0) and np.all(fem["integ_coarse"] == 0.0)
    assert np.array_equal(fem["cost"], ref["cost"]) and np.array_equal(fem["end_state"], ref["end_state"])
    ue = u[fem["end_state"]]
    assert ulp_diff(fem["eta_fine"] * ue, ref["fine"]).max() <= 4
    assert ulp_diff(fem["eta_coarse"] * ue, ref["coarse"]).max() <= 4


@pytest.mark.gpu
def test_gpu_fem_scalar_simpson_exact(gpu):
    """test_paths.cpp:360-392: n = 1, a = -1.3: the fem_single value is u0 e^{beta a} plus the
    Simpson sum of e^{s a} g, and within the Simpson bound of the closed form."""
    import paper_1904_12754_b200 as P

    aval, g, u0, beta, steps = -1.3, 0.7, 2.0, 1.0, 16
    with P.Context(P.SparseMatrix.from_dense([[aval]]), [u0], load=[g]) as ctx:
        rec = ctx.sample_records(beta, 0, 4, 1, 16, np.zeros(1, np.uint64), lane=P.LANE_FEM)
    dt = beta / steps
    w = np.array([(1.0 if j in (0, steps) else (4.0 if j % 2 else 2.0)) * dt / 3.0 for j in range(steps + 1)])
    simpson = float(np.sum(w * np.exp(np.arange(steps + 1) * dt * aval) * g))
    assert rec["value"][0] == pytest.approx(u0 * math.exp(beta * aval) + simpson, rel=1e-14)
    exact = u0 * math.exp(beta * aval) + g / (-aval) * (1.0 - math.exp(beta * aval))
    assert abs(rec["value"][0] - exact) < 1.5 * beta / 180.0 * dt ** 4 * aval ** 4 * g


@pytest.mark.gpu
def test_gpu_convdiff_toy_vs_duhamel_oracle(gpu, golden_fem, oracle_lib):
    """test_apps.cpp:175-212: the three-node toy system against the dense Duhamel oracle
    x = e^{tA}u0 + int_0^t e^{sA} g ds (fine Simpson grid), A = -M^{-1}K, g = M^{-1}F."""
    import paper_1904_12754_b200 as P

    m = golden_fem["systems"]["toy3"]
    a, md, load, u0, t = system(m)
    gen = scaled(a, md)
    g = load / md
    x = oracle_lib.dense_expmv(gen, u0, t)
    panels = 512
    h = t / panels
    for j in range(panels + 1):
        wj = (1.0 if j in (0, panels) else (4.0 if j % 2 else 2.0)) / 3.0
        x = x + wj * h * oracle_lib.dense_expmv(gen, g, h * j)
    sysm = P.FemSystem(md, P.SparseMatrix(a.n, a.row_ptr, a.col, a.val), load, u0)
    for node in range(3):
        r = P.solve_convdiff_point(sysm, node, t, P.MlmcOptions(epsilon=5e-3, seed=31 + node))
        assert r.converged
        assert abs(r.estimate - x[node]) < 3 * r.statistical_error + r.bias_estimate + r.quadrature_bound + 1e-4


@pytest.mark.gpu
def test_gpu_fem_quadrature_reuses_path_draws_and_errors(gpu, golden_fem):
    """test_apps.cpp:214-240 (same per-level cost with and without the load) and the fem
    errors: coupled below level 2, missing load, bad row scale."""
    import paper_1904_12754_b200 as P

    m = golden_fem["systems"]["toy3"]
    with_load, t = _ctx(P, m)
    without, _ = _ctx(P, m, zero_load=True)
    with with_load, without:
        for level in (1, 2, 3, 4):
            a = P.run_level(P.MlmcProblem(with_load, 1, 0.9, P.SampleMode.fem), level, level == 1, 0, 4000, 8)
            b = P.run_level(P.MlmcProblem(without, 1, 0.9, P.SampleMode.fem), level, level == 1, 0, 4000, 8)
            assert a.cost == b.cost
        with pytest.raises(P.InvalidArgument, match="divisible by 4"):
            P.run_level(P.MlmcProblem(with_load, 0, t, P.SampleMode.fem), 1, False, 0, 10, 1)
        assert P.run_level(P.MlmcProblem(with_load, 0, t, P.SampleMode.fem), 1, False, 0, 0, 1).samples == 0
        with pytest.raises(P.OutOfRange):
            P.run_level(P.MlmcProblem(with_load, 3, t, P.SampleMode.fem), 2, True, 0, 10, 1)
    a, md, load, u0, t = system(m)
    sa = P.SparseMatrix(a.n, a.row_ptr, a.col, a.val)
    with P.Context(sa, u0, row_scale=-1.0 / md) as ctx:
        with pytest.raises(P.InvalidArgument, match="load length"):
            P.run_level(P.MlmcProblem(ctx, 0, t, P.SampleMode.fem), 2, True, 0, 10, 1)
        with pytest.raises(P.InvalidArgument, match="load length"):
            P.mlmc_driver(P.MlmcProblem(ctx, 0, t, P.SampleMode.fem), P.MlmcOptions(epsilon=0.1))
    with pytest.raises(P.InvalidArgument, match="row scale"):
        P.Context(sa, u0, row_scale=np.array([1.0, np.nan, 1.0]))
    sysm = P.FemSystem(md, sa, load, u0)
    with pytest.raises(P.InvalidArgument):
        P.solve_convdiff_point(sysm, 0, 0.0)
    with pytest.raises(P.OutOfRange):
        P.solve_convdiff_point(sysm, 3, 1.0)
