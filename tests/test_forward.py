"""Forward mode (SampleMode::forward): the estimator of sum(e^{tA} u) from paths on A^T whose
start state is drawn with probability u_i / sum(u) (make_initial_distribution /
sample_initial, paths.cpp:12-36; forward_single / forward_coupled, paths.cpp:144-181; lane 1,
mlmc.cpp:86, 94-96, 112-120).  This is total communicability (communicability.cpp:10-21).

CPU tests pin the oracle's restatement to golden_forward.json (produced by the reference,
tests/golden/make_golden.py forward()); GPU tests hold the CUDA path to the same bar as entry
mode: integer work bit-exact, per-sample values <= 4 ulp, run_level sums 1e-12,
drivers on the reference's decision sequence, plus the reference's own forward KATs
(test_paths.cpp:251-323).
"""
import math

import numpy as np
import pytest

from oracle import CSR

NAMES = ["k2", "signed3", "absorb3", "grid8", "smallw150", "pref300"]
ULP_TOL = 4


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


def csr_t(m) -> CSR:
    c = m["csr_t"]
    return CSR(c["n"], np.array(c["row_ptr"], np.int64), np.array(c["col"], np.int64), unhex(c["val"]))


def ulp_diff(a, b):
    ia = np.asarray(a, np.float64).view(np.int64)
    ib = np.asarray(b, np.float64).view(np.int64)
    ia = np.where(ia < 0, np.int64(-(2 ** 63)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2 ** 63)) - ib, ib)
    return np.abs(ia - ib)


# ------------------------------------------------------------------ CPU: oracle vs reference
@pytest.mark.parametrize("name", NAMES)
def test_oracle_forward_samples_and_run_level(golden_forward, oracle_lib, name):
    m = golden_forward["matrices"][name]
    ch = oracle_lib.chain(csr_t(m))
    u, beta = unhex(m["u"]), float.fromhex(m["beta"])
    for s in m["samples"]:
        got = ch.forward_samples(u, beta, s["level"], s["base"], s["seed"], np.array(s["idx"], np.uint64))
        assert np.array_equal(got["fine"], unhex(s["fine"]))
        assert np.array_equal(got["coarse"], unhex(s["coarse"]))
        assert np.array_equal(got["cost"], np.array(s["cost"], np.uint64))
    for r in m["run_level"]:
        got = ch.forward_run_level(u, beta, r["level"], r["base"], r["first"], r["count"], r["seed"], threads=3)
        assert got["sum"] == float.fromhex(r["sum"]) and got["sum_sq"] == float.fromhex(r["sum_sq"])
        assert got["samples"] == r["samples"] and got["cost"] == r["cost"]


@pytest.mark.parametrize("name", ["smallw150", "grid16"])
def test_oracle_forward_driver(golden_forward, oracle_lib, name):
    d = golden_forward["drivers"][name]
    ch = oracle_lib.chain(csr_t(d))
    res = ch.forward_driver(unhex(d["u"]), float.fromhex(d["beta"]), seeds=d["seeds"], epsilon=d["epsilon"], threads=4)
    for got, exp in zip(res, d["results"]):
        assert got["estimate"] == float.fromhex(exp["estimate"])
        assert got["statistical_error"] == float.fromhex(exp["statistical_error"])
        assert (got["l0"], got["L"], got["total_cost"], got["converged"]) == (exp["l0"], exp["L"], exp["total_cost"],
                                                                            exp["converged"])
        assert [int(x) for x in got["levels"]["samples"]] == [x["samples"] for x in exp["levels"]]
        # and the estimate is an estimate of sum(e^{tA}u)
        assert abs(got["estimate"] - float.fromhex(d["exact_sum"])) < 3 * got["statistical_error"] + d["epsilon"]


def test_oracle_forward_errors(oracle_lib):
    """make_initial_distribution's errors (paths.cpp:17-22; test_paths.cpp:288-293)."""
    from oracle import InvalidArgument

    ch = oracle_lib.chain(CSR.from_dense([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(InvalidArgument, match="nonnegative"):
        ch.forward_samples(np.array([1.0, -0.5]), 1.0, 2, 1, 1, np.arange(2, dtype=np.uint64))
    with pytest.raises(InvalidArgument, match=r"sum\(u\) > 0"):
        ch.forward_run_level(np.array([0.0, 0.0]), 1.0, 2, 1, 0, 10, 1)


@pytest.mark.parametrize("name", NAMES + ["grid16"])
def test_product_transpose_matches_reference(golden_forward, name):
    """SparseMatrix.transposed (host, product side) gives the reference's A^T CSR bit for bit."""
    import paper_1904_12754_b200 as P

    m = golden_forward["matrices"].get(name) or golden_forward["drivers"][name]
    t = csr_t(m)
    a = P.SparseMatrix(t.n, t.row_ptr, t.col, t.val).transposed()  # (A^T)^T = A
    back = a.transposed()
    assert np.array_equal(back.row_ptr, t.row_ptr) and np.array_equal(back.col, t.col)
    assert np.array_equal(back.val, t.val)


# ------------------------------------------------------------------ GPU
def _ctx(P, m, sampler=None):
    t = csr_t(m)
    a = P.SparseMatrix(t.n, t.row_ptr, t.col, t.val)
    return P.Context(a, unhex(m["u"]), device=0, **({} if sampler is None else {"sampler": sampler}))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_forward_per_sample_golden(gpu, golden_forward, name):
    import paper_1904_12754_b200 as P

    m = golden_forward["matrices"][name]
    beta = float.fromhex(m["beta"])
    with _ctx(P, m) as ctx:
        for s in m["samples"]:
            idx = np.array(s["idx"], np.uint64)
            got = ctx.sample_debug(beta, 0, s["level"], s["base"], s["seed"], idx, lane=P.LANE_FORWARD)
            assert np.array_equal(got["cost"], np.array(s["cost"], np.uint64)), (name, s["level"], s["base"])
            assert ulp_diff(got["fine"], unhex(s["fine"])).max() <= ULP_TOL
            assert ulp_diff(got["coarse"], unhex(s["coarse"])).max() <= ULP_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_forward_run_level_golden(gpu, golden_forward, name):
    import paper_1904_12754_b200 as P

    m = golden_forward["matrices"][name]
    beta = float.fromhex(m["beta"])
    with _ctx(P, m) as ctx:
        prob = P.MlmcProblem(ctx, 0, beta, P.SampleMode.forward)
        for r in m["run_level"]:
            got = P.run_level(prob, r["level"], bool(r["base"]), r["first"], r["count"], r["seed"])
            assert got.samples == r["samples"] and got.cost == r["cost"]
            assert got.sum == pytest.approx(float.fromhex(r["sum"]), rel=1e-12, abs=1e-13)
            assert got.sum_sq == pytest.approx(float.fromhex(r["sum_sq"]), rel=1e-12, abs=1e-13)


@pytest.mark.gpu
def test_gpu_forward_per_sample_oracle_random(gpu, golden_forward, oracle_lib):
    """2,000 random (level, seed, sample) draws on smallw150^T and pref300^T against the oracle:
    start state, path, cost, jumps, end state exact; values <= 4 ulp."""
    import paper_1904_12754_b200 as P

    rng = np.random.default_rng(5)
    for name in ["smallw150", "pref300"]:
        m = golden_forward["matrices"][name]
        u, beta = unhex(m["u"]), float.fromhex(m["beta"])
        och = oracle_lib.chain(csr_t(m))
        with _ctx(P, m) as ctx:
            for level in range(0, 6):
                for base in ([1] if level == 0 else [1, 0]):
                    idx = rng.integers(0, 2 ** 40, 200).astype(np.uint64)
                    seed = int(rng.integers(0, 2 ** 63))
                    got = ctx.sample_debug(beta, 0, level, base, seed, idx, lane=P.LANE_FORWARD)
                    exp = och.samples(u, 0, beta, level, base, seed, idx, lane=1)
                    assert np.array_equal(got["cost"], exp["cost"]) and np.array_equal(got["jumps"], exp["jumps"])
                    assert np.array_equal(got["end_state"], exp["end_state"])
                    assert ulp_diff(got["fine"], exp["fine"]).max() <= ULP_TOL
                    assert ulp_diff(got["coarse"], exp["coarse"]).max() <= ULP_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["smallw150", "grid16"])
def test_gpu_forward_driver_golden(gpu, golden_forward, name):
    """mlmc_driver in forward mode takes the reference's decision sequence per seed."""
    import paper_1904_12754_b200 as P

    d = golden_forward["drivers"][name]
    beta = float.fromhex(d["beta"])
    with _ctx(P, d) as ctx:
        res, lv = P.mlmc_driver_forward(ctx, beta, d["seeds"], P.MlmcOptions(epsilon=d["epsilon"]))
        for k, exp in enumerate(d["results"]):
            r = res[k]
            assert (int(r["l0"]), int(r["L"]), int(r["total_cost"]), bool(r["converged"])) == (
                exp["l0"], exp["L"], exp["total_cost"], exp["converged"])
            assert float(r["estimate"]) == pytest.approx(float.fromhex(exp["estimate"]), rel=1e-12)
            assert [int(x) for x in lv[k, : int(r["nlevels"])]["samples"]] == [x["samples"] for x in exp["levels"]]
        # the single-run form (the reference's own call, seeded by options.seed)
        one = P.mlmc_driver(P.MlmcProblem(ctx, 0, beta, P.SampleMode.forward),
                            P.MlmcOptions(epsilon=d["epsilon"], seed=d["seeds"][0]))
        assert one.estimate == pytest.approx(float.fromhex(d["results"][0]["estimate"]), rel=1e-12)
        assert one.total_cost == d["results"][0]["total_cost"]


@pytest.mark.gpu
def test_gpu_forward_k2_exactly_2e(gpu):
    """test_paths.cpp:275-286: on K2 every forward path has value 2e."""
    import paper_1904_12754_b200 as P

    k2 = P.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 0.0]])
    with P.Context(k2.transposed(), np.ones(2)) as ctx:
        got = ctx.sample_debug(1.0, 0, 2, 1, 11, np.arange(500, dtype=np.uint64), lane=P.LANE_FORWARD)
        assert np.allclose(got["fine"], 2.0 * math.e, rtol=1e-15, atol=0)
        st = P.run_level(P.MlmcProblem(ctx, 0, 1.0, P.SampleMode.forward), 6, True, 0, 10000, 3)
        assert st.sum / st.samples == pytest.approx(2.0 * math.e, rel=1e-13)


@pytest.mark.gpu
def test_gpu_forward_diagonal_mean(gpu):
    """test_paths.cpp:251-273: E = sum_i e^{beta d_i} on a diagonal matrix, within 4 SE."""
    import paper_1904_12754_b200 as P

    a = P.SparseMatrix.from_triplets(3, [0, 1, 2], [0, 1, 2], [0.3, -0.2, 1.1])
    with P.Context(a.transposed(), np.ones(3)) as ctx:
        st = P.run_level(P.MlmcProblem(ctx, 0, 1.0, P.SampleMode.forward), 2, True, 0, 200000, 10)
        mean = st.sum / st.samples
        se = math.sqrt((st.sum_sq / st.samples - mean * mean) / st.samples)
        assert abs(mean - (math.exp(0.3) + math.exp(-0.2) + math.exp(1.1))) < 4 * se


@pytest.mark.gpu
def test_gpu_forward_small_world_strang(gpu, golden_forward):
    """test_paths.cpp:295-323: forward mean on smallw(150)^T at 8 steps vs the transpose Strang
    product sum_j u_j (S_{A^T} 1)_j, within 4 SE."""
    import paper_1904_12754_b200 as P
    from oracle import Reference, have_reference

    d = golden_forward["drivers"]["smallw150"]
    u = unhex(d["u"])
    with _ctx(P, d) as ctx:
        beta = 1.0 / ctx.d_max
        st = P.run_level(P.MlmcProblem(ctx, 0, beta, P.SampleMode.forward), 3, True, 0, 400000, 14)
        mean = st.sum / st.samples
        se = math.sqrt((st.sum_sq / st.samples - mean * mean) / st.samples)
    if have_reference():
        ref = Reference().chain(csr_t(d))
        expect = float(np.dot(u, ref.strang_reference(np.ones(u.size), beta, 8)))
        assert abs(mean - expect) < 4 * se
    else:  # the Strang bias at 8 steps is far below 4 SE here; the exact sum stands in
        assert abs(mean - float.fromhex(d["exact_sum"])) < 4 * se + 1e-3 * abs(mean)


@pytest.mark.gpu
def test_gpu_forward_errors(gpu):
    """Reference errors: negative u / zero sum (paths.cpp:17-22), unknown lane -> ENOTIMPL, fem
    without a load -> invalid_argument (mlmc.cpp:156-157),
    entry is not validated in forward mode (mlmc.cpp:154)."""
    import paper_1904_12754_b200 as P

    k2t = P.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 0.0]]).transposed()
    with P.Context(k2t, np.array([1.0, -0.5])) as ctx:
        prob = P.MlmcProblem(ctx, 0, 1.0, P.SampleMode.forward)
        with pytest.raises(P.InvalidArgument, match="nonnegative"):
            P.run_level(prob, 2, True, 0, 10, 1)
        with pytest.raises(P.InvalidArgument, match="nonnegative"):
            P.mlmc_driver(prob, P.MlmcOptions(epsilon=0.1))
        ctx.set_vector(np.zeros(2))
        with pytest.raises(P.InvalidArgument, match=r"sum\(u\) > 0"):
            P.run_level(prob, 2, True, 0, 10, 1)
        ctx.set_vector(np.ones(2))  # set_vector rebuilds the start distribution
        st = P.run_level(P.MlmcProblem(ctx, 12345, 1.0, P.SampleMode.forward), 2, True, 0, 100, 1)
        assert st.sum / st.samples == pytest.approx(2.0 * math.e, rel=1e-13)
        with pytest.raises(P.InvalidArgument, match="load length"):  # fem without a load
            P.run_level(P.MlmcProblem(ctx, 0, 1.0, P.SampleMode.fem), 2, True, 0, 10, 1)
        with pytest.raises(P.NotImplementedMode):
            ctx.run_level_batch(1.0, 0, 2, 1, 0, 10, 1, lane=3)


@pytest.mark.gpu
def test_gpu_forward_event_sampler_statistical(gpu, golden_forward):
    """The event-driven sampler in forward mode: same law, so its level means agree with the
    reference-order sampler's within combined SE (levels 0..4 on smallw150^T)."""
    import paper_1904_12754_b200 as P

    d = golden_forward["drivers"]["smallw150"]
    beta = float.fromhex(d["beta"])
    stats = {}
    for sampler in ("reference", "event"):
        with _ctx(P, d, sampler=sampler) as ctx:
            stats[sampler] = [P.run_level(P.MlmcProblem(ctx, 0, beta, P.SampleMode.forward), lvl, lvl == 0, 0,
                                          200000, 77 + lvl) for lvl in range(5)]
    for a, b in zip(stats["reference"], stats["event"]):
        se = math.sqrt(a.variance() / a.samples + b.variance() / b.samples)
        assert abs(a.mean() - b.mean()) < 4 * se + 1e-12


@pytest.mark.gpu
def test_gpu_total_and_node_communicability(gpu, golden_forward, oracle_lib):
    """communicability.cpp:10-35 on pref(300, 3, 7) (test_mc.cpp:125-143 analogue): the forward
    driver's 1^T e^{beta A} 1 and the entry driver's (e^{beta A} 1)_node against dense_expmv."""
    import paper_1904_12754_b200 as P

    t = csr_t(golden_forward["matrices"]["pref300"])
    a = P.SparseMatrix(t.n, t.row_ptr, t.col, t.val).transposed()
    beta = 1.0 / oracle_lib.chain(t).d_max  # spectral_scale(dec of A^T), chain.cpp:98-102
    exact = oracle_lib.dense_expmv(CSR(a.n, a.row_ptr, a.col, a.val), np.ones(a.n), beta)
    eps = 0.5
    tc = P.total_communicability(a, options=P.MlmcOptions(epsilon=eps, seed=4))
    assert tc.converged
    assert abs(tc.estimate - exact.sum()) < 3 * tc.statistical_error + eps
    for node in (0, 150):
        nc = P.node_communicability(a, node, beta, P.MlmcOptions(epsilon=1e-2, seed=node))
        assert nc.converged and abs(nc.estimate - exact[node]) < 3 * nc.statistical_error + 1e-2
    with pytest.raises(P.DomainError):
        P.total_communicability(P.SparseMatrix.from_dense(np.zeros((2, 2))))
