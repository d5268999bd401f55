"""The reference's statistical known-answer tests of the path sampler (test_paths.cpp:41-224),
run on the CUDA path with the same streams: evolve_interval's no-jump frequency and terminal
distribution (a level-0 single sample over one interval is evolve_interval), single_functional
against the Strang product, the coupled level-1 mean against the transition-matrix
enumeration, and telescoping.  Exact references are computed here with dense expm."""
import math

import numpy as np
import pytest
from scipy.linalg import expm

import paper_1904_12754_b200 as P

pytestmark = pytest.mark.gpu


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


def dense(a: P.SparseMatrix):
    m = np.zeros((a.n, a.n))
    for i in range(a.n):
        for k in range(int(a.row_ptr[i]), int(a.row_ptr[i + 1])):
            m[i, a.col[k]] = a.val[k]
    return m


def generator(a: P.SparseMatrix):
    """The chain's generator Q: q_ij = |a_ij| off the diagonal, q_ii = -rate_i."""
    m = np.abs(dense(a))
    np.fill_diagonal(m, 0.0)
    np.fill_diagonal(m, -m.sum(axis=1))
    return m


def strang(a: P.SparseMatrix, d, u, beta, steps):  # oracle.cpp:79-99
    dt = beta / steps
    t = np.diag(d) - dense(a)
    h = np.exp(0.5 * dt * d)
    e = expm(-dt * t)
    x = np.array(u, np.float64)
    for _ in range(steps):
        x = h * (e @ (h * x))
    return x


def test_evolve_interval_survival_and_terminal_distribution(gpu):
    # test_paths.cpp:41-49: a diagonal matrix never moves
    a = P.SparseMatrix.from_triplets(3, [0, 1], [0, 1], [1.0, -2.0])
    with P.Context(a, np.ones(3)) as ctx:
        r = ctx.sample_debug(5.0, 1, 0, 1, 1, np.zeros(1, np.uint64))
        assert r["end_state"][0] == 1 and r["jumps"][0] == 0 and r["fine"][0] > 0
    # test_paths.cpp:51-63: P(no jump in [0, 1]) = e^{-1} on K2
    k2 = P.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 0.0]])
    n = 1_000_000
    with P.Context(k2, np.ones(2)) as ctx:
        r = ctx.sample_debug(1.0, 0, 0, 1, 12, np.arange(n, dtype=np.uint64))
    p = math.exp(-1.0)
    assert abs((r["jumps"] == 0).mean() - p) < 3 * math.sqrt(p * (1 - p) / n)
    # test_paths.cpp:65-82: terminal state distribution = row 0 of e^{tQ}, t = 1.7
    a = P.SparseMatrix.from_triplets(3, [0, 0, 1, 1, 2], [1, 2, 0, 2, 0], [1.0, 0.5, 0.7, 0.2, 0.4])
    n = 400_000
    with P.Context(a, np.ones(3)) as ctx:
        r = ctx.sample_debug(1.7, 0, 0, 1, 13, np.arange(n, dtype=np.uint64))
    prow = expm(1.7 * generator(a))[0]
    hits = np.bincount(r["end_state"], minlength=3) / n
    assert np.all(np.abs(hits - prow) < 3 * np.sqrt(prow * (1 - prow) / n))


def test_single_functional_unbiased_for_strang(gpu, golden):
    """test_paths.cpp:113-133 on smallw(100, 2, 0.1, 5): level 4 (16 steps), seed 9."""
    m = golden["matrices"]["smallw100"]
    c = m["csr"]
    a = P.SparseMatrix(c["n"], np.array(c["row_ptr"]), np.array(c["col"]), unhex(c["val"]))
    u = np.ones(a.n)
    with P.Context(a, u) as ctx:
        beta = 1.0 / ctx.d_max
        st = P.run_level(P.MlmcProblem(ctx, 0, beta), 4, True, 0, 400_000, 9)
        d = ctx.decomposition()["d"]
    ref = strang(a, d, u, beta, 16)[0]
    mean = st.mean()
    assert abs(mean - ref) < 4 * math.sqrt(st.variance() / st.samples)


def test_coupled_level1_matches_enumeration(gpu):
    """test_paths.cpp:148-196: E[P_fine - P_coarse] and E[P_fine] on the two-state chain."""
    a = P.SparseMatrix.from_dense([[0.2, 1.0], [0.5, -0.3]])
    u = np.array([0.7, 1.3])
    beta, n = 0.8, 1_000_000
    dt = beta / 2
    with P.Context(a, u) as ctx:
        d = ctx.decomposition()["d"]
        r = ctx.sample_debug(beta, 0, 1, 0, 5, np.arange(n, dtype=np.uint64))
    pm = expm(dt * generator(a))
    expect = expect_f = 0.0
    for j in range(2):
        for k in range(2):
            fine = math.exp(dt * (0.5 * d[0] + d[j] + 0.5 * d[k]))
            coarse = math.exp(dt * (d[0] + d[k]))
            w = pm[0, j] * pm[j, k] * u[k]
            expect += w * (fine - coarse)
            expect_f += w * fine
    diff = r["fine"] - r["coarse"]
    assert abs(diff.mean() - expect) < 3 * diff.std() / math.sqrt(n)
    assert abs(r["fine"].mean() - expect_f) < 3 * r["fine"].std() / math.sqrt(n)


def test_telescoping(gpu, golden):
    """test_paths.cpp:198-224: the coarse mean at level l equals the fine mean at level l-1."""
    m = golden["matrices"]["smallw100"]
    c = m["csr"]
    a = P.SparseMatrix(c["n"], np.array(c["row_ptr"]), np.array(c["col"]), unhex(c["val"]))
    n, lv = 300_000, 4
    with P.Context(a, np.ones(a.n)) as ctx:
        beta = 1.0 / ctx.d_max
        cp = ctx.sample_debug(beta, 0, lv, 0, 6, np.arange(n, dtype=np.uint64))
        fn = ctx.sample_debug(beta, 0, lv - 1, 1, 7, np.arange(n, dtype=np.uint64))
    se = math.sqrt(cp["coarse"].var() / n + fn["fine"].var() / n)
    assert abs(cp["coarse"].mean() - fn["fine"].mean()) < 4 * se
