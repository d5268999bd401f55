"""Classical Monte Carlo (mc.hpp / mc.cpp:42-113) on the GPU sampler: mc_single_entry,
mc_forward_scalar, mc_auto.  Streams stream_for(seed, bit_width(steps), s, lane); one
Welford accumulator per 512-sample chunk, folded in sample order, chunks merged in order by
Chan's formula (parallel.hpp:80-104) -- the reference's statistics, not just its law.

CPU: the oracle's restatement against golden_mc.json (made by the reference).  GPU: samples,
steps and wall_cost exact; estimates 1e-13 and standard errors 1e-9 relative (per-sample
values differ from glibc's by <= 4 ulp through exp); mc_auto's pilot-driven step and sample
counts exact; the reference's KATs (test_mc.cpp:107-143) and error paths.
"""
import math

import numpy as np
import pytest

from oracle import CSR

NAMES = ["grid8", "smallw100", "pref300"]


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


def csr(m, key="csr"):
    c = m[key]
    return CSR(c["n"], np.array(c["row_ptr"], np.int64), np.array(c["col"], np.int64), unhex(c["val"]))


@pytest.mark.parametrize("name", NAMES)
def test_oracle_mc_matches_reference(golden_mc, oracle_lib, name):
    m = golden_mc["matrices"][name]
    u, beta = unhex(m["u"]), float.fromhex(m["beta"])
    ch, cht = oracle_lib.chain(csr(m)), oracle_lib.chain(csr(m, "csr_t"))
    for r in m["single"]:
        got = ch.mc_single_entry(u, r["entry"], beta, float.fromhex(r["dt"]), r["req_samples"], r["seed"])
        assert got["estimate"] == float.fromhex(r["estimate"]) and got["std_error"] == float.fromhex(r["std_error"])
        assert (got["samples"], got["steps"], got["wall_cost"]) == (r["samples"], r["steps"], r["wall_cost"])
    for r in m["forward"]:
        got = cht.mc_forward_scalar(u, beta, float.fromhex(r["dt"]), r["req_samples"], r["seed"])
        assert got["estimate"] == float.fromhex(r["estimate"]) and got["std_error"] == float.fromhex(r["std_error"])
        assert got["wall_cost"] == r["wall_cost"]


# ------------------------------------------------------------------ GPU
def _ctx(P, m, key="csr"):
    c = csr(m, key)
    return P.Context(P.SparseMatrix(c.n, c.row_ptr, c.col, c.val), unhex(m["u"]))


def _same(got, r):
    assert (got.samples, got.steps, got.wall_cost) == (r["samples"], r["steps"], r["wall_cost"])
    assert got.dt == float.fromhex(r["dt"])
    assert got.estimate == pytest.approx(float.fromhex(r["estimate"]), rel=1e-13, abs=1e-15)
    assert got.std_error == pytest.approx(float.fromhex(r["std_error"]), rel=1e-9, abs=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_mc_golden(gpu, golden_mc, name):
    import paper_1904_12754_b200 as P

    m = golden_mc["matrices"][name]
    beta = float.fromhex(m["beta"])
    with _ctx(P, m) as ctx:
        for r in m["single"]:
            _same(P.mc_single_entry(ctx, r["entry"], beta, float.fromhex(r["dt"]), r["req_samples"], r["seed"]), r)
        for r in m["auto"]:
            _same(P.mc_auto(ctx, r["entry"], beta, r["epsilon"], r["seed"]), r)
        # the batch form runs several entries in one pass with the same per-run results
        rs = m["single"][:2]
        dt = float.fromhex(rs[0]["dt"])
        got = P.mc_batch(ctx, [rs[0]["entry"], rs[0]["entry"]], [rs[0]["seed"], rs[0]["seed"] + 1],
                         rs[0]["req_samples"], beta, dt)
        _same(got[0], rs[0])
        assert got[1].estimate != got[0].estimate
    with _ctx(P, m, "csr_t") as ctx_t:
        for r in m["forward"]:
            _same(P.mc_forward_scalar(ctx_t, beta, float.fromhex(r["dt"]), r["req_samples"], r["seed"]), r)


@pytest.mark.gpu
def test_gpu_mc_kats_and_errors(gpu):
    """test_mc.cpp:107-123 (zero matrix: exactly n, std_error 0; K2: 2e) and the errors of
    mc_single_entry / checked_steps / mc_auto."""
    import paper_1904_12754_b200 as P

    z = P.SparseMatrix.from_triplets(5, [], [], [])
    with P.Context(z.transposed(), np.ones(5)) as ctx:
        r = P.mc_forward_scalar(ctx, 3.0, 1.5, 500, 1)
        assert r.estimate == 5.0 and r.std_error == 0.0 and r.steps == 2
    k2 = P.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 0.0]])
    with P.Context(k2.transposed(), np.ones(2)) as ctx:
        r = P.mc_forward_scalar(ctx, 1.0, 1.0 / 64.0, 5000, 2)
        assert r.estimate == pytest.approx(2.0 * math.e, rel=1e-13) and r.std_error < 1e-13
        with pytest.raises(P.InvalidArgument, match="nonnegative"):
            ctx.set_vector(np.array([1.0, -1.0]))
            P.mc_forward_scalar(ctx, 1.0, 0.5, 10, 0)
    with P.Context(k2, np.ones(2)) as ctx:
        r = P.mc_single_entry(ctx, 0, 1.0, 1.0 / 16, 1000, 3)
        assert r.estimate == pytest.approx(math.e, rel=1e-13)
        with pytest.raises(P.InvalidArgument, match="at least 2"):
            P.mc_single_entry(ctx, 0, 1.0, 0.25, 1, 3)
        with pytest.raises(P.OutOfRange):
            P.mc_single_entry(ctx, 2, 1.0, 0.25, 10, 3)
        with pytest.raises(P.InvalidArgument, match="integer step count"):
            P.mc_single_entry(ctx, 0, 1.0, 0.3, 10, 3)
        with pytest.raises(P.InvalidArgument, match="positive"):
            P.mc_single_entry(ctx, 0, -1.0, 0.25, 10, 3)
        with pytest.raises(P.InvalidArgument, match="epsilon"):
            P.mc_auto(ctx, 0, 1.0, 0.0, 3)


@pytest.mark.gpu
def test_gpu_mc_matches_oracle_on_c1_rows(gpu, oracle_lib):
    """Random C1 rows and step counts (including non powers of two) against the oracle."""
    import paper_1904_12754_b200 as P
    from paper_1904_12754_b200 import configs

    cfg = configs.make_config("c1")
    och = oracle_lib.chain(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val))
    rng = np.random.default_rng(9)
    with P.Context(cfg.a, cfg.u) as ctx:
        for _ in range(6):
            entry = int(rng.integers(0, cfg.a.n))
            steps = int(rng.integers(1, 40))
            samples = int(rng.integers(2, 3000))
            seed = int(rng.integers(0, 2 ** 40))
            dt = cfg.beta / steps
            got = P.mc_single_entry(ctx, entry, cfg.beta, dt, samples, seed)
            exp = och.mc_single_entry(cfg.u, entry, cfg.beta, dt, samples, seed)
            assert (got.samples, got.steps, got.wall_cost, got.jumps) == (exp["samples"], exp["steps"],
                                                                          exp["wall_cost"], exp["jumps"])
            assert got.estimate == pytest.approx(exp["estimate"], rel=1e-13)
            assert got.std_error == pytest.approx(exp["std_error"], rel=1e-9, abs=1e-15)


@pytest.mark.gpu
def test_gpu_mc_event_sampler_statistical(gpu, golden_mc):
    """Classical MC on the event-driven sampler (same law, different draws): its estimates agree
    with the reference-order sampler's within combined standard errors; costs follow the same
    cost model (jumps + non-absorbing step ends + steps)."""
    import paper_1904_12754_b200 as P

    m = golden_mc["matrices"]["smallw100"]
    beta = float.fromhex(m["beta"])
    res = {}
    for sampler in ("reference", "event"):
        c = csr(m)
        with P.Context(P.SparseMatrix(c.n, c.row_ptr, c.col, c.val), unhex(m["u"]), sampler=sampler) as ctx:
            res[sampler] = [P.mc_single_entry(ctx, e, beta, beta / 8, 200000, 21 + e) for e in (0, 50, 99)]
    for a, b in zip(res["reference"], res["event"]):
        assert abs(a.estimate - b.estimate) < 4 * math.sqrt(a.std_error ** 2 + b.std_error ** 2)
        assert a.steps == b.steps == 8
