"""GPU: BASELINE configs 3-5 on scaled-down instances of the same generators.

C5 (3-D convection-diffusion: non-uniform rows, mixed signs, degree 6 -> the CDF binary-search
path) runs the reference-order sampler: per-sample and per-driver parity with the oracle is
exact.  C3 (Barabasi-Albert, the reference's pref) and C4 (R-MAT) run the event-driven sampler
they are configured with: every component within 3 combined standard errors of the reference
driver -- exceedances consistent with Binomial(n, 0.0027) (tail probability >= 1e-3) -- and the
RMS rule against the deterministic e^{beta A} 1.  The configured sizes and eps are pinned against
the reference driver in tests/test_gpu_scale_parity.py.
"""
import math

import numpy as np
import pytest

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs
from oracle import CSR
from scipy.stats import binom

pytestmark = pytest.mark.gpu


def _csr(a):
    return CSR(a.n, a.row_ptr, a.col, a.val)


def _ulps(a, b):
    ia = np.asarray(a, np.float64).view(np.int64)
    ib = np.asarray(b, np.float64).view(np.int64)
    ia = np.where(ia < 0, np.int64(-(2 ** 63)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2 ** 63)) - ib, ib)
    return np.abs(ia - ib)


def test_c5_small_exact_parity(gpu, oracle_lib):
    cfg = configs.make_config("c5-12")
    och = oracle_lib.chain(_csr(cfg.a))
    rng = np.random.default_rng(5)
    with P.Context(cfg.a, cfg.u) as ctx:
        dec = ctx.decomposition()
        ref = och.decomposition()
        for k in ("d", "rate", "row_ptr", "jump_cdf", "jump_target", "sign"):
            assert np.array_equal(dec[k], ref[k]), k
        for level in range(0, 5):
            for base in ([1] if level == 0 else [1, 0]):
                rows = rng.integers(0, cfg.a.n, 200)
                idx = rng.integers(0, 2 ** 40, 200).astype(np.uint64)
                got = ctx.sample_debug(cfg.beta, rows, level, base, 1000 + rows, idx)
                for k in range(200):
                    e = och.samples(cfg.u, int(rows[k]), cfg.beta, level, base, 1000 + int(rows[k]), idx[k:k + 1])
                    assert got["cost"][k] == e["cost"][0] and got["end_state"][k] == e["end_state"][0]
                    assert _ulps(got["fine"][k], e["fine"][0]) <= 4 and _ulps(got["coarse"][k], e["coarse"][0]) <= 4
        rows = np.array([0, 5, 700, 1727])
        opts = dict(epsilon=2e-2, max_levels_above_l0=cfg.max_levels_above_l0)
        res, _ = P.mlmc_driver_rows(ctx, cfg.beta, rows, configs.row_seeds(rows), P.MlmcOptions(**opts))
    exp = och.driver_rows(cfg.u, cfg.beta, rows, configs.row_seeds(rows), threads=8, **opts)
    for k, e in enumerate(exp):
        assert int(res["total_cost"][k]) == e["total_cost"] and int(res["L"][k]) == e["L"]
        assert float(res["estimate"][k]) == pytest.approx(e["estimate"], rel=1e-10, abs=1e-12)


def _statistical_check(cfg, rows, eps, oracle_lib):
    with P.Context(cfg.a, cfg.u, sampler=cfg.sampler) as ctx:
        res, _ = P.mlmc_driver_rows(ctx, cfg.beta, rows, configs.row_seeds(rows), P.MlmcOptions(epsilon=eps))
    och = oracle_lib.chain(_csr(cfg.a))
    ref = och.driver_rows(cfg.u, cfg.beta, rows, configs.row_seeds(rows) + 7, epsilon=eps, threads=16)
    est_r = np.array([r["estimate"] for r in ref])
    se_r = np.array([r["statistical_error"] for r in ref])
    z = np.abs(res["estimate"] - est_r) / np.sqrt(res["statistical_error"] ** 2 + se_r ** 2 + 1e-300)
    assert res["converged"].all()
    k = int(np.sum(z > 3))
    assert k == 0 or binom.sf(k - 1, len(z), 0.0027) >= 1e-3, (k, len(z), z)
    exact = oracle_lib.dense_expmv(_csr(cfg.a), cfg.u, cfg.beta)[rows]
    err = res["estimate"] - exact
    assert math.sqrt(float(np.mean(err ** 2))) <= eps
    return res, exact


def test_c3_small_ba_statistical(gpu, oracle_lib):
    cfg = configs.make_config("c3-20000")
    assert cfg.sampler == "event"
    deg = np.diff(cfg.a.row_ptr)
    order = np.argsort(deg)
    # degree-stratified; the hubs are pinned at the configured size against the reference driver
    # (tests/test_gpu_scale_parity.py) -- the CPU reference needs hours for them at this eps
    rows = np.sort(np.r_[order[:: len(order) // 24][:24], order[-200]])
    _statistical_check(cfg, rows, 1e-2, oracle_lib)


def test_c4_small_rmat_statistical(gpu, oracle_lib):
    cfg = configs.make_config("c4-13")
    deg = np.diff(cfg.a.row_ptr)
    iso = np.flatnonzero(deg == 0)[:4]
    order = np.argsort(deg)
    nz = order[deg[order] > 0]
    rows = np.sort(np.r_[iso, nz[:: len(nz) // 20][:20]])
    res, exact = _statistical_check(cfg, rows, 1e-2, oracle_lib)
    isolated = np.isin(rows, iso)
    assert np.all(res["estimate"][isolated] == 1.0) and np.all(exact[isolated] == 1.0)  # absorbing rows: exactly u
    assert np.all(res["statistical_error"][isolated] == 0.0)
