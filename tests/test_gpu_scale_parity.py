"""GPU parity at the CONFIGURED sizes and eps (BASELINE configs C2, C3, C4 family; eps = 1e-3).

The reference side is the UNMODIFIED reference's mlmc_driver run on the same components, committed
as fixtures by tests/golden/make_scale_fixtures.py (the CPU reference takes hours on the C3 / R-MAT
components and /root/reference is absent on the GPU box).  The matrices are regenerated here by the
product's host generators and pinned to the fixtures by a SHA-256 of their CSR and by beta's bits.

Rules (north_star):
  * statistical: |x_gpu - x_ref| <= 3 sqrt(SE_gpu^2 + SE_ref^2) on every component, up to a count of
    exceedances consistent with Binomial(n, p) (tail probability >= 1e-3).  p = 0.0027 (the normal
    tail) on C2.  On the graph configs the REFERENCE ITSELF meets neither that p nor eps: against
    a rerun of itself with other row seeds 9-14 of 355 C3 components lie beyond 3 combined SE
    (3-4 %, sd of z 1.4; on R-MAT scale 20 the estimates move by ~4 reported SE from seed to
    seed), and against the deterministic e^{beta A} 1 its estimates carry a bias of -1.5e-3 (C3)
    / -1.9e-3 (R-MAT 20) and an RMS error of 2.1e-3 / 3.4e-3 at eps = 1e-3 -- the driver's SE and
    bias estimates come from sample moments of heavy-tailed level corrections (most samples of a
    coupled level are exactly 0, a few are large) and understate both.  Parity with the reference
    there means REPRODUCING ITS ERROR LAW, so the graph test checks, on the same components and
    against the deterministic value (oracle dense_expmv), that the event sampler's errors have
    the reference's mean (two-sample test, 4 sd), the reference's RMS (within 25 %) and the
    reference's distribution (two-sample Kolmogorov-Smirnov); where reruns of the reference
    exist (C3: tests/golden/scale_c3_reseed.json, written by scripts/scale_diag.py from the
    reference-order sampler -- the reference draw for draw, as this file asserts -- with shifted
    row seeds) the 3-SE rule is applied with the reference's own seed-to-seed exceedance rate as
    p, with mean signed z within 4 sd / sqrt(n) and a KS test of |z| against the reference's own;
  * reference-order sampler (draw for draw the reference): identical decision sequences (same l0,
    L, samples per level, cost) on >= 99 % of the components and equal estimates there;
  * event-driven sampler (statistically equivalent paths): the statistical rule, plus
    level means equal to the reference-order sampler's at l0 .. l0+3 within 4 combined SE.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.stats import binom

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import configs

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
P_3SE = 0.0027  # two-sided normal tail beyond 3 sigma


def _fixture(name):
    path = os.path.join(HERE, "golden", f"scale_{name}.json")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path} (tests/golden/make_scale_fixtures.py {name})")
    with open(path) as f:
        return json.load(f)


def _csr_hash(a):
    import hashlib

    h = hashlib.sha256()
    for x in (np.ascontiguousarray(a.row_ptr, np.int64), np.ascontiguousarray(a.col, np.int64),
              np.ascontiguousarray(a.val, np.float64)):
        h.update(x.tobytes())
    return h.hexdigest()


_CFG_CACHE = {}


def _make_config(name):
    """The configured-size graphs take a minute to generate: the tests of one run share them."""
    if name not in _CFG_CACHE:
        _CFG_CACHE.clear()  # one large matrix at a time (C4: 8 GB of host CSR)
        _CFG_CACHE[name] = configs.make_config(name)
    return _CFG_CACHE[name]


def binomial_consistent(k, n, p=P_3SE, alpha=1e-3):
    """P(X >= k) for X ~ Binomial(n, p) is at least alpha."""
    return k == 0 or float(binom.sf(k - 1, n, p)) >= alpha


def _ref_arrays(fx):
    done = [r for r in fx["rows"] if not r.get("timed_out")]
    rows = np.array([r["row"] for r in done], np.int64)
    est = np.array([float.fromhex(r["estimate"]) for r in done])
    se = np.array([float.fromhex(r["statistical_error"]) for r in done])
    return done, rows, est, se


def _config(name, fx):
    cfg = configs.make_config(name)
    assert _csr_hash(cfg.a) == fx["csr_sha256"], "matrix differs from the fixture's"
    assert cfg.beta == float.fromhex(fx["beta"]), (cfg.beta, fx["beta"])
    return cfg


def _solve(cfg, rows, sampler):
    with P.Context(cfg.a, cfg.u, sampler=sampler) as ctx:
        res, lv = P.mlmc_driver_rows(ctx, cfg.beta, rows, configs.row_seeds(rows),
                                     P.MlmcOptions(epsilon=1e-3))  # the reference's options: no budget
    return res, lv


def _same_decisions(res, lv, done):
    same = np.zeros(len(done), bool)
    for k, r in enumerate(done):
        g = res[k]
        if (int(g["l0"]), int(g["L"]), int(g["total_cost"])) != (r["l0"], r["L"], r["total_cost"]):
            continue
        n_l = int(g["nlevels"])
        same[k] = n_l == len(r["levels"]) and all(
            int(a["samples"]) == b["samples"] and int(a["cost"]) == b["cost"] for a, b in zip(lv[k][:n_l], r["levels"]))
    return same


def _statistical(res, est, se, label, p=P_3SE):
    diff = np.abs(res["estimate"] - est)
    # components whose samples are all equal (degree-1 rows of a graph: SE 0) agree to rounding
    z = np.where(diff <= 1e-12 * np.maximum(1.0, np.abs(est)), 0.0,
                 diff / np.sqrt(res["statistical_error"] ** 2 + se ** 2 + 1e-300))
    k = int(np.sum(z > 3.0))
    print(f"{label}: {len(z)} components, {k} beyond 3 combined SE (expected {p * len(z):.2f}), max z {z.max():.2f}")
    assert binomial_consistent(k, len(z), p=p), (k, len(z), np.sort(z)[-8:])
    return z


def _reference_null(name, rows, est, se):
    """The reference's own seed-to-seed z values on these components (the reseed fixture): signed
    z of every pair of reference runs (the CPU reference's fixture and the reference-order
    sampler's shifted-seed runs), and the pooled rate of |z| > 3."""
    fx = _fixture(f"{name}_reseed")
    assert fx["rows"] == rows.tolist()
    runs = [(est, se)]
    for key, r in fx["runs"].items():
        if key.startswith("reference_") and key != "reference_0":
            runs.append((np.array([float.fromhex(x) for x in r["estimate"]]),
                         np.array([float.fromhex(x) for x in r["statistical_error"]])))
    assert len(runs) >= 2
    # the shift-0 reference-order run IS the fixture (the reference draw for draw)
    r0 = fx["runs"]["reference_0"]
    assert np.mean(np.abs(np.array([float.fromhex(x) for x in r0["estimate"]]) - est) <= 1e-10 * np.abs(est)) >= 0.99
    zs = []
    for i in range(len(runs)):
        for j in range(i + 1, len(runs)):
            zs.append((runs[i][0] - runs[j][0]) / np.sqrt(runs[i][1] ** 2 + runs[j][1] ** 2))
    zs = np.concatenate(zs)
    return zs, float(np.mean(np.abs(zs) > 3.0))


def _statistical_vs_null(res, est, se, label, znull, p_null):
    """The statistical rule with the reference's own exceedance rate, plus unbiasedness and equality
    of the z distributions (module docstring)."""
    from scipy.stats import ks_2samp

    sz = (res["estimate"] - est) / np.sqrt(res["statistical_error"] ** 2 + se ** 2)
    n = len(sz)
    k = int(np.sum(np.abs(sz) > 3.0))
    ks = ks_2samp(np.abs(sz), np.abs(znull))
    print(f"{label}: {n} components, {k} beyond 3 combined SE; the reference against its own reruns: "
          f"{p_null * n:.1f} expected ({p_null:.4f}, nominal {P_3SE}); mean signed z {sz.mean():+.3f} "
          f"(sd {sz.std():.2f}), KS p-value vs the reference's own |z| {ks.pvalue:.3f}")
    assert binomial_consistent(k, n, p=max(p_null, P_3SE)), (k, n, p_null)
    assert abs(sz.mean()) <= 4.0 * sz.std() / math.sqrt(n), sz.mean()
    assert ks.pvalue >= 1e-3, ks
    return np.abs(sz)


def _same_error_law(res, est, exact, label, eps):
    """The event sampler's errors against the deterministic value follow the reference's own error
    law on the same components: same mean (two-sample test, 4 sd), same RMS (within 25 %), same
    distribution (two-sample KS).  Neither has to meet eps: the reference does not on these graphs."""
    from scipy.stats import ks_2samp

    e_gpu, e_ref = res["estimate"] - exact, est - exact
    n = len(e_gpu)
    rms_g, rms_r = math.sqrt(float(np.mean(e_gpu ** 2))), math.sqrt(float(np.mean(e_ref ** 2)))
    sd = math.sqrt(float(e_gpu.var() + e_ref.var()) / n)
    ks = ks_2samp(e_gpu, e_ref)
    print(f"{label} vs the deterministic value (eps {eps:g}): mean error {e_gpu.mean():+.2e} (reference "
          f"{e_ref.mean():+.2e}, difference {abs(e_gpu.mean() - e_ref.mean()) / sd:.2f} sd), RMS {rms_g:.2e} "
          f"(reference {rms_r:.2e}), KS p-value {ks.pvalue:.3f}")
    assert abs(e_gpu.mean() - e_ref.mean()) <= 4.0 * sd
    assert 0.8 <= rms_g / rms_r <= 1.25, (rms_g, rms_r)
    assert ks.pvalue >= 1e-3, ks


def test_c2_full_size_vs_reference_driver(gpu):
    """C2 at n = 2^20: 512 seed-chosen components, reference-order sampler (the config's)."""
    fx = _fixture("c2")
    cfg = _config("c2", fx)
    done, rows, est, se = _ref_arrays(fx)
    assert len(done) >= 256
    res, lv = _solve(cfg, rows, "reference")
    assert res["converged"].all()
    same = _same_decisions(res, lv, done)
    assert same.mean() >= 0.99, same.mean()
    assert np.allclose(res["estimate"][same], est[same], rtol=1e-10, atol=1e-13)
    _statistical(res, est, se, "C2")


@pytest.mark.parametrize("name", ["c3", "c4-20"])
def test_graph_full_size_vs_reference_driver(gpu, oracle_lib, name):
    """C3 (BA n = 1e6, full graph) and R-MAT scale 20 at eps = 1e-3 on >= 256 degree-stratified
    components, hubs included wherever the reference finished them within the fixture's cap.

    * event-driven sampler (the configs' sampler): statistical rule vs the reference's estimates;
    * reference-order sampler: identical decision sequences on >= 99 %."""
    fx = _fixture(name)
    cfg = _config(name, fx)
    done, rows, est, se = _ref_arrays(fx)
    assert len(done) >= 256, len(done)
    strata = np.array([r["stratum"] for r in done])
    # every stratum was attempted; a stratum may be missing from the comparison only when the
    # reference itself finished none of its components within the fixture's cap (hub rows:
    # the reference has no budget and needs hours for them)
    attempted = {r["stratum"] for r in fx["rows"]}
    assert attempted == set(range(len(fx["strata"]))), attempted
    for s in range(len(fx["strata"])):
        if s not in set(strata.tolist()):
            rs = [r for r in fx["rows"] if r["stratum"] == s]
            assert all(r.get("timed_out") for r in rs), s
            print(f"  stratum {fx['strata'][s]}: the reference finished none of {len(rs)} within "
                  f"{fx['cap_seconds']} s ({sum(bool(r.get('skipped')) for r in rs)} not attempted after "
                  f"consecutive timeouts of lighter components)")
    res_e, _ = _solve(cfg, rows, "event")
    assert res_e["converged"].mean() >= 0.99
    from oracle import CSR

    exact = oracle_lib.dense_expmv(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val), cfg.u, cfg.beta)[rows]
    _same_error_law(res_e, est, exact, f"{name} event sampler", 1e-3)
    p_null = P_3SE
    if os.path.exists(os.path.join(HERE, "golden", f"scale_{name}_reseed.json")):
        znull, p_null = _reference_null(name, rows, est, se)
        z = _statistical_vs_null(res_e, est, se, f"{name} event sampler", znull, p_null)
    else:  # no rerun of the reference within reach (R-MAT 20: > 46 GPU-minutes): reported, not asserted
        sz = (res_e["estimate"] - est) / np.sqrt(res_e["statistical_error"] ** 2 + se ** 2 + 1e-300)
        z = np.abs(sz)
        print(f"{name} event sampler: {int(np.sum(z > 3))} of {len(z)} beyond 3 combined SE, sd of z {sz.std():.2f} "
              "(no reference rerun for this config; the reported SE understates the seed-to-seed spread)")
    for s in sorted(set(strata.tolist())):
        m = strata == s
        print(f"  stratum {fx['strata'][s]}: {m.sum()} components, max z {z[m].max():.2f}")
    res_r, lv_r = _solve(cfg, rows, "reference")
    same = _same_decisions(res_r, lv_r, done)
    print(f"{name} reference-order sampler: identical decision sequences on {same.mean():.4f}")
    assert same.mean() >= 0.99
    assert np.allclose(res_r["estimate"][same], est[same], rtol=1e-10, atol=1e-13)
    # draw for draw the reference: the same seeds give the same estimates (z = 0 on the identical ones)
    _statistical(res_r, est, se, f"{name} reference-order sampler", p=max(p_null, P_3SE))


def _level_means(name, strata, per_stratum, l0_expected, m):
    cfg = _make_config(name)
    deg = np.diff(cfg.a.row_ptr)
    rng = np.random.default_rng(7)
    rows = []
    for lo, hi in strata:
        cand = np.where((deg >= lo) & (deg <= hi))[0]
        rows += list(rng.choice(cand, size=per_stratum, replace=False))
    rows = np.array(rows, np.int64)
    with P.Context(cfg.a, cfg.u) as ctx:
        l0 = P.initial_level(cfg.beta, ctx.d_max)
    assert l0_expected is None or l0 == l0_expected
    entry = np.repeat(rows, 4)
    level = np.tile(np.arange(l0, l0 + 4), len(rows))
    base = (level == l0).astype(np.int32)
    seeds = 777 + entry.astype(np.uint64)
    out = {}
    for sampler in ("event", "reference"):
        with P.Context(cfg.a, cfg.u, sampler=sampler) as ctx:
            out[sampler] = ctx.run_level_batch(cfg.beta, entry, level, base, 0, m, seeds)
    e, r = out["event"], out["reference"]
    me, mr = e["sum"] / m, r["sum"] / m
    ve = e["sum_sq"] / m - me ** 2
    vr = r["sum_sq"] / m - mr ** 2
    z = np.abs(me - mr) / np.sqrt((ve + vr) / m + 1e-300)
    k = int(np.sum(z > 4.0))
    print(f"{name} level means: {len(z)} (component, level) pairs, degrees {deg[rows].min()} .. {deg[rows].max()}, "
          f"{k} beyond 4 SE, max z {z.max():.2f}")
    assert binomial_consistent(k, len(z), p=6.3e-5)
    uc_e = e["cost"].astype(np.float64).sum() / (m * len(z))
    uc_r = r["cost"].astype(np.float64).sum() / (m * len(z))
    assert uc_e == pytest.approx(uc_r, rel=0.02)


def test_c3_event_vs_reference_order_level_means(gpu):
    """On the full C3 graph (l0 = 7): per-level sample means of the event-driven sampler equal the
    reference-order sampler's (which is the reference draw for draw) at levels 7 (base) .. 10
    (coupled), 2^18 samples each, on degree-stratified components: within 4 combined SE up to a
    Binomial-consistent count, and unit costs within 2 %."""
    _level_means("c3", [(5, 5), (6, 7), (8, 11), (12, 19), (20, 49), (50, 199), (200, 1 << 40)], 3, 7, 1 << 18)


def test_c4_configured_size_event_vs_reference_order_level_means(gpu):
    """The same at C4's configured size -- R-MAT scale 24, 2^24 rows, 5.2e8 chain edges, tables and
    edge records far beyond L2 -- where the CPU reference cannot run a driver in reasonable time
    (its run_level rebuilds an O(n) table per call): levels l0 = 8 .. 11, 2^16 samples each, 28
    components from degree 1 to the hubs."""
    _level_means("c4", [(1, 1), (2, 3), (4, 7), (8, 15), (16, 63), (64, 255), (256, 1 << 40)], 4, 8, 1 << 16)


def _ulps(a, b):
    ia, ib = np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64)
    ia = np.where(ia < 0, np.int64(-(2 ** 63)) - ia, ia)
    ib = np.where(ib < 0, np.int64(-(2 ** 63)) - ib, ib)
    return np.abs(ia - ib)


def test_c4_configured_size_per_sample_parity(gpu, oracle_lib):
    """C4 at its configured size (R-MAT scale 24: 2^24 rows, 5.2e8 chain edges, hub rows hundreds
    wide) against the oracle, sample by sample, at levels l0 = 8 .. 10 on components from degree 1
    to the hubs: the reference-order sampler's cost, jump count and end state exact, values within
    4 ulp -- the draw-for-draw pin the scale-20 fixture gives through the driver, on the full graph."""
    from oracle import CSR

    cfg = _make_config("c4")
    och = oracle_lib.chain(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val))
    deg = np.diff(cfg.a.row_ptr)
    rng = np.random.default_rng(44)
    rows = []
    for lo, hi in [(1, 1), (2, 3), (4, 7), (8, 15), (16, 63), (64, 255), (256, 1 << 40)]:
        cand = np.where((deg >= lo) & (deg <= hi))[0]
        rows += list(rng.choice(cand, size=6, replace=False))
    rows = np.array(rows, np.int64)
    with P.Context(cfg.a, cfg.u) as ctx:
        l0 = P.initial_level(cfg.beta, ctx.d_max)
        for level in range(l0, l0 + 3):
            for base in ([1] if level == l0 else [0]):
                idx = rng.integers(0, 2 ** 40, len(rows)).astype(np.uint64)
                got = ctx.sample_debug(cfg.beta, rows, level, base, 1000 + rows, idx)
                for k, r in enumerate(rows):
                    e = och.samples(cfg.u, int(r), cfg.beta, level, base, 1000 + int(r), idx[k:k + 1])
                    assert got["cost"][k] == e["cost"][0] and got["jumps"][k] == e["jumps"][0], (r, level, base)
                    assert got["end_state"][k] == e["end_state"][0], (r, level, base)
                    assert _ulps(got["fine"][k], e["fine"][0]) <= 4 and _ulps(got["coarse"][k], e["coarse"][0]) <= 4
        sel = rows[::6]  # one component per stratum through run_level (sums of 3000 samples)
        b = ctx.run_level_batch(cfg.beta, sel, l0, 1, 0, 3000, 1000 + sel)
        for k, r in enumerate(sel):
            o = och.run_level(cfg.u, int(r), cfg.beta, l0, 1, 0, 3000, 1000 + int(r))
            assert int(b["cost"][k]) == o["cost"] and int(b["jumps"][k]) == o["jumps"], r
            assert abs(float(b["sum"][k]) - o["sum"]) <= 1e-12 * max(1.0, math.sqrt(3000 * o["sum_sq"]))


def test_c5_configured_size_event_vs_reference_order_level_means(gpu):
    """C5 at its configured size -- the 3-D convection-diffusion operator on 256^3 (n = 2^24,
    non-uniform rows with mixed signs: the event sampler picks through its alias tables, the
    reference-order sampler through the reference's CDF search): levels l0 .. l0+3, 2^16 samples
    each, components from the corners (4 stored entries per row, the diagonal included) to the
    interior (7)."""
    _level_means("c5", [(4, 4), (5, 5), (6, 6), (7, 7)], 6, None, 1 << 16)


def test_c5_configured_size_per_sample_parity(gpu, oracle_lib):
    """C5 at its configured size against the oracle, sample by sample (the config has no driver
    fixture: the reference needs hours per component at eps = 1e-4): the reference-order sampler's
    cost, jump count and end state are exact and its values within 4 ulp on 256^3's non-uniform,
    mixed-sign rows, at levels 0 .. 4 (base and coupled) with sample indices up to 2^40."""
    from oracle import CSR

    cfg = _make_config("c5")
    och = oracle_lib.chain(CSR(cfg.a.n, cfg.a.row_ptr, cfg.a.col, cfg.a.val))
    deg = np.diff(cfg.a.row_ptr)
    rng = np.random.default_rng(55)
    rows = np.concatenate([rng.choice(np.where(deg == k)[0], size=min(30, int(np.sum(deg == k))), replace=False)
                           for k in (4, 5, 6, 7)])

    def ulps(a, b):
        ia, ib = np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64)
        ia = np.where(ia < 0, np.int64(-(2 ** 63)) - ia, ia)
        ib = np.where(ib < 0, np.int64(-(2 ** 63)) - ib, ib)
        return np.abs(ia - ib)

    with P.Context(cfg.a, cfg.u) as ctx:
        for level in range(0, 5):
            for base in ([1] if level == 0 else [1, 0]):
                idx = rng.integers(0, 2 ** 40, len(rows)).astype(np.uint64)
                got = ctx.sample_debug(cfg.beta, rows, level, base, 1000 + rows, idx)
                for k, r in enumerate(rows):
                    e = och.samples(cfg.u, int(r), cfg.beta, level, base, 1000 + int(r), idx[k:k + 1])
                    assert got["cost"][k] == e["cost"][0] and got["jumps"][k] == e["jumps"][0], (r, level, base)
                    assert got["end_state"][k] == e["end_state"][0], (r, level, base)
                    assert ulps(got["fine"][k], e["fine"][0]) <= 4 and ulps(got["coarse"][k], e["coarse"][0]) <= 4
        # run_level at level 0 (the level-0 walker) and level 3 (the general walker): exact counts
        sel = rows[::10]
        for level, base in ((0, 1), (3, 0)):
            b = ctx.run_level_batch(cfg.beta, sel, level, base, 0, 2000, 1000 + sel)
            for k, r in enumerate(sel):
                o = och.run_level(cfg.u, int(r), cfg.beta, level, base, 0, 2000, 1000 + int(r))
                assert int(b["cost"][k]) == o["cost"] and int(b["jumps"][k]) == o["jumps"], (r, level)
                assert abs(float(b["sum"][k]) - o["sum"]) <= 1e-12 * max(1.0, math.sqrt(2000 * o["sum_sq"]))
