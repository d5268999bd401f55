"""Pin the CPU oracle (oracle/expmc_oracle.c) against the reference's own outputs.

golden.json is produced by tests/golden/make_golden.py from the UNMODIFIED reference library
(oracle/_ref).  The restatement must reproduce every value BIT FOR BIT: Philox uniforms
(rng.hpp), decompositions (chain.cpp:15-71), per-sample functionals (paths.cpp:99-141),
run_level sums (mlmc.cpp:76-148) and full mlmc_driver runs (mlmc.cpp:170-260).  The
known-answer cases of the reference's own unit tests (test_paths.cpp, test_mlmc.cpp) are
re-checked here against the oracle as well.
"""
import math

import numpy as np
import pytest

from oracle import CSR, Oracle, have_reference


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


def csr_of(m):
    c = m["csr"]
    return CSR(c["n"], np.array(c["row_ptr"], np.int64), np.array(c["col"], np.int64), unhex(c["val"]))


def test_uniforms_match_reference(golden, oracle_lib):
    for rec in golden["uniforms"]:
        got = oracle_lib.uniforms(*rec["key"], len(rec["values"]))
        assert np.array_equal(got, unhex(rec["values"])), rec["key"]


def test_survey_appendix_a_anchors(oracle_lib):
    # SURVEY.md Appendix A (first four uniforms of three keys), rng.hpp:21-79
    anchors = {(0, 0, 0, 0): ["0x1.78af58993601bp-1", "0x1.989fa35785a7p-2", "0x1.634ae9d612fdfp-1", "0x1.f1c99948b964p-1"],
               (42, 3, 12345, 0): ["0x1.6d10b04e3519p-2", "0x1.0ab112f3d453p-5", "0x1.cde5c5b8452fp-3", "0x1.14dd3a134a6d4p-3"],
               (7, 5, 2 ** 40, 2): ["0x1.d3f2f35abc52cp-3", "0x1.6439eb9818c72p-2", "0x1.633406c5126c7p-1", "0x1.99bbcd3a20f78p-1"]}
    for key, vals in anchors.items():
        assert np.array_equal(oracle_lib.uniforms(*key, 4), unhex(vals))
    # coupled anchors on the two-state chain of test_paths.cpp:150-151
    ch = oracle_lib.chain(CSR.from_dense([[0.2, 1.0], [0.5, -0.3]]))
    s = ch.samples(np.array([0.7, 1.3]), 0, 0.8, 1, 0, 5, np.arange(4))
    assert [x.hex() for x in s["fine"]] == ["0x1.63cf254ff38f8p+1", "0x1.63cf254ff38f8p+1", "0x1.dd031457e932fp+0",
                                            "0x1.d404191a4d342p+0"]
    assert [x.hex() for x in s["coarse"]] == ["0x1.234fd8f19b1c2p+1"] * 3 + ["0x1.d404191a4d342p+0"]
    assert list(s["cost"]) == [5, 5, 5, 4]


@pytest.mark.parametrize("name", ["two_state", "k2", "diag", "signed3", "absorb3", "grid8", "smallw100", "pref300"])
def test_decomposition_matches_reference(golden, oracle_lib, name):
    m = golden["matrices"][name]
    dec = oracle_lib.chain(csr_of(m)).decomposition()
    assert np.array_equal(dec["d"], unhex(m["d"]))
    assert np.array_equal(dec["rate"], unhex(m["rate"]))
    assert np.array_equal(dec["row_ptr"], np.array(m["row_ptr"]))
    assert np.array_equal(dec["jump_cdf"], unhex(m["jump_cdf"]))
    assert np.array_equal(dec["jump_target"], np.array(m["jump_target"]))
    assert np.array_equal(dec["sign"], np.array(m["sign"], np.uint8))
    assert dec["d_max"] == float.fromhex(m["d_max"]) and dec["d_bar"] == float.fromhex(m["d_bar"])


@pytest.mark.parametrize("name", ["two_state", "k2", "diag", "signed3", "absorb3", "grid8", "smallw100", "pref300"])
def test_samples_and_run_level_match_reference(golden, oracle_lib, name):
    m = golden["matrices"][name]
    ch = oracle_lib.chain(csr_of(m))
    u = unhex(m["u"])
    beta = float.fromhex(m["beta"])
    for s in m["samples"]:
        got = ch.samples(u, s["entry"], beta, s["level"], s["base"], s["seed"], np.array(s["idx"], np.uint64))
        assert np.array_equal(got["fine"], unhex(s["fine"]))
        assert np.array_equal(got["coarse"], unhex(s["coarse"]))
        assert np.array_equal(got["cost"], np.array(s["cost"], np.uint64))
    for r in m["run_level"]:
        got = ch.run_level(u, r["entry"], beta, r["level"], r["base"], r["first"], r["count"], r["seed"], threads=3)
        assert got["sum"] == float.fromhex(r["sum"]) and got["sum_sq"] == float.fromhex(r["sum_sq"])
        assert got["samples"] == r["samples"] and got["cost"] == r["cost"]


@pytest.mark.parametrize("name", ["grid16", "c1"])
def test_driver_matches_reference(golden, oracle_lib, name):
    d = golden["drivers"][name]
    a = oracle_lib.grid_laplacian(d["g"])
    u = oracle_lib.grid_vector(12345, a.n)
    ch = oracle_lib.chain(a)
    res = ch.driver_rows(u, float.fromhex(d["beta"]), d["rows"], [1000 + r for r in d["rows"]], epsilon=d["epsilon"],
                         threads=4)
    for got, ref in zip(res, d["results"]):
        assert got["estimate"] == float.fromhex(ref["estimate"])
        assert got["statistical_error"] == float.fromhex(ref["statistical_error"])
        assert got["bias_estimate"] == float.fromhex(ref["bias_estimate"])
        assert (got["l0"], got["L"], got["total_cost"], got["converged"]) == (ref["l0"], ref["L"], ref["total_cost"],
                                                                               ref["converged"])
        for lv, rl in zip(got["levels"], ref["levels"]):
            assert lv["sum"] == float.fromhex(rl["sum"]) and lv["samples"] == rl["samples"] and lv["cost"] == rl["cost"]
    exact = oracle_lib.dense_expmv(a, u, float.fromhex(d["beta"]))
    assert np.array_equal(exact[d["rows"]], unhex(d["exact"]))


# ---------------------------------------------------------------- reference unit-test KATs
def test_kat_diagonal_single_exact(oracle_lib):  # test_paths.cpp:84-99
    ch = oracle_lib.chain(CSR.from_dense([[0.75, 0.0], [0.0, -0.5]]))
    s = ch.samples(np.array([3.0, 5.0]), 0, 2.0, 3, 1, 2, np.arange(50))
    assert np.all(s["fine"] == s["fine"][0]) and np.all(s["cost"] == 8)
    assert s["fine"][0] == pytest.approx(3.0 * math.exp(2.0 * 0.75), rel=1e-14)


def test_kat_k2_is_e(oracle_lib):  # test_paths.cpp:101-111
    ch = oracle_lib.chain(CSR.from_dense([[0.0, 1.0], [1.0, 0.0]]))
    s = ch.samples(np.ones(2), 0, 1.0, 4, 1, 3, np.arange(1000))
    assert np.all(s["fine"] == math.exp(1.0))


def test_kat_coupled_zero_on_diagonal(oracle_lib):  # test_paths.cpp:135-146
    ch = oracle_lib.chain(CSR.from_dense([[1.5, 0.0], [0.0, 0.25]]))
    s = ch.samples(np.array([2.0, 1.0]), 0, 2.0, 3, 0, 4, np.arange(100))
    assert np.all(s["fine"] - s["coarse"] == 0.0)
    assert s["fine"][0] == pytest.approx(2.0 * math.exp(3.0), rel=1e-14)


def test_kat_sign_parity(oracle_lib):  # test_paths.cpp:226-249 (via the per-sample path, level 0)
    pos = CSR.from_dense([[0, 1.0, 0], [1.0, 0, 0.5], [0, 0.5, 0]])
    neg = CSR.from_dense([[0, -1.0, 0], [-1.0, 0, -0.5], [0, -0.5, 0]])
    u = np.array([1.0, 2.0, 3.0])
    a = oracle_lib.chain(pos).samples(u, 0, 2.0, 0, 1, 8, np.arange(200))
    b = oracle_lib.chain(neg).samples(u, 0, 2.0, 0, 1, 8, np.arange(200))
    assert np.array_equal(a["end_state"], b["end_state"]) and np.array_equal(a["jumps"], b["jumps"])
    assert np.array_equal(b["fine"], a["fine"] * np.where(a["jumps"] % 2 == 0, 1.0, -1.0))


def test_kat_run_level_diagonal_zero(oracle_lib):  # test_mlmc.cpp:94-108
    ch = oracle_lib.chain(CSR.from_dense([[1.5, 0.0], [0.0, 0.5]]))
    r = ch.run_level(np.array([1.0, 2.0]), 0, 1.0, 3, 0, 0, 500, 9)
    assert r["sum"] == 0.0 and r["sum_sq"] == 0.0 and r["samples"] == 500


def test_kat_driver_diagonal_exact(oracle_lib):  # test_mlmc.cpp:145-163
    ch = oracle_lib.chain(CSR.from_dense([[0.75, 0.0], [0.0, -0.25]]))
    (r,) = ch.driver_rows(np.array([3.0, 1.0]), 2.0, [0], [5], epsilon=1e-6)
    # test_mlmc.cpp:159 asks for exact ==; the reference itself misses by 4.8e-14 (a mean of
    # 1000 identical values is not exact), as SURVEY §4 records -- pin the reference's value.
    assert r["converged"] and r["estimate"] == pytest.approx(3.0 * math.exp(1.5), rel=1e-14)
    assert r["estimate"].hex() == "0x1.ae3dfd977a7fdp+3"
    assert r["statistical_error"] == 0.0 and r["bias_estimate"] == 0.0
    assert all(lv["samples"] == 1000 for lv in r["levels"])


def test_kat_driver_k2(oracle_lib):  # test_mlmc.cpp:165-182
    ch = oracle_lib.chain(CSR.from_dense([[0.0, 1.0], [1.0, 0.0]]))
    res = ch.driver_rows(np.ones(2), 1.0, [0] * 10, list(range(10)), epsilon=1e-3)
    for r in res:
        assert r["converged"] and abs(r["estimate"] - math.e) <= 1e-3


def test_allocation_and_bias_closed_forms(oracle_lib):  # test_mlmc.cpp:17-88
    assert oracle_lib.initial_level(0.25, 4.0) == 1 and oracle_lib.initial_level(1.0, 7.0) == 4
    assert oracle_lib.initial_level(1.0, 0.25) == 0 and oracle_lib.initial_level(1.0, -3.0) == 0
    assert list(oracle_lib.optimal_allocation([1.0], [1.0], 0.1)) == [200]
    m = oracle_lib.optimal_allocation([1.0, 0.25], [1.0, 4.0], 0.1)
    assert m[0] / m[1] == pytest.approx(4.0)
    tail = 4.0 ** -6 / 3.0
    assert oracle_lib.bias_estimate([4.0 ** -l for l in range(1, 7)]) == pytest.approx(tail, rel=1e-9)


def test_oracle_errors(oracle_lib):
    from oracle import InvalidArgument, OutOfRange

    ch = oracle_lib.chain(CSR.from_dense([[0.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(OutOfRange):
        ch.run_level(np.ones(2), 2, 1.0, 1, 0, 0, 10, 1)
    with pytest.raises(InvalidArgument):
        ch.run_level(np.ones(2), 0, 1.0, 63, 0, 0, 10, 1)
    with pytest.raises(InvalidArgument):
        oracle_lib.chain(CSR(2, np.array([0, 1, 1]), np.array([1]), np.array([np.nan])))


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference here)")
def test_oracle_equals_reference_on_c1_rows(oracle_lib):
    from oracle import Reference

    ref = Reference()
    a = oracle_lib.grid_laplacian(64)
    u = oracle_lib.grid_vector(12345, a.n)
    rows = [3, 700, 2222, 4000]
    got = oracle_lib.chain(a).driver_rows(u, 1.0, rows, [1000 + r for r in rows], threads=4)
    exp = ref.chain(a).driver_rows(u, 1.0, rows, [1000 + r for r in rows], threads=4)
    for g, e in zip(got, exp):
        assert g["estimate"] == e["estimate"] and g["total_cost"] == e["total_cost"]
        assert g["total_jumps"] == e["total_jumps"]  # jumps formula is exact here
