"""Self-check of the reference build the oracle is pinned to: the reference's own unit tests
(/root/reference/proj/tests, compiled in place by `make -C oracle reftests` against
oracle/_ref/libexpmc_ref.so, with the doctest-subset shim oracle/doctest_shim/doctest.h) must
give the known result -- 104 test cases, all passing except the two genuine reference failures
recorded in SURVEY.md §4:
  * test_mlmc.cpp:145 "driver on a diagonal matrix converges at warmup with the exact value"
    (demands exact == for a mean of 1000 equal values; the reference misses by 4.8e-14), and
  * test_mc.cpp:92 "mc_auto achieves the requested accuracy most of the time" (17 of 20 hits
    where the test wants 18).
Runs only where the reference sources exist (this container), never on the GPU box."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
KNOWN_FAILURES = {"driver on a diagonal matrix converges at warmup with the exact value",
                  "mc_auto achieves the requested accuracy most of the time"}


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference sources not present")
def test_reference_unit_tests_pass_on_the_oracle_build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "reftests"], check=True)
    r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "unit_tests")], capture_output=True, text=True,
                       timeout=1200)
    failed = {line[len("FAILED: "):].rsplit(" (", 1)[0] for line in r.stdout.splitlines() if line.startswith("FAILED: ")}
    summary = [line for line in r.stdout.splitlines() if line.startswith("[doctest-shim]")]
    assert summary and "test cases: 104" in summary[0], r.stdout[-2000:]
    assert failed == KNOWN_FAILURES, r.stdout[-4000:]
