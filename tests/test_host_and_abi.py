"""CPU-side checks of the product library: it loads without a GPU, exports every symbol the
C header declares, its host-side driver helpers equal the reference's, argument validation
raises the reference's exception types, and the config inputs equal the oracle's."""
import os
import re

import numpy as np
import pytest

import paper_1904_12754_b200 as P
from paper_1904_12754_b200 import _lib, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "expmc_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(expmc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 18
    lib = _lib.load()
    for n in names:
        assert hasattr(lib, n), n
    assert {s[0] for s in _lib.SYMBOLS} == set(names)


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_version_string():
    assert "sm_100a" in P.version()


def test_initial_level_matches_reference(oracle_lib):  # mlmc.cpp:19-23; test_mlmc.cpp:17-23
    cases = [(0.25, 4.0), (1.0, 7.0), (1.0, 0.25), (1.0, 0.0), (1.0, -3.0), (1 / 66.3, 4469.0), (0.5, 0.0)]
    for b, d in cases:
        assert P.initial_level(b, d) == oracle_lib.initial_level(b, d)
    with pytest.raises(P.InvalidArgument):
        P.initial_level(0.0, 1.0)


def test_optimal_allocation_matches_reference(oracle_lib):  # mlmc.cpp:25-43
    rng = np.random.default_rng(3)
    for _ in range(200):
        k = rng.integers(1, 8)
        v = rng.uniform(0, 2, k) * (rng.uniform(size=k) > 0.2)
        c = rng.uniform(1, 50, k)
        eps = 10 ** rng.uniform(-4, -1)
        assert np.array_equal(P.optimal_allocation(v, c, eps), oracle_lib.optimal_allocation(v, c, eps))
    assert list(P.optimal_allocation([1.0], [1.0], 0.1)) == [200]
    with pytest.raises(P.InvalidArgument):
        P.optimal_allocation([1.0], [0.0], 0.1)
    with pytest.raises(P.InvalidArgument):
        P.optimal_allocation([1.0], [1.0], 0.0)


def test_bias_estimate_matches_reference(oracle_lib):  # mlmc.cpp:45-51
    rng = np.random.default_rng(4)
    for _ in range(100):
        m = rng.normal(size=rng.integers(2, 9))
        assert P.bias_estimate(m) == oracle_lib.bias_estimate(m)
    assert P.bias_estimate([0.0, 0.0]) == 0.0
    with pytest.raises(P.InvalidArgument):
        P.bias_estimate([1.0])


def test_config_inputs_equal_oracle(oracle_lib):
    for g in (1, 2, 5, 64):
        a = configs.grid_laplacian(g)
        b = oracle_lib.grid_laplacian(g)
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col) and np.array_equal(a.val, b.val)
    assert np.array_equal(configs.grid_vector(12345, 5000), oracle_lib.grid_vector(12345, 5000))


def test_numpy_philox_matches_golden(golden):
    for rec in golden["uniforms"]:
        seed, level, sample, lane = rec["key"]
        got = configs.philox_first_uniform(seed, level, np.array([sample], np.uint64), lane)[0]
        assert got == float.fromhex(rec["values"][0])


def test_from_triplets_semantics():  # sparse.cpp:12-49
    a = P.SparseMatrix.from_triplets(3, [2, 0, 0, 1, 0], [0, 1, 1, 1, 2], [1.0, 0.5, 0.25, -1.0, 0.0])
    assert list(a.row_ptr) == [0, 1, 2, 3] and list(a.col) == [1, 1, 0] and list(a.val) == [0.75, -1.0, 1.0]
    with pytest.raises(P.OutOfRange):
        P.SparseMatrix.from_triplets(2, [0], [2], [1.0])
    with pytest.raises(P.InvalidArgument):
        P.SparseMatrix.from_triplets(2, [0], [1], [np.inf])
    # cancelling duplicates vanish
    b = P.SparseMatrix.from_triplets(2, [0, 0], [1, 1], [1.0, -1.0])
    assert b.nnz == 0


def test_ctx_create_validates_before_touching_the_gpu():
    bad = P.SparseMatrix(2, np.array([0, 1, 3]), np.array([1, 0, 1]), np.array([1.0, 1.0, 1.0]))
    bad.row_ptr[-1] = 5  # row_ptr[n] != nnz of the arrays handed over -> rejected on the host
    with pytest.raises(P.InvalidArgument):
        P.Context(P.SparseMatrix(2, np.array([1, 1, 1]), np.array([], np.int64), np.array([])), np.ones(2))
    with pytest.raises(P.InvalidArgument):
        P.Context(P.SparseMatrix.identity(3), np.ones(2))


def test_no_gpu_means_loud_cuda_error():
    if P.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(P.CudaError):
        P.Context(P.SparseMatrix.identity(2), np.ones(2))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1904_12754_b200")
    for dirpath, _d, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "expmc_oracle" not in src, f
