"""CPU: the config input generators (csrc/gen.cpp) -- BA equals the reference's pref bit for bit
(golden pref(300, 3, 7) and, when oracle/_ref is built, larger instances), R-MAT / 3-D
convection-diffusion structure, power iteration vs numpy."""
import numpy as np
import pytest

from oracle import have_reference
from paper_1904_12754_b200 import configs


def test_ba_equals_reference_pref_golden(golden):
    m = golden["matrices"]["pref300"]["csr"]
    a = configs.gen_ba(300, 3, 7)
    assert np.array_equal(a.row_ptr, np.array(m["row_ptr"])) and np.array_equal(a.col, np.array(m["col"]))
    assert np.all(a.val == 1.0)


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")
def test_ba_equals_reference_pref_large():
    from oracle import Reference

    for (n, d, seed) in [(5000, 5, 1), (2000, 1, 3), (1500, 7, 11)]:
        a = configs.gen_ba(n, d, seed)
        r = Reference().pref(n, d, seed).a
        assert np.array_equal(a.row_ptr, r.row_ptr) and np.array_equal(a.col, r.col) and np.array_equal(a.val, r.val)


def test_ba_c3_shape():
    a = configs.gen_ba(100_000, 5, 1)
    assert a.nnz == 2 * (10 + 5 * (100_000 - 5))  # clique (10 edges) + 5 per node, both directions
    deg = np.diff(a.row_ptr)
    assert deg.min() >= 5 and deg.max() > 200


def test_rmat_properties():
    a = configs.gen_rmat(12, 16, seed=3)
    n = 1 << 12
    assert a.n == n and np.all(a.val == 1.0)
    r = np.repeat(np.arange(n), np.diff(a.row_ptr))
    assert not np.any(r == a.col)  # no self loops
    key = set(zip(r.tolist(), a.col.tolist()))
    assert all((j, i) in key for (i, j) in list(key)[:20000])  # symmetric
    assert a.nnz <= 2 * 16 * n
    for i in range(0, n, 97):  # sorted, duplicate-free rows
        c = a.col[a.row_ptr[i]:a.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    b = configs.gen_rmat(12, 16, seed=3)
    assert np.array_equal(a.col, b.col)  # deterministic across thread schedules


def test_convdiff3d_structure():
    g = 5
    a = configs.gen_convdiff3d(g, 10.0, 0)
    n = g ** 3
    dense = np.zeros((n, n))
    for z in range(g):
        for y in range(g):
            for x in range(g):
                r = (z * g + y) * g + x
                dense[r, r] = -6.0
                for (dx, dy, dz, w) in [(-1, 0, 0, 6.0), (1, 0, 0, -4.0), (0, -1, 0, 1.0), (0, 1, 0, 1.0),
                                        (0, 0, -1, 1.0), (0, 0, 1, 1.0)]:
                    xx, yy, zz = x + dx, y + dy, z + dz
                    if 0 <= xx < g and 0 <= yy < g and 0 <= zz < g:
                        dense[r, (zz * g + yy) * g + xx] = w
    got = np.zeros((n, n))
    r = np.repeat(np.arange(n), np.diff(a.row_ptr))
    got[r, a.col] = a.val
    assert np.array_equal(got, dense)


def test_power_iteration_matches_numpy():
    a = configs.gen_ba(3000, 3, 5)
    lam = configs.power_iteration(a, 50)
    d = np.zeros((a.n, a.n))
    d[np.repeat(np.arange(a.n), np.diff(a.row_ptr)), a.col] = a.val
    x = np.ones(a.n)
    for _ in range(50):
        y = d @ x
        lam_np = np.linalg.norm(y) / np.linalg.norm(x)
        x = y / np.linalg.norm(y)
    assert lam == pytest.approx(lam_np, rel=1e-12)
    assert lam <= np.linalg.eigvalsh(d)[-1] * (1 + 1e-12)
