"""Host input pipeline (csrc/io.cpp, no GPU): the native multi-threaded Matrix Market reader,
vector reader and canonical-CSR builder against the reference's own read_matrix_market
(io.cpp:69-128), read_vector (io.cpp:154-167) and SparseMatrix::from_triplets
(sparse.cpp:12-49), compiled in place (oracle/_ref).  Results must be bit-identical and error
messages identical ("path:line: what", std::runtime_error -> IoError).

Inputs are generated here (seeded): general and symmetric files, comments, blank and CRLF
lines, duplicate keys (pairs and runs of three or more, which take the reference's own sort),
entries cancelling to zero, files large enough to be parsed in many chunks, and each of the
reader's error paths, placed in late chunks so the line numbers cross chunk boundaries.
"""
import os

import numpy as np
import pytest

import paper_1904_12754_b200 as P
from oracle import OracleError, have_reference

needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle import Reference

    return Reference()


def write_mm(path, n, entries, symmetric=False, comments=(), crlf=False, header=None, size_line=None):
    nl = "\r\n" if crlf else "\n"
    lines = [header or f"%%MatrixMarket matrix coordinate real {'symmetric' if symmetric else 'general'}"]
    lines += [f"% {c}" for c in comments]
    lines.append(size_line if size_line is not None else f"{n} {n} {len(entries)}")
    for (i, j, v) in entries:
        lines.append(f"{i} {j} {v if isinstance(v, str) else repr(float(v))}")
    with open(path, "w", newline="") as f:
        f.write(nl.join(lines) + nl)
    return str(path)


def same(a: P.SparseMatrix, r):
    return (a.n == r.n and np.array_equal(a.row_ptr, r.a.row_ptr) and np.array_equal(a.col, r.a.col)
            and np.array_equal(a.val.view(np.int64), r.a.val.view(np.int64)))


def random_entries(rng, n, m, dup_frac=0.1, triple_frac=0.0):
    i = rng.integers(1, n + 1, m)
    j = rng.integers(1, n + 1, m)
    v = rng.standard_normal(m) * 10.0 ** rng.integers(-3, 4, m)
    ent = list(zip(i.tolist(), j.tolist(), v.tolist()))
    k = int(dup_frac * m)
    for t in range(k):  # duplicate pairs (and a cancelling pair now and then)
        a = ent[rng.integers(0, m)]
        ent.append((a[0], a[1], -a[2] if t % 7 == 0 else float(rng.standard_normal())))
    for t in range(int(triple_frac * m)):  # runs of three or more
        a = ent[rng.integers(0, m)]
        for _ in range(int(rng.integers(2, 5))):
            ent.append((a[0], a[1], float(rng.standard_normal() * 1e3)))
    order = rng.permutation(len(ent))
    return [ent[q] for q in order]


@needs_ref
@pytest.mark.parametrize("symmetric", [False, True])
@pytest.mark.parametrize("triples", [0.0, 0.02])
def test_read_matrix_market_bitwise(tmp_path, ref, symmetric, triples):
    rng = np.random.default_rng(7 + int(symmetric) + int(100 * triples))
    n = 3000
    ent = random_entries(rng, n, 120000, triple_frac=triples)
    if symmetric:
        ent = [(max(i, j), min(i, j), v) for (i, j, v) in ent]
    path = write_mm(tmp_path / "a.mtx", n, ent, symmetric, comments=["seeded", ""])
    got = P.read_matrix_market(path)
    assert same(got, ref.read_matrix_market(path))


@needs_ref
def test_read_matrix_market_layout_variants(tmp_path, ref):
    rng = np.random.default_rng(3)
    ent = random_entries(rng, 50, 400)
    for k, kw in enumerate([dict(crlf=True), dict(comments=["a", "b", "c"]),
                            dict(header="%%MATRIXMARKET Matrix Coordinate REAL General extra")]):
        path = write_mm(tmp_path / f"v{k}.mtx", 50, ent, **kw)
        assert same(P.read_matrix_market(path), ref.read_matrix_market(path))
    # blank lines and comment lines between entries; tabs and leading spaces
    lines = ["%%MatrixMarket matrix coordinate real general", "", "% c", "4 4 3", "1 1 2.5", "", "%x",
             "  2\t3   -1e-3", "4 4 7", ""]
    path = tmp_path / "blank.mtx"
    path.write_text("\n".join(lines))
    assert same(P.read_matrix_market(str(path)), ref.read_matrix_market(str(path)))


def _ref_error(ref, fn, path):
    with pytest.raises(OracleError) as e:
        fn(path)
    return str(e.value)


@needs_ref
def test_read_matrix_market_errors_match(tmp_path, ref):
    rng = np.random.default_rng(5)
    big = random_entries(rng, 400, 60000, dup_frac=0.0)  # ~1.5 MB: several parse chunks
    cases = {
        "empty": "",
        "header": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
        "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
        "pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
        "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
        "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
        "short": "%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1\n",
        "nosize": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
        "badsize": "%%MatrixMarket matrix coordinate real general\n3 3\n",
        "sizetok": "%%MatrixMarket matrix coordinate real general\n3 x 1\n1 1 1\n",
        "zero": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
        "rect": "%%MatrixMarket matrix coordinate real general\n3 4 1\n1 1 1\n",
        "count": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n",
        "toomany": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 1\n2 2 2\n",
        "range": "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n",
        "range0": "%%MatrixMarket matrix coordinate real general\n3 3 1\n0 1 1\n",
        "real": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 abc\n",
        "int": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1.0 1 1\n",
        "plus": "%%MatrixMarket matrix coordinate real general\n3 3 1\n+1 1 1\n",
        "nan": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 nan\n",
        "inf": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 -inf\n",
        "fields": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 1 1\n",
        "spaces": "%%MatrixMarket matrix coordinate real general\n3 3 1\n   \n1 1 1\n",
        "crlfblank": "%%MatrixMarket matrix coordinate real general\r\n3 3 1\r\n\r\n1 1 1\r\n",
    }
    for name, text in cases.items():
        path = tmp_path / f"{name}.mtx"
        path.write_bytes(text.encode())
        msg = _ref_error(ref, ref.read_matrix_market, str(path))
        with pytest.raises(P.IoError) as e:
            P.read_matrix_market(str(path))
        assert str(e.value) == msg, name
    # errors deep in a large file: the reported line must cross the chunk boundaries
    for pos, bad in [(45000, "x 1 1"), (59000, "1 1 1 1"), (30001, "401 2 1")]:
        ent = list(big)
        ent[pos] = tuple(bad.split()) if bad.count(" ") == 2 else ent[pos]
        path = write_mm(tmp_path / "big.mtx", 400, ent)
        if bad.count(" ") != 2:
            lines = open(path).read().split("\n")
            lines[pos + 2] = bad
            open(path, "w").write("\n".join(lines))
        msg = _ref_error(ref, ref.read_matrix_market, path)
        with pytest.raises(P.IoError) as e:
            P.read_matrix_market(path)
        assert str(e.value) == msg
    with pytest.raises(P.IoError, match="cannot open"):
        P.read_matrix_market(str(tmp_path / "missing.mtx"))


@needs_ref
def test_from_triplets_bitwise_with_long_duplicate_runs(ref):
    rng = np.random.default_rng(11)
    n, m = 500, 40000
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    v = rng.standard_normal(m) * 10.0 ** rng.integers(-8, 9, m)
    # long runs on a few keys: the sum order is the reference's std::sort order
    hot = rng.integers(0, m, 50)
    r = np.concatenate([r, np.repeat(r[hot], 6)])
    c = np.concatenate([c, np.repeat(c[hot], 6)])
    v = np.concatenate([v, rng.standard_normal(300) * 1e6])
    perm = rng.permutation(r.size)
    r, c, v = r[perm], c[perm], v[perm]
    assert same(P.SparseMatrix.from_triplets(n, r, c, v), ref.from_triplets(n, r, c, v))
    # pairs only (the parallel path) and cancellation to zero
    r2 = np.concatenate([np.arange(n), np.arange(n)])
    c2 = np.concatenate([np.arange(n)[::-1], np.arange(n)[::-1]])
    v2 = np.concatenate([np.ones(n), -np.ones(n)])
    v2[:10] = 2.0
    assert same(P.SparseMatrix.from_triplets(n, r2, c2, v2), ref.from_triplets(n, r2, c2, v2))


def test_from_triplets_errors_and_empty():
    with pytest.raises(P.OutOfRange, match="outside"):
        P.SparseMatrix.from_triplets(3, [0, 3], [0, 0], [1.0, 1.0])
    with pytest.raises(P.InvalidArgument, match="NaN or Inf"):
        P.SparseMatrix.from_triplets(3, [0, 1], [0, 0], [np.inf, 1.0])
    with pytest.raises(P.InvalidArgument, match="nonnegative"):
        P.SparseMatrix.from_triplets(-1, [], [], [])
    # the first failing triplet decides the error type
    with pytest.raises(P.InvalidArgument):
        P.SparseMatrix.from_triplets(3, [0, 5], [0, 0], [np.nan, 1.0])
    e = P.SparseMatrix.from_triplets(4, [], [], [])
    assert e.n == 4 and e.nnz == 0 and np.array_equal(e.row_ptr, np.zeros(5))


@needs_ref
def test_read_vector_and_fem_system(tmp_path, ref):
    rng = np.random.default_rng(2)
    x = rng.standard_normal(5000)
    p = tmp_path / "v.txt"
    p.write_text("% header\n" + "\n".join(" ".join(repr(float(t)) for t in x[k:k + 3]) for k in range(0, 5000, 3)) + "\n")
    got = P.read_vector(str(p))
    assert np.array_equal(got.view(np.int64), ref.read_vector(str(p)).view(np.int64))
    assert np.array_equal(got, x)
    for name, text in {"empty": "% nothing\n", "bad": "1.0\n2.0 x\n"}.items():
        q = tmp_path / f"{name}.txt"
        q.write_text(text)
        msg = _ref_error(ref, ref.read_vector, str(q))
        with pytest.raises(P.IoError) as e:
            P.read_vector(str(q))
        assert str(e.value) == msg
    # a lumped FEM system (fem.cpp:12-37) written out and read back both ways
    n = 40
    md = rng.uniform(0.5, 2.0, n)
    k_ent = [(i + 1, i + 1, 2.0 + rng.random()) for i in range(n)] + \
            [(i + 1, (i + 1) % n + 1, -0.5 * rng.random()) for i in range(n)]
    files = dict(mass=write_mm(tmp_path / "m.mtx", n, [(i + 1, i + 1, md[i]) for i in range(n)]),
                 stiffness=write_mm(tmp_path / "k.mtx", n, k_ent))
    for nm in ("load", "u0"):
        f = tmp_path / f"{nm}.txt"
        f.write_text("\n".join(repr(float(t)) for t in rng.standard_normal(n)) + "\n")
        files[nm] = str(f)
    sysm = P.load_fem_system(files["mass"], files["stiffness"], files["load"], files["u0"])
    exp = ref.load_fem_system(files["mass"], files["stiffness"], files["load"], files["u0"])
    assert np.array_equal(sysm.mass_diag, exp["mass_diag"]) and np.array_equal(sysm.load, exp["load"])
    assert np.array_equal(sysm.u0, exp["u0"]) and np.array_equal(sysm.stiffness.val, exp["stiffness"].val)
    bad = write_mm(tmp_path / "bad_mass.mtx", n, [(i + 1, i + 1, md[i]) for i in range(n)] + [(1, 2, 0.1)])
    with pytest.raises(P.InvalidArgument, match="not lumped"):
        P.load_fem_system(bad, files["stiffness"], files["load"], files["u0"])
    neg = write_mm(tmp_path / "neg_mass.mtx", n, [(i + 1, i + 1, -md[i]) for i in range(n)])
    with pytest.raises(P.InvalidArgument, match="positive"):
        P.load_fem_system(neg, files["stiffness"], files["load"], files["u0"])
    short = tmp_path / "short.txt"
    short.write_text("1.0\n")
    with pytest.raises(P.InvalidArgument, match="disagree"):
        P.load_fem_system(files["mass"], files["stiffness"], str(short), files["u0"])
