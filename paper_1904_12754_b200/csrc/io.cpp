// Host input pipeline: Matrix Market / vector readers and the canonical-CSR builder.
//
// Restates, with the reference's exact results and error messages:
//   read_matrix_market        io.cpp:69-128   coordinate real general|symmetric, 1-based,
//                                             line-numbered std::runtime_error messages
//   read_vector               io.cpp:154-167
//   SparseMatrix::from_triplets  sparse.cpp:12-49  sort by (row, col), duplicates summed,
//                                             zero sums dropped
// but multi-threaded: the file is parsed in newline-aligned chunks in parallel (line numbers
// recovered by a prefix sum of per-chunk line counts; the first error in file order wins), and
// the CSR is built by a stable bucket pass over rows plus per-row sorts.
//
// Duplicate summation order.  The reference sums the duplicates of an (i, j) key in the order
// std::sort leaves them, which is not the input order.  Two addends commute exactly, so the
// parallel build is bit-identical whenever no key occurs three or more times; if one does, the
// builder re-runs the reference's own algorithm (std::sort with the same comparator, the same
// standard library) on the original triplet sequence, so the result is bit-identical always.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <omp.h>

#include "internal.hpp"

using namespace expmc_b200;

namespace {

struct Triplet {  // sparse.hpp Triplet
    int64_t row, col;
    double value;
};

[[noreturn]] void fail_at(const std::string& path, size_t line, const std::string& what) {
    throw Status(EXPMC_EIO, path + ":" + std::to_string(line) + ": " + what);
}

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// split_ws (io.cpp:25-31): whitespace-separated tokens of one line, at most `cap` of them
// counted exactly (the caller only needs to know whether there are exactly 3).
struct Tokens {
    const char* b[4];
    const char* e[4];
    int count = 0;  // saturates at 4
};

inline Tokens split(const char* p, const char* end) {
    Tokens t;
    while (p < end) {
        while (p < end && is_ws(*p)) ++p;
        if (p >= end) break;
        const char* s = p;
        while (p < end && !is_ws(*p)) ++p;
        if (t.count < 4) {
            t.b[t.count] = s;
            t.e[t.count] = p;
        }
        if (t.count < 4) ++t.count;
    }
    return t;
}

std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

// parse_index / parse_double (io.cpp:40-54): std::from_chars over the whole token.
inline bool parse_index(const char* b, const char* e, int64_t& v) {
    const auto r = std::from_chars(b, e, v);
    return r.ec == std::errc{} && r.ptr == e;
}

inline bool parse_double(const char* b, const char* e, double& v) {
    const auto r = std::from_chars(b, e, v);
    return r.ec == std::errc{} && r.ptr == e;
}

std::string read_file(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw Status(EXPMC_EIO, "cannot open '" + path + "'");
    std::string s;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, got);
    std::fclose(f);
    return s;
}

// One line per std::getline call: [b, e) without the '\n'; returns false at the end.
inline bool next_line(const char*& p, const char* end, const char*& b, const char*& e) {
    if (p >= end) return false;
    b = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    e = nl ? nl : end;
    p = nl ? nl + 1 : end;
    return true;
}

// ------------------------------------------------------------------ from_triplets
void check_triplets(int64_t n, const std::vector<Triplet>& t) {  // sparse.cpp:13-19, first failure wins
    if (n < 0) throw Status(EXPMC_EINVAL, "matrix dimension must be nonnegative");
    const int64_t m = static_cast<int64_t>(t.size());
    int64_t bad = m;
#pragma omp parallel for schedule(static) reduction(min : bad)
    for (int64_t k = 0; k < m; ++k) {
        const Triplet& x = t[static_cast<size_t>(k)];
        if (x.row < 0 || x.row >= n || x.col < 0 || x.col >= n || !std::isfinite(x.value)) bad = std::min(bad, k);
    }
    if (bad < m) {
        const Triplet& x = t[static_cast<size_t>(bad)];
        if (x.row < 0 || x.row >= n || x.col < 0 || x.col >= n)
            throw Status(EXPMC_ERANGE, "triplet index outside [0, n)");
        throw Status(EXPMC_EINVAL, "matrix entry is NaN or Inf");
    }
}

// The reference's algorithm verbatim in structure: std::sort by (row, col), then one pass
// summing each key's run and dropping zero sums.
void from_triplets_sequential(int64_t n, std::vector<Triplet> t, expmc_matrix& m) {
    std::sort(t.begin(), t.end(),
              [](const Triplet& a, const Triplet& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
    m.n = n;
    m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    m.col.clear();
    m.val.clear();
    m.col.reserve(t.size());
    m.val.reserve(t.size());
    size_t k = 0;
    while (k < t.size()) {
        const int64_t i = t[k].row, j = t[k].col;
        double v = t[k].value;
        ++k;
        while (k < t.size() && t[k].row == i && t[k].col == j) v += t[k++].value;
        if (v != 0.0) {
            m.col.push_back(j);
            m.val.push_back(v);
            m.row_ptr[static_cast<size_t>(i) + 1] = static_cast<int64_t>(m.val.size());
        }
    }
    for (size_t i = 1; i <= static_cast<size_t>(n); ++i) m.row_ptr[i] = std::max(m.row_ptr[i], m.row_ptr[i - 1]);
}

// Parallel build; returns false (and leaves m unspecified) if some key has >= 3 entries.
// The bucket pass over rows is not stable (atomic slots): only the order inside a key's run
// could depend on it, and a run of two sums to the same value either way.
bool from_triplets_parallel(int64_t n, const std::vector<Triplet>& t, expmc_matrix& m) {
    const int64_t cnt = static_cast<int64_t>(t.size());
    std::vector<int64_t> start(static_cast<size_t>(n) + 1, 0);
    std::vector<int64_t> fill(static_cast<size_t>(n), 0);
    std::vector<Triplet> byrow(static_cast<size_t>(cnt));
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < cnt; ++k) {
#pragma omp atomic
        ++start[static_cast<size_t>(t[static_cast<size_t>(k)].row) + 1];
    }
    for (int64_t i = 0; i < n; ++i) start[static_cast<size_t>(i) + 1] += start[static_cast<size_t>(i)];
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < cnt; ++k) {
        const size_t r = static_cast<size_t>(t[static_cast<size_t>(k)].row);
        int64_t slot;
#pragma omp atomic capture
        slot = fill[r]++;
        byrow[static_cast<size_t>(start[r] + slot)] = t[static_cast<size_t>(k)];
    }
    std::vector<int64_t>().swap(fill);
    // per row: sort by column, count distinct nonzero sums, detect triple keys
    std::vector<int64_t> rowcnt(static_cast<size_t>(n) + 1, 0);
    int triple = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : triple)
    for (int64_t i = 0; i < n; ++i) {
        Triplet* b = byrow.data() + start[static_cast<size_t>(i)];
        Triplet* e = byrow.data() + start[static_cast<size_t>(i) + 1];
        std::sort(b, e, [](const Triplet& x, const Triplet& y) { return x.col < y.col; });
        int64_t c = 0;
        for (Triplet* p = b; p < e;) {
            Triplet* q = p + 1;
            while (q < e && q->col == p->col) ++q;
            if (q - p >= 3) triple = 1;
            const double v = (q - p == 2) ? p[0].value + p[1].value : p[0].value;
            if (v != 0.0) ++c;
            p = q;
        }
        rowcnt[static_cast<size_t>(i) + 1] = c;
    }
    if (triple) return false;
    m.n = n;
    m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    for (int64_t i = 0; i < n; ++i) m.row_ptr[static_cast<size_t>(i) + 1] = m.row_ptr[static_cast<size_t>(i)] + rowcnt[static_cast<size_t>(i) + 1];
    const size_t nnz = static_cast<size_t>(m.row_ptr[static_cast<size_t>(n)]);
    m.col.resize(nnz);
    m.val.resize(nnz);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
        const Triplet* b = byrow.data() + start[static_cast<size_t>(i)];
        const Triplet* e = byrow.data() + start[static_cast<size_t>(i) + 1];
        size_t o = static_cast<size_t>(m.row_ptr[static_cast<size_t>(i)]);
        for (const Triplet* p = b; p < e;) {
            const Triplet* q = p + 1;
            while (q < e && q->col == p->col) ++q;
            const double v = (q - p == 2) ? p[0].value + p[1].value : p[0].value;
            if (v != 0.0) {
                m.col[o] = p->col;
                m.val[o] = v;
                ++o;
            }
            p = q;
        }
    }
    return true;
}

void from_triplets(int64_t n, std::vector<Triplet>&& t, expmc_matrix& m) {
    check_triplets(n, t);
    if (!from_triplets_parallel(n, t, m)) from_triplets_sequential(n, std::move(t), m);
}

// ------------------------------------------------------------------ read_matrix_market
struct ChunkOut {
    std::vector<Triplet> trips;
    int64_t lines = 0;   // getline calls that returned a line
    int64_t seen = 0;    // entry lines
    int64_t err_line = -1;  // 0-based line within the chunk of the first error
    std::string err;
};

void parse_entries(const char* p, const char* end, bool symmetric, int64_t rows, ChunkOut& out) {
    const char *b, *e;
    while (next_line(p, end, b, e)) {
        const int64_t ln = out.lines++;
        if (b == e || *b == '%') continue;
        const Tokens tk = split(b, e);
        if (tk.count != 3) {
            out.err_line = ln;
            out.err = "expected 'i j value'";
            return;
        }
        int64_t i = 0, j = 0;
        double v = 0.0;
        if (!parse_index(tk.b[0], tk.e[0], i)) {
            out.err_line = ln;
            out.err = "expected an integer, got '" + std::string(tk.b[0], tk.e[0]) + "'";
            return;
        }
        if (!parse_index(tk.b[1], tk.e[1], j)) {
            out.err_line = ln;
            out.err = "expected an integer, got '" + std::string(tk.b[1], tk.e[1]) + "'";
            return;
        }
        if (!parse_double(tk.b[2], tk.e[2], v)) {
            out.err_line = ln;
            out.err = "expected a real number, got '" + std::string(tk.b[2], tk.e[2]) + "'";
            return;
        }
        if (i < 1 || i > rows || j < 1 || j > rows) {
            out.err_line = ln;
            out.err = "index (" + std::string(tk.b[0], tk.e[0]) + ", " + std::string(tk.b[1], tk.e[1]) +
                      ") outside 1.." + std::to_string(rows);
            return;
        }
        if (!std::isfinite(v)) {
            out.err_line = ln;
            out.err = "value is NaN or Inf";
            return;
        }
        out.trips.push_back({i - 1, j - 1, v});
        if (symmetric && i != j) out.trips.push_back({j - 1, i - 1, v});
        ++out.seen;
    }
}

void read_matrix_market_impl(const std::string& path, expmc_matrix& m) {
    const std::string data = read_file(path);
    const char* p = data.data();
    const char* end = p + data.size();
    const char *b, *e;
    size_t lineno = 1;
    bool symmetric = false;
    if (!next_line(p, end, b, e)) fail_at(path, 1, "empty file");
    // header (io.cpp:75-86)
    {
        const std::string header(b, e);
        std::vector<std::string> h;
        for (const char* q = header.data(); q < header.data() + header.size();) {
            while (q < header.data() + header.size() && is_ws(*q)) ++q;
            const char* s = q;
            while (q < header.data() + header.size() && !is_ws(*q)) ++q;
            if (q > s) h.emplace_back(s, q);
        }
        if (h.size() < 5 || lower(h[0]) != "%%matrixmarket" || lower(h[1]) != "matrix")
            fail_at(path, 1, "malformed Matrix Market header");
        if (lower(h[2]) != "coordinate") fail_at(path, 1, "only coordinate format is supported");
        const std::string field = lower(h[3]);
        if (field == "pattern") fail_at(path, 1, "pattern files carry no values: unsupported");
        if (field != "real") fail_at(path, 1, "only real matrices are supported");
        const std::string sym = lower(h[4]);
        if (sym != "general" && sym != "symmetric") fail_at(path, 1, "only general or symmetric symmetry is supported");
        symmetric = sym == "symmetric";
    }
    // size line (io.cpp:88-100)
    int64_t rows = 0, cols = 0, declared = 0;
    while (next_line(p, end, b, e)) {
        ++lineno;
        if (b == e || *b == '%') continue;
        const Tokens tk = split(b, e);
        if (tk.count != 3) fail_at(path, lineno, "expected 'rows cols nnz'");
        for (int q = 0; q < 3; ++q) {
            int64_t& dst = q == 0 ? rows : (q == 1 ? cols : declared);
            if (!parse_index(tk.b[q], tk.e[q], dst))
                fail_at(path, lineno, "expected an integer, got '" + std::string(tk.b[q], tk.e[q]) + "'");
        }
        break;
    }
    if (rows <= 0 || cols <= 0) fail_at(path, lineno, "missing or invalid size line");
    if (rows != cols)
        fail_at(path, lineno, "matrix is not square (" + std::to_string(rows) + "x" + std::to_string(cols) + ")");
    // entries (io.cpp:102-125): newline-aligned chunks parsed in parallel
    const size_t body = static_cast<size_t>(end - p);
    const int nt = std::max(1, std::min<int>(omp_get_max_threads(), static_cast<int>(body / (1 << 20)) + 1));
    std::vector<const char*> cut(static_cast<size_t>(nt) + 1);
    cut[0] = p;
    cut[static_cast<size_t>(nt)] = end;
    for (int c = 1; c < nt; ++c) {
        const char* q = p + body * static_cast<size_t>(c) / static_cast<size_t>(nt);
        q = std::max(q, cut[static_cast<size_t>(c) - 1]);
        const char* nl = q < end ? static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(end - q))) : nullptr;
        cut[static_cast<size_t>(c)] = nl ? nl + 1 : end;
    }
    std::vector<ChunkOut> out(static_cast<size_t>(nt));
#pragma omp parallel for schedule(static, 1) num_threads(nt)
    for (int c = 0; c < nt; ++c) {
        ChunkOut& o = out[static_cast<size_t>(c)];
        o.trips.reserve(static_cast<size_t>(cut[static_cast<size_t>(c) + 1] - cut[static_cast<size_t>(c)]) / 16);
        parse_entries(cut[static_cast<size_t>(c)], cut[static_cast<size_t>(c) + 1], symmetric, rows, o);
    }
    int64_t seen = 0;
    size_t total = 0;
    for (int c = 0; c < nt; ++c) {  // first error in file order
        const ChunkOut& o = out[static_cast<size_t>(c)];
        if (o.err_line >= 0) fail_at(path, lineno + static_cast<size_t>(o.err_line) + 1, o.err);
        lineno += static_cast<size_t>(o.lines);
        seen += o.seen;
        total += o.trips.size();
    }
    if (seen != declared)
        fail_at(path, lineno,
                "file declares " + std::to_string(declared) + " entries but has " + std::to_string(seen));
    std::vector<Triplet> trips(total);
    std::vector<size_t> off(static_cast<size_t>(nt) + 1, 0);
    for (int c = 0; c < nt; ++c) off[static_cast<size_t>(c) + 1] = off[static_cast<size_t>(c)] + out[static_cast<size_t>(c)].trips.size();
#pragma omp parallel for schedule(static, 1) num_threads(nt)
    for (int c = 0; c < nt; ++c) {
        std::copy(out[static_cast<size_t>(c)].trips.begin(), out[static_cast<size_t>(c)].trips.end(),
                  trips.begin() + static_cast<std::ptrdiff_t>(off[static_cast<size_t>(c)]));
        std::vector<Triplet>().swap(out[static_cast<size_t>(c)].trips);
    }
    from_triplets(rows, std::move(trips), m);
}

// read_vector (io.cpp:154-167)
std::vector<double> read_vector_impl(const std::string& path) {
    const std::string data = read_file(path);
    const char* p = data.data();
    const char* end = p + data.size();
    const char *b, *e;
    std::vector<double> v;
    size_t lineno = 0;
    while (next_line(p, end, b, e)) {
        ++lineno;
        if (b != e && *b == '%') continue;
        for (const char* q = b; q < e;) {
            while (q < e && is_ws(*q)) ++q;
            if (q >= e) break;
            const char* s = q;
            while (q < e && !is_ws(*q)) ++q;
            double x = 0.0;
            if (!parse_double(s, q, x)) fail_at(path, lineno, "expected a real number, got '" + std::string(s, q) + "'");
            v.push_back(x);
        }
    }
    if (v.empty()) throw Status(EXPMC_EIO, path + ": empty vector file");
    return v;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EXPMC_OK;
    } catch (const Status& s) {
        set_error(s.what());
        return s.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return EXPMC_EINTERNAL;
    } catch (const std::exception& e) {
        set_error(e.what());
        return EXPMC_EINTERNAL;
    }
}

}  // namespace

extern "C" {

int expmc_read_matrix_market(const char* path, expmc_matrix** out) {
    return guarded([&] {
        if (!path || !out) throw Status(EXPMC_EINVAL, "null argument");
        auto* m = new expmc_matrix;
        try {
            read_matrix_market_impl(path, *m);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

int expmc_read_vector(const char* path, int64_t cap, double* out, int64_t* n) {
    return guarded([&] {
        if (!path || !n || (cap > 0 && !out)) throw Status(EXPMC_EINVAL, "null argument");
        const std::vector<double> v = read_vector_impl(path);
        *n = static_cast<int64_t>(v.size());
        if (out && cap > 0) std::memcpy(out, v.data(), static_cast<size_t>(std::min<int64_t>(cap, *n)) * sizeof(double));
    });
}

int expmc_csr_from_triplets(int64_t n, int64_t count, const int64_t* rows, const int64_t* cols, const double* vals,
                            expmc_matrix** out) {
    return guarded([&] {
        if (!out || count < 0 || (count > 0 && (!rows || !cols || !vals))) throw Status(EXPMC_EINVAL, "null argument");
        std::vector<Triplet> t(static_cast<size_t>(count));
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < count; ++k) t[static_cast<size_t>(k)] = Triplet{rows[k], cols[k], vals[k]};
        auto* m = new expmc_matrix;
        try {
            from_triplets(n, std::move(t), *m);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

}  // extern "C"
