// Host-side input generators for the BASELINE configs C3-C5 and the spectral scale.
// Not on the hot path (netgen/io are host input code); native because C3/C4 are
// 10^7-10^9-entry graphs.  Every generator is deterministic in its seed.
//
//   expmc_gen_ba          Barabasi-Albert graph: the reference's `pref` algorithm
//                         (netgen.cpp:61-107: d-clique seed, each new node attaches to
//                         min(d, v) distinct nodes drawn from the endpoint list -- degree-
//                         proportional -- with stream_for(seed, 1, v, lane 3)), restated.
//   expmc_gen_rmat        R-MAT (Chakrabarti et al.) on 2^scale nodes, edge_factor * 2^scale
//                         edges, quadrant probabilities (a, b, c, 1-a-b-c), self-loops dropped,
//                         symmetrised, duplicates collapsed to weight 1.
//   expmc_gen_convdiff3d  7-point convection-diffusion on g^3 interior nodes: diag -6,
//                         off-diagonal 1, except along `axis` where the upwind neighbour is
//                         1 + Pe/2 and the downwind one 1 - Pe/2 (Pe = cell Peclet, C5).
//   expmc_power_iteration lambda_max estimate: x_0 = 1, x_{k+1} = A x_k / |A x_k|_2,
//                         lambda = |A x_k|_2 / |x_k|_2 after `iters` steps.
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "expmc_b200.h"
#include "internal.hpp"

using namespace expmc_b200;


namespace {

// Philox4x32-10 host stream, the reference's RngStream (rng.hpp:21-73).
struct HostStream {
    uint32_t k0, k1, c1, c2, c3, block = 0;
    uint64_t buf[2]{};
    int cached = 0;
    HostStream(uint64_t seed, uint32_t level, uint64_t sample, uint32_t lane)
        : k0(static_cast<uint32_t>(seed)),
          k1(static_cast<uint32_t>(seed >> 32)),
          c1(static_cast<uint32_t>(sample)),
          c2(static_cast<uint32_t>(sample >> 32)),
          c3((level & 0xFFFFFFu) | (lane << 24)) {}
    double next() {
        if (cached == 0) {
            uint32_t a = block++, b = c1, c = c2, d = c3, x = k0, y = k1;
            for (int r = 0; r < 10; ++r) {
                const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * a;
                const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c;
                const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ b ^ x;
                const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ d ^ y;
                b = static_cast<uint32_t>(p1);
                d = static_cast<uint32_t>(p0);
                a = n0;
                c = n2;
                x += 0x9E3779B9u;
                y += 0xBB67AE85u;
            }
            buf[0] = (static_cast<uint64_t>(a) << 32) | b;
            buf[1] = (static_cast<uint64_t>(c) << 32) | d;
            cached = 2;
        }
        return static_cast<double>(buf[--cached] >> 11) * 0x1.0p-53;
    }
};

constexpr uint32_t kGenLane = 3;   // netgen's lane (netgen.cpp:16)
constexpr uint32_t kRmatLane = 5;  // unused by the reference (lanes 0-3, 7)

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

// CSR from per-row neighbour lists (sorted, duplicates collapsed), all values `w`.
expmc_matrix* csr_from_lists(int64_t n, std::vector<std::vector<int64_t>>& nbrs, double w) {
    auto* m = new expmc_matrix;
    m->n = n;
    m->row_ptr.assign(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
        auto& l = nbrs[static_cast<size_t>(i)];
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
        m->row_ptr[static_cast<size_t>(i) + 1] = static_cast<int64_t>(l.size());
    }
    for (int64_t i = 0; i < n; ++i) m->row_ptr[static_cast<size_t>(i) + 1] += m->row_ptr[static_cast<size_t>(i)];
    m->col.resize(static_cast<size_t>(m->row_ptr.back()));
    m->val.assign(m->col.size(), w);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) {
        const auto& l = nbrs[static_cast<size_t>(i)];
        std::copy(l.begin(), l.end(), m->col.begin() + m->row_ptr[static_cast<size_t>(i)]);
    }
    return m;
}

}  // namespace

extern "C" {

int expmc_gen_ba(int64_t n, int64_t d, uint64_t seed, expmc_matrix** out) {
    return guarded([&] {
        if (n < 3) throw Status(EXPMC_EINVAL, "pref needs n >= 3");
        if (d < 1 || d >= n) throw Status(EXPMC_EINVAL, "pref needs 1 <= d < n");
        std::vector<std::vector<int64_t>> nbrs(static_cast<size_t>(n));
        std::vector<int64_t> endpoints;
        endpoints.reserve(2 * static_cast<size_t>(n) * static_cast<size_t>(d));
        for (int64_t i = 0; i < d; ++i)  // d-clique seed
            for (int64_t j = i + 1; j < d; ++j) {
                nbrs[static_cast<size_t>(i)].push_back(j);
                nbrs[static_cast<size_t>(j)].push_back(i);
                endpoints.push_back(i);
                endpoints.push_back(j);
            }
        std::vector<int64_t> picked;
        for (int64_t v = std::max<int64_t>(d, 1); v < n; ++v) {
            HostStream s(seed, 1, static_cast<uint64_t>(v), kGenLane);
            const size_t snapshot = endpoints.size();  // degrees frozen before v's edges
            picked.clear();
            const int64_t want = std::min(d, v);
            while (static_cast<int64_t>(picked.size()) < want) {
                int64_t t;
                if (snapshot == 0) {
                    t = static_cast<int64_t>(s.next() * static_cast<double>(v));
                    if (t >= v) t = v - 1;
                } else {
                    size_t pos = static_cast<size_t>(s.next() * static_cast<double>(snapshot));
                    if (pos >= snapshot) pos = snapshot - 1;
                    t = endpoints[pos];
                }
                if (std::find(picked.begin(), picked.end(), t) == picked.end()) picked.push_back(t);
            }
            for (int64_t t : picked) {
                nbrs[static_cast<size_t>(v)].push_back(t);
                nbrs[static_cast<size_t>(t)].push_back(v);
                endpoints.push_back(v);
                endpoints.push_back(t);
            }
        }
        *out = csr_from_lists(n, nbrs, 1.0);
    });
}

int expmc_gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                   expmc_matrix** out) {
    return guarded([&] {
        if (scale < 1 || scale > 30) throw Status(EXPMC_EINVAL, "R-MAT scale outside [1, 30]");
        if (edge_factor < 1) throw Status(EXPMC_EINVAL, "edge factor must be >= 1");
        if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) throw Status(EXPMC_EINVAL, "bad R-MAT probabilities");
        const int64_t n = int64_t{1} << scale;
        const int64_t m = edge_factor * n;
        const double ab = a + b, abc = a + b + c;
        auto edge = [&](int64_t e, int64_t& i, int64_t& j) {
            HostStream s(seed, 2, static_cast<uint64_t>(e), kRmatLane);
            i = j = 0;
            for (int32_t l = 0; l < scale; ++l) {
                const double u = s.next();
                const int bi = u >= ab;
                const int bj = (u >= a && u < ab) || u >= abc;
                i = (i << 1) | bi;
                j = (j << 1) | bj;
            }
        };
        // pass 1: degree of every row in the symmetrised multigraph (self-loops dropped)
        std::vector<std::atomic<uint32_t>> cnt(static_cast<size_t>(n));
        for (auto& x : cnt) x.store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < m; ++e) {
            int64_t i, j;
            edge(e, i, j);
            if (i == j) continue;
            cnt[static_cast<size_t>(i)].fetch_add(1, std::memory_order_relaxed);
            cnt[static_cast<size_t>(j)].fetch_add(1, std::memory_order_relaxed);
        }
        std::vector<int64_t> start(static_cast<size_t>(n) + 1, 0);
        for (int64_t i = 0; i < n; ++i) start[static_cast<size_t>(i) + 1] = start[static_cast<size_t>(i)] + cnt[static_cast<size_t>(i)].load();
        std::vector<uint32_t> cols(static_cast<size_t>(start.back()));
        std::vector<std::atomic<int64_t>> pos(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) pos[static_cast<size_t>(i)].store(start[static_cast<size_t>(i)], std::memory_order_relaxed);
        // pass 2: place both directions, then sort + dedupe each row (deterministic result)
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < m; ++e) {
            int64_t i, j;
            edge(e, i, j);
            if (i == j) continue;
            cols[static_cast<size_t>(pos[static_cast<size_t>(i)].fetch_add(1, std::memory_order_relaxed))] = static_cast<uint32_t>(j);
            cols[static_cast<size_t>(pos[static_cast<size_t>(j)].fetch_add(1, std::memory_order_relaxed))] = static_cast<uint32_t>(i);
        }
        std::vector<int64_t> uniq(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(dynamic, 4096)
        for (int64_t i = 0; i < n; ++i) {
            auto* b0 = cols.data() + start[static_cast<size_t>(i)];
            auto* b1 = cols.data() + start[static_cast<size_t>(i) + 1];
            std::sort(b0, b1);
            uniq[static_cast<size_t>(i) + 1] = std::unique(b0, b1) - b0;
        }
        auto* mat = new expmc_matrix;
        mat->n = n;
        mat->row_ptr.assign(static_cast<size_t>(n) + 1, 0);
        for (int64_t i = 0; i < n; ++i) mat->row_ptr[static_cast<size_t>(i) + 1] = mat->row_ptr[static_cast<size_t>(i)] + uniq[static_cast<size_t>(i) + 1];
        mat->col.resize(static_cast<size_t>(mat->row_ptr.back()));
        mat->val.assign(mat->col.size(), 1.0);
#pragma omp parallel for schedule(dynamic, 4096)
        for (int64_t i = 0; i < n; ++i) {
            const auto* b0 = cols.data() + start[static_cast<size_t>(i)];
            std::copy(b0, b0 + uniq[static_cast<size_t>(i) + 1], mat->col.begin() + mat->row_ptr[static_cast<size_t>(i)]);
        }
        *out = mat;
    });
}

int expmc_gen_convdiff3d(int64_t g, double peclet, int32_t axis, expmc_matrix** out) {
    return guarded([&] {
        if (g < 1 || g > 2048) throw Status(EXPMC_EINVAL, "grid size outside [1, 2048]");
        if (axis < 0 || axis > 2) throw Status(EXPMC_EINVAL, "velocity axis must be 0 (x), 1 (y) or 2 (z)");
        const int64_t n = g * g * g;
        auto* m = new expmc_matrix;
        m->n = n;
        m->row_ptr.assign(static_cast<size_t>(n) + 1, 0);
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            const int64_t x = r % g, y = (r / g) % g, z = r / (g * g);
            m->row_ptr[static_cast<size_t>(r) + 1] = 1 + (x > 0) + (x + 1 < g) + (y > 0) + (y + 1 < g) + (z > 0) + (z + 1 < g);
        }
        for (int64_t r = 0; r < n; ++r) m->row_ptr[static_cast<size_t>(r) + 1] += m->row_ptr[static_cast<size_t>(r)];
        m->col.resize(static_cast<size_t>(m->row_ptr.back()));
        m->val.resize(m->col.size());
        const double up = 1.0 + 0.5 * peclet, down = 1.0 - 0.5 * peclet;
        const int64_t stride[3] = {1, g, g * g};
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            const int64_t c3[3] = {r % g, (r / g) % g, r / (g * g)};
            int64_t k = m->row_ptr[static_cast<size_t>(r)];
            // ascending column order: -z, -y, -x, self, +x, +y, +z
            for (int dim = 2; dim >= 0; --dim)
                if (c3[dim] > 0) {
                    m->col[static_cast<size_t>(k)] = r - stride[dim];
                    m->val[static_cast<size_t>(k++)] = dim == axis ? up : 1.0;  // upwind neighbour
                }
            m->col[static_cast<size_t>(k)] = r;
            m->val[static_cast<size_t>(k++)] = -6.0;
            for (int dim = 0; dim <= 2; ++dim)
                if (c3[dim] + 1 < g) {
                    m->col[static_cast<size_t>(k)] = r + stride[dim];
                    m->val[static_cast<size_t>(k++)] = dim == axis ? down : 1.0;  // downwind neighbour
                }
        }
        *out = m;
    });
}

int expmc_matrix_info(const expmc_matrix* m, int64_t* n, int64_t* nnz) {
    return guarded([&] {
        if (!m || !n || !nnz) throw Status(EXPMC_EINVAL, "null argument");
        *n = m->n;
        *nnz = static_cast<int64_t>(m->col.size());
    });
}

int expmc_matrix_copy(const expmc_matrix* m, int64_t* row_ptr, int64_t* col, double* val) {
    return guarded([&] {
        if (!m) throw Status(EXPMC_EINVAL, "null matrix");
        if (row_ptr) std::memcpy(row_ptr, m->row_ptr.data(), m->row_ptr.size() * sizeof(int64_t));
        if (col) std::memcpy(col, m->col.data(), m->col.size() * sizeof(int64_t));
        if (val) std::memcpy(val, m->val.data(), m->val.size() * sizeof(double));
    });
}

void expmc_matrix_destroy(expmc_matrix* m) { delete m; }

int expmc_power_iteration(const expmc_csr* A, int32_t iters, double* lambda) {
    return guarded([&] {
        if (!A || !lambda || iters < 1) throw Status(EXPMC_EINVAL, "bad power-iteration arguments");
        const int64_t n = A->n;
        std::vector<double> x(static_cast<size_t>(n), 1.0), y(static_cast<size_t>(n));
        double lam = 0.0, xn = std::sqrt(static_cast<double>(n));
        for (int32_t it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                double acc = 0.0;
                for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) acc += A->val[k] * x[static_cast<size_t>(A->col[k])];
                y[static_cast<size_t>(i)] = acc;
            }
            double s = 0.0;  // sequential: lambda (hence beta) must not depend on the thread count
            for (int64_t i = 0; i < n; ++i) s += y[static_cast<size_t>(i)] * y[static_cast<size_t>(i)];
            const double yn = std::sqrt(s);
            lam = yn / xn;
            if (!(yn > 0.0)) break;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; ++i) x[static_cast<size_t>(i)] = y[static_cast<size_t>(i)] / yn;
            xn = 1.0;
        }
        *lambda = lam;
    });
}

}  // extern "C"
