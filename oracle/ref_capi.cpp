// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/core),
// compiled in place by oracle/Makefile into oracle/_ref/libexpmc_ref.so.  It lets the
// Python tests, the golden-vector generator and bench.py's CPU baseline call the
// reference's own code path:
//   RngStream / stream_for          rng.hpp:21-79
//   decompose                       chain.cpp:75 -> decompose_impl chain.cpp:15-71
//   LevelSampler::single / coupled  paths.cpp:84-141
//   run_level                       mlmc.cpp:163-168 (run_level_ex 76-148)
//   mlmc_driver                     mlmc.cpp:170-260
//   dense_expmv / strang_reference  oracle.cpp:31-60, 79-99
//   smallw / pref                   netgen.cpp:30-107
//   forward mode                    paths.cpp:12-36, 144-181
//   fem mode, decompose_scaled,     paths.cpp:183-245, chain.cpp:80-85, mlmc.cpp:66-75,
//     solve_convdiff_point, io        fem.cpp:10-73, io.cpp:69-167
// Exceptions map to status codes: 1 invalid_argument, 2 out_of_range, 3 domain_error, 9 other.

#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "expmc/chain.hpp"
#include "expmc/communicability.hpp"
#include "expmc/fem.hpp"
#include "expmc/io.hpp"
#include "expmc/harness.hpp"
#include "expmc/mc.hpp"
#include "expmc/mlmc.hpp"
#include "expmc/netgen.hpp"
#include "expmc/oracle.hpp"
#include "expmc/paths.hpp"
#include "expmc/rng.hpp"
#include "expmc/sparse.hpp"

using namespace expmc;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

struct RefMatrix {
    SparseMatrix a;
    ChainDecomposition dec;
};

SparseMatrix from_csr(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val) {
    std::vector<Triplet> trips;
    trips.reserve(static_cast<std::size_t>(row_ptr[n]));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) trips.push_back({i, col[k], val[k]});
    return SparseMatrix::from_triplets(n, std::move(trips));
}

void export_csr(const SparseMatrix& m, int64_t* row_ptr, int64_t* col, double* val) {
    const auto rp = m.row_ptr();
    const auto ci = m.col_idx();
    const auto vv = m.values();
    std::memcpy(row_ptr, rp.data(), rp.size() * sizeof(int64_t));
    std::memcpy(col, ci.data(), ci.size() * sizeof(int64_t));
    std::memcpy(val, vv.data(), vv.size() * sizeof(double));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_uniforms(uint64_t seed, uint32_t level, uint64_t sample, uint32_t lane, int64_t count,
                  double* out) {
    RngStream s = stream_for(seed, level, sample, lane);
    for (int64_t i = 0; i < count; ++i) out[i] = s.next_uniform();
}

int ref_matrix_create(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                      void** out) {
    return guarded([&] {
        auto* m = new RefMatrix;
        try {
            m->a = from_csr(n, row_ptr, col, val);
            m->dec = decompose(m->a);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

void ref_matrix_destroy(void* h) { delete static_cast<RefMatrix*>(h); }

// sizes: n, nnz of the canonical CSR, number of chain edges
void ref_matrix_sizes(void* h, int64_t* n, int64_t* nnz, int64_t* edges) {
    auto* m = static_cast<RefMatrix*>(h);
    *n = m->a.size();
    *nnz = m->a.nnz();
    *edges = static_cast<int64_t>(m->dec.jump_target.size());
}

void ref_matrix_csr(void* h, int64_t* row_ptr, int64_t* col, double* val) {
    export_csr(static_cast<RefMatrix*>(h)->a, row_ptr, col, val);
}

void ref_matrix_decomposition(void* h, double* d, double* rate, int64_t* row_ptr, double* cdf,
                              int64_t* target, uint8_t* sign, double* weight, double* d_max,
                              double* d_bar) {
    const ChainDecomposition& dec = static_cast<RefMatrix*>(h)->dec;
    std::memcpy(d, dec.d.data(), dec.d.size() * sizeof(double));
    std::memcpy(rate, dec.rate.data(), dec.rate.size() * sizeof(double));
    std::memcpy(row_ptr, dec.row_ptr.data(), dec.row_ptr.size() * sizeof(int64_t));
    std::memcpy(cdf, dec.jump_cdf.data(), dec.jump_cdf.size() * sizeof(double));
    std::memcpy(target, dec.jump_target.data(), dec.jump_target.size() * sizeof(int64_t));
    std::memcpy(sign, dec.sign.data(), dec.sign.size());
    std::memcpy(weight, dec.jump_weight.data(), dec.jump_weight.size() * sizeof(double));
    *d_max = dec.d_max;
    *d_bar = dec.d_bar;
}

// Per-sample functionals through LevelSampler (paths.cpp:99-141), entry mode,
// stream_for(seed, level, sample_idx[i], lane).  base != 0 -> single (value in fine,
// coarse = 0), else coupled.
int ref_samples(void* h, const double* u, int64_t entry, double beta, int level, int base,
                uint64_t seed, uint32_t lane, int64_t count, const uint64_t* sample_idx,
                double* fine, double* coarse, uint64_t* cost) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        const index_t steps = index_t{1} << level;
        const double dt = beta / static_cast<double>(steps);
        const LevelSampler sampler(m->dec, dt, steps);
        const std::span<const double> uu(u, static_cast<std::size_t>(m->dec.n));
        for (int64_t i = 0; i < count; ++i) {
            RngStream s = stream_for(seed, static_cast<uint32_t>(level), sample_idx[i], lane);
            if (base) {
                const FunctionalSample f = sampler.single(uu, entry, s);
                fine[i] = f.value;
                coarse[i] = 0.0;
                cost[i] = f.cost;
            } else {
                const CoupledSample c = sampler.coupled(uu, entry, s);
                fine[i] = c.eta_fine;
                coarse[i] = c.eta_coarse;
                cost[i] = c.cost;
            }
        }
    });
}

// run_level (mlmc.hpp:86-88), entry mode.
int ref_run_level(void* h, const double* u, int64_t entry, double beta, int level, int base,
                  uint64_t first, uint64_t count, uint64_t seed, int threads, double* sum,
                  double* sum_sq, uint64_t* samples, uint64_t* cost) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.entry = entry;
        p.beta = beta;
        const LevelStats st = run_level(p, level, base != 0, first, count, seed, threads);
        *sum = st.sum;
        *sum_sq = st.sum_sq;
        *samples = st.samples;
        *cost = st.cost;
    });
}

struct RefOptions {
    double epsilon;
    uint64_t seed;
    int32_t threads;
    int32_t l0_override;
    uint64_t warmup;
    int32_t max_levels_above_l0;
    int32_t max_iterations;
};

struct RefResult {
    double estimate;
    double statistical_error;
    double bias_estimate;
    int32_t l0;
    int32_t L;
    uint64_t total_cost;
    int32_t converged;
    int32_t nlevels;
};

struct RefLevel {
    int32_t level;
    int32_t pad;
    double sum;
    double sum_sq;
    uint64_t samples;
    uint64_t cost;
};

// mlmc_driver (mlmc.cpp:170-260) for each row of `rows`, row r with seed row_seed[r].
// levels_out: nrows x max_levels records (nullable).
int ref_mlmc_driver_rows(void* h, const double* u, double beta, const RefOptions* o, int64_t nrows,
                         const int64_t* rows, const uint64_t* row_seed, RefResult* out,
                         RefLevel* levels_out, int32_t max_levels) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.beta = beta;
        MlmcOptions opt;
        opt.epsilon = o->epsilon;
        opt.threads = o->threads;
        opt.l0_override = o->l0_override;
        opt.warmup = o->warmup;
        opt.max_levels_above_l0 = o->max_levels_above_l0;
        opt.max_iterations = o->max_iterations;
        for (int64_t r = 0; r < nrows; ++r) {
            p.entry = rows[r];
            opt.seed = row_seed[r];
            const MlmcResult res = mlmc_driver(p, opt);
            RefResult& q = out[r];
            q.estimate = res.estimate;
            q.statistical_error = res.statistical_error;
            q.bias_estimate = res.bias_estimate;
            q.l0 = res.l0;
            q.L = res.L;
            q.total_cost = res.total_cost;
            q.converged = res.converged ? 1 : 0;
            q.nlevels = static_cast<int32_t>(res.levels.size());
            if (levels_out) {
                for (std::size_t l = 0; l < res.levels.size() && l < static_cast<std::size_t>(max_levels); ++l) {
                    RefLevel& lv = levels_out[r * max_levels + static_cast<int64_t>(l)];
                    lv.level = res.levels[l].level;
                    lv.pad = 0;
                    lv.sum = res.levels[l].sum;
                    lv.sum_sq = res.levels[l].sum_sq;
                    lv.samples = res.levels[l].samples;
                    lv.cost = res.levels[l].cost;
                }
            }
        }
    });
}

// Forward mode (SampleMode::forward, mlmc.cpp:86,112-121; paths.cpp:12-36,143-181): the matrix
// handle must hold A^T; stream lane 1.
int ref_forward_samples(void* h, const double* u, double beta, int level, int base, uint64_t seed, int64_t count,
                        const uint64_t* sample_idx, double* fine, double* coarse, uint64_t* cost) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        const index_t steps = index_t{1} << level;
        const double dt = beta / static_cast<double>(steps);
        const LevelSampler sampler(m->dec, dt, steps);
        const InitialDistribution init =
            make_initial_distribution(std::span<const double>(u, static_cast<std::size_t>(m->dec.n)));
        for (int64_t i = 0; i < count; ++i) {
            RngStream s = stream_for(seed, static_cast<uint32_t>(level), sample_idx[i], 1u);
            if (base) {
                const FunctionalSample f = sampler.forward_single(init, s);
                fine[i] = f.value;
                coarse[i] = 0.0;
                cost[i] = f.cost;
            } else {
                const CoupledSample c = sampler.forward_coupled(init, s);
                fine[i] = c.eta_fine;
                coarse[i] = c.eta_coarse;
                cost[i] = c.cost;
            }
        }
    });
}

int ref_forward_run_level(void* h, const double* u, double beta, int level, int base, uint64_t first,
                          uint64_t count, uint64_t seed, int threads, double* sum, double* sum_sq, uint64_t* samples,
                          uint64_t* cost) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.beta = beta;
        p.mode = SampleMode::forward;
        const LevelStats st = run_level(p, level, base != 0, first, count, seed, threads);
        *sum = st.sum;
        *sum_sq = st.sum_sq;
        *samples = st.samples;
        *cost = st.cost;
    });
}

int ref_forward_driver(void* h, const double* u, double beta, const RefOptions* o, RefResult* out,
                       RefLevel* levels_out, int32_t max_levels) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.beta = beta;
        p.mode = SampleMode::forward;
        MlmcOptions opt;
        opt.epsilon = o->epsilon;
        opt.seed = o->seed;
        opt.threads = o->threads;
        opt.l0_override = o->l0_override;
        opt.warmup = o->warmup;
        opt.max_levels_above_l0 = o->max_levels_above_l0;
        opt.max_iterations = o->max_iterations;
        const MlmcResult res = mlmc_driver(p, opt);
        out->estimate = res.estimate;
        out->statistical_error = res.statistical_error;
        out->bias_estimate = res.bias_estimate;
        out->l0 = res.l0;
        out->L = res.L;
        out->total_cost = res.total_cost;
        out->converged = res.converged ? 1 : 0;
        out->nlevels = static_cast<int32_t>(res.levels.size());
        for (std::size_t l = 0; levels_out && l < res.levels.size() && l < static_cast<std::size_t>(max_levels); ++l) {
            levels_out[l].level = res.levels[l].level;
            levels_out[l].pad = 0;
            levels_out[l].sum = res.levels[l].sum;
            levels_out[l].sum_sq = res.levels[l].sum_sq;
            levels_out[l].samples = res.levels[l].samples;
            levels_out[l].cost = res.levels[l].cost;
        }
    });
}

int ref_transpose(void* h, void** out) {
    return guarded([&] {
        auto* m = new RefMatrix;
        m->a = static_cast<RefMatrix*>(h)->a.transposed();
        m->dec = decompose(m->a);
        *out = m;
    });
}

int ref_initial_level(double beta, double d_max, int* out) {
    return guarded([&] { *out = initial_level(beta, d_max); });
}

int ref_optimal_allocation(int64_t n, const double* v, const double* c, double eps, uint64_t* out) {
    return guarded([&] {
        const auto m = optimal_allocation(std::span<const double>(v, static_cast<std::size_t>(n)),
                                          std::span<const double>(c, static_cast<std::size_t>(n)), eps);
        for (std::size_t i = 0; i < m.size(); ++i) out[i] = m[i];
    });
}

int ref_bias_estimate(int64_t n, const double* means, double* out) {
    return guarded([&] { *out = bias_estimate(std::span<const double>(means, static_cast<std::size_t>(n))); });
}

int ref_dense_expmv(void* h, const double* u, double beta, double* out) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        const auto x = dense_expmv(m->a, std::span<const double>(u, static_cast<std::size_t>(m->a.size())), beta);
        std::memcpy(out, x.data(), x.size() * sizeof(double));
    });
}

int ref_strang_reference(void* h, const double* u, double beta, int64_t steps, double* out) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        const auto x = strang_reference(m->dec, std::span<const double>(u, static_cast<std::size_t>(m->dec.n)), beta, steps);
        std::memcpy(out, x.data(), x.size() * sizeof(double));
    });
}

// Graph generators (netgen.cpp): returns a matrix handle.
int ref_pref(int64_t n, int64_t d, uint64_t seed, void** out) {
    return guarded([&] {
        auto* m = new RefMatrix;
        m->a = pref(n, d, seed);
        m->dec = decompose(m->a);
        *out = m;
    });
}

int ref_smallw(int64_t n, int64_t k, double p, uint64_t seed, void** out) {
    return guarded([&] {
        auto* m = new RefMatrix;
        m->a = smallw(n, k, p, seed);
        m->dec = decompose(m->a);
        *out = m;
    });
}

// ---------------------------------------------------------------- fem mode
// decompose_scaled (chain.cpp:80-85): tables of diag(row_scale) A.
int ref_matrix_create_scaled(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                             const double* row_scale, void** out) {
    return guarded([&] {
        auto* m = new RefMatrix;
        try {
            m->a = from_csr(n, row_ptr, col, val);
            m->dec = decompose_scaled(m->a, std::span<const double>(row_scale, static_cast<std::size_t>(n)));
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

}  // extern "C"

namespace {
// scaled_simpson (mlmc.cpp:66-75) is internal to mlmc.cpp; restated for the per-sample shim.
std::vector<double> simpson_scaled(index_t panels, double step) {
    std::vector<double> w(static_cast<std::size_t>(panels) + 1);
    const double h = step / 3.0;
    for (std::size_t j = 0; j < w.size(); ++j) {
        const bool end = (j == 0 || j + 1 == w.size());
        w[j] = h * (end ? 1.0 : (j % 2 == 1 ? 4.0 : 2.0));
    }
    return w;
}

MlmcOptions to_options(const RefOptions* o) {
    MlmcOptions opt;
    opt.epsilon = o->epsilon;
    opt.seed = o->seed;
    opt.threads = o->threads;
    opt.l0_override = o->l0_override;
    opt.warmup = o->warmup;
    opt.max_levels_above_l0 = o->max_levels_above_l0;
    opt.max_iterations = o->max_iterations;
    return opt;
}

void from_result(const MlmcResult& res, RefResult* out, RefLevel* levels_out, int32_t max_levels) {
    out->estimate = res.estimate;
    out->statistical_error = res.statistical_error;
    out->bias_estimate = res.bias_estimate;
    out->l0 = res.l0;
    out->L = res.L;
    out->total_cost = res.total_cost;
    out->converged = res.converged ? 1 : 0;
    out->nlevels = static_cast<int32_t>(res.levels.size());
    for (std::size_t l = 0; levels_out && l < res.levels.size() && l < static_cast<std::size_t>(max_levels); ++l) {
        levels_out[l].level = res.levels[l].level;
        levels_out[l].pad = 0;
        levels_out[l].sum = res.levels[l].sum;
        levels_out[l].sum_sq = res.levels[l].sum_sq;
        levels_out[l].samples = res.levels[l].samples;
        levels_out[l].cost = res.levels[l].cost;
    }
}
}  // namespace

extern "C" {

// fem_single / fem_coupled (paths.cpp:183-245) with run_level_ex's weights (mlmc.cpp:89-92),
// stream_for(seed, level, idx[i], 2).  value = the run_level sample: fem_single's value, or
// u[terminal] (eta_f - eta_c) + (integ_f - integ_c) (mlmc.cpp:126-133).
int ref_fem_samples(void* h, const double* u, const double* load, int64_t entry, double beta, int level, int base,
                    uint64_t seed, int64_t count, const uint64_t* sample_idx, double* value, double* eta_f,
                    double* eta_c, double* integ_f, double* integ_c, int64_t* terminal, uint64_t* cost) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        const std::size_t n = static_cast<std::size_t>(m->dec.n);
        const index_t steps = index_t{1} << level;
        const double dt = beta / static_cast<double>(steps);
        const LevelSampler sampler(m->dec, dt, steps);
        const std::vector<double> fw = simpson_scaled(steps, dt);
        const std::vector<double> cw = base ? std::vector<double>{} : simpson_scaled(steps / 2, 2.0 * dt);
        const std::span<const double> us(u, n), ls(load, n);
        for (int64_t i = 0; i < count; ++i) {
            RngStream s = stream_for(seed, static_cast<uint32_t>(level), sample_idx[i], 2u);
            if (base) {
                const FemSample f = sampler.fem_single(us, ls, entry, fw, s);
                value[i] = f.value;
                eta_f[i] = eta_c[i] = integ_f[i] = integ_c[i] = 0.0;
                terminal[i] = -1;
                cost[i] = f.cost;
            } else {
                const FemCoupledSample c = sampler.fem_coupled(ls, entry, fw, cw, s);
                const double du = u[c.terminal_state] * (c.eta_fine - c.eta_coarse);
                const double di = c.integ_fine - c.integ_coarse;
                value[i] = du + di;
                eta_f[i] = c.eta_fine;
                eta_c[i] = c.eta_coarse;
                integ_f[i] = c.integ_fine;
                integ_c[i] = c.integ_coarse;
                terminal[i] = c.terminal_state;
                cost[i] = c.cost;
            }
        }
    });
}

int ref_fem_run_level(void* h, const double* u, const double* load, int64_t entry, double beta, int level, int base,
                      uint64_t first, uint64_t count, uint64_t seed, int threads, double* sum, double* sum_sq,
                      uint64_t* samples, uint64_t* cost) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.load = std::span<const double>(load, static_cast<std::size_t>(m->dec.n));
        p.entry = entry;
        p.beta = beta;
        p.mode = SampleMode::fem;
        const LevelStats st = run_level(p, level, base != 0, first, count, seed, threads);
        *sum = st.sum;
        *sum_sq = st.sum_sq;
        *samples = st.samples;
        *cost = st.cost;
    });
}

int ref_fem_driver(void* h, const double* u, const double* load, int64_t entry, double beta, const RefOptions* o,
                   RefResult* out, RefLevel* levels_out, int32_t max_levels, double* quadrature_bound) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.load = std::span<const double>(load, static_cast<std::size_t>(m->dec.n));
        p.entry = entry;
        p.beta = beta;
        p.mode = SampleMode::fem;
        const MlmcResult res = mlmc_driver(p, to_options(o));
        from_result(res, out, levels_out, max_levels);
        *quadrature_bound = res.quadrature_bound;
    });
}

// solve_convdiff_point (fem.cpp:51-73) on a FemSystem given by arrays.
int ref_solve_convdiff_point(int64_t n, const double* mass_diag, const int64_t* row_ptr, const int64_t* col,
                             const double* val, const double* load, const double* u0, int64_t node, double t,
                             const RefOptions* o, RefResult* out, RefLevel* levels_out, int32_t max_levels,
                             double* quadrature_bound) {
    return guarded([&] {
        FemSystem sys;
        sys.mass_diag.assign(mass_diag, mass_diag + n);
        sys.stiffness = from_csr(n, row_ptr, col, val);
        sys.load.assign(load, load + n);
        sys.u0.assign(u0, u0 + n);
        const MlmcResult res = solve_convdiff_point(sys, node, t, to_options(o));
        from_result(res, out, levels_out, max_levels);
        *quadrature_bound = res.quadrature_bound;
    });
}

// load_fem_system (fem.cpp:12-37): sizes first (arrays NULL), then the data.
int ref_load_fem_system(const char* mass, const char* stiffness, const char* load_path, const char* u0_path,
                        int64_t* n, int64_t* nnz, double* mass_diag, int64_t* row_ptr, int64_t* col, double* val,
                        double* load, double* u0) {
    return guarded([&] {
        const FemSystem sys = load_fem_system(mass, stiffness, load_path, u0_path);
        *n = sys.size();
        *nnz = sys.stiffness.nnz();
        if (!mass_diag) return;
        std::memcpy(mass_diag, sys.mass_diag.data(), sys.mass_diag.size() * sizeof(double));
        export_csr(sys.stiffness, row_ptr, col, val);
        std::memcpy(load, sys.load.data(), sys.load.size() * sizeof(double));
        std::memcpy(u0, sys.u0.data(), sys.u0.size() * sizeof(double));
    });
}

// read_matrix_market (io.cpp:69-128) -> matrix handle; read_vector (io.cpp:154-167).
int ref_read_matrix_market(const char* path, void** out) {
    return guarded([&] {
        auto* m = new RefMatrix;
        try {
            m->a = read_matrix_market(path);
            m->dec = decompose(m->a);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

// SparseMatrix::from_triplets (sparse.cpp:12-49) on a triplet list, in list order.
int ref_from_triplets(int64_t n, int64_t count, const int64_t* rows, const int64_t* cols, const double* vals,
                      void** out) {
    return guarded([&] {
        std::vector<Triplet> t;
        t.reserve(static_cast<std::size_t>(count));
        for (int64_t k = 0; k < count; ++k) t.push_back({rows[k], cols[k], vals[k]});
        auto* m = new RefMatrix;
        try {
            m->a = SparseMatrix::from_triplets(n, std::move(t));
            m->dec = decompose(m->a);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

// Classical MC (mc.cpp:42-113).  out = {estimate, std_error, samples, dt, steps, wall_cost}.
struct RefMc {
    double estimate, std_error;
    uint64_t samples;
    double dt;
    int64_t steps;
    uint64_t wall_cost;
};

static void put_mc(const McResult& r, RefMc* out) {
    *out = RefMc{r.estimate, r.std_error, r.samples, r.dt, r.steps, r.wall_cost};
}

int ref_mc_single_entry(void* h, const double* u, int64_t entry, double beta, double dt, uint64_t samples,
                        uint64_t seed, int threads, RefMc* out) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        put_mc(mc_single_entry(m->dec, std::span<const double>(u, static_cast<std::size_t>(m->dec.n)), entry, beta,
                               dt, samples, seed, threads),
               out);
    });
}

int ref_mc_forward_scalar(void* h, const double* u, double beta, double dt, uint64_t samples, uint64_t seed,
                          int threads, RefMc* out) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        put_mc(mc_forward_scalar(m->dec, std::span<const double>(u, static_cast<std::size_t>(m->dec.n)), beta, dt,
                                 samples, seed, threads),
               out);
    });
}

int ref_mc_auto(void* h, const double* u, int64_t entry, double beta, double epsilon, uint64_t seed, int threads,
                RefMc* out) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        put_mc(mc_auto(m->dec, std::span<const double>(u, static_cast<std::size_t>(m->dec.n)), entry, beta, epsilon,
                       seed, threads),
               out);
    });
}

// Paper-figure harness (harness.cpp:41-144), entry mode.
int ref_fit_slope(int loglog, int64_t n, const double* x, const double* y, double* out) {
    return guarded([&] {
        const std::span<const double> xs(x, static_cast<std::size_t>(n)), ys(y, static_cast<std::size_t>(n));
        *out = loglog ? fit_loglog_slope(xs, ys) : fit_log2_slope(xs, ys);
    });
}

int ref_bench_levels(void* h, const double* u, int64_t entry, double beta, int l0, int count, uint64_t samples,
                     uint64_t seed, int threads, double* rows /* count x 5 */, double* slopes /* 3 */) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.entry = entry;
        p.beta = beta;
        const LevelDecayReport r = bench_levels(p, l0, count, samples, seed, threads);
        for (std::size_t i = 0; i < r.rows.size(); ++i) {
            rows[5 * i + 0] = r.rows[i].level;
            rows[5 * i + 1] = r.rows[i].dt;
            rows[5 * i + 2] = r.rows[i].mean;
            rows[5 * i + 3] = r.rows[i].variance;
            rows[5 * i + 4] = r.rows[i].cost_per_sample;
        }
        slopes[0] = r.slope_mean;
        slopes[1] = r.slope_variance;
        slopes[2] = r.slope_cost_tail;
    });
}

int ref_bench_l0(void* h, const double* u, int64_t entry, double beta, int l0_min, int l0_max, double epsilon,
                 uint64_t seed, int threads, double* costs, int* best, int* heuristic) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.entry = entry;
        p.beta = beta;
        const L0Report r = bench_l0(p, l0_min, l0_max, epsilon, seed, threads);
        for (std::size_t i = 0; i < r.points.size(); ++i) costs[i] = r.points[i].cost;
        *best = r.best_l0;
        *heuristic = r.heuristic_l0;
    });
}

int ref_bench_complexity(void* h, const double* u, int64_t entry, double beta, int64_t neps, const double* eps,
                         uint64_t seed, int threads, double* mlmc_cost, double* mc_cost, double* slopes) {
    return guarded([&] {
        auto* m = static_cast<RefMatrix*>(h);
        MlmcProblem p;
        p.dec = &m->dec;
        p.u = std::span<const double>(u, static_cast<std::size_t>(m->dec.n));
        p.entry = entry;
        p.beta = beta;
        const ComplexityReport r =
            bench_complexity(p, std::span<const double>(eps, static_cast<std::size_t>(neps)), seed, threads);
        for (std::size_t i = 0; i < r.mlmc.size(); ++i) {
            mlmc_cost[i] = r.mlmc[i].cost;
            mc_cost[i] = r.mc[i].cost;
        }
        slopes[0] = r.slope_mlmc;
        slopes[1] = r.slope_mc;
    });
}

int ref_read_vector(const char* path, int64_t cap, double* out, int64_t* n) {
    return guarded([&] {
        const std::vector<double> v = read_vector(path);
        *n = static_cast<int64_t>(v.size());
        if (out) std::memcpy(out, v.data(), std::min<int64_t>(cap, *n) * sizeof(double));
    });
}

int ref_total_communicability(void* h, double beta, const RefOptions* o, RefResult* out) {
    return guarded([&] {
        const MlmcResult res = total_communicability(static_cast<RefMatrix*>(h)->a,
                                                     beta > 0.0 ? std::optional<double>(beta) : std::nullopt,
                                                     to_options(o));
        from_result(res, out, nullptr, 0);
    });
}

}  // extern "C"
