// expmc_b200.hpp -- header-only C++17 shim over the C-ABI (expmc_b200.h) that keeps the
// reference's C++ surface for the MLMC path (expmc/mlmc.hpp:15-98): the same type names, the
// same argument meaning, and the same exception types (std::invalid_argument,
// std::out_of_range, std::domain_error) for the same bad inputs.
//
//   reference                                    this header
//   -------------------------------------------  ---------------------------------------------
//   ChainDecomposition dec = decompose(A);       expmc::b200::Context ctx(A, u, device);
//   MlmcProblem p{&dec, u, {}, entry, beta};     expmc::b200::MlmcProblem p{&ctx, entry, beta};
//   LevelStats s = run_level(p, l, base, f, m,   LevelStats s = run_level(p, l, base, f, m, seed);
//                            seed, threads);
//   MlmcResult r = mlmc_driver(p, opts);         MlmcResult r = mlmc_driver(p, opts);
//   (one driver call per component)              mlmc_driver_rows(ctx, beta, rows, seeds, opts)
//   p.mode = SampleMode::forward (dec of A^T)    p.mode = SampleMode::forward (ctx of A^T)
//   total_communicability(A, beta, opts)         total_communicability(A, beta, opts)
//   node_communicability(A, node, beta, opts)    node_communicability(A, node, beta, opts)
//
// Link with paper_1904_12754_b200/_lib/libexpmc_b200.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "expmc_b200.h"

namespace expmc::b200 {

inline void check(int rc) {
    if (rc == EXPMC_OK) return;
    const std::string msg = expmc_last_error();
    switch (rc) {
        case EXPMC_EINVAL: throw std::invalid_argument(msg);
        case EXPMC_ERANGE: throw std::out_of_range(msg);
        case EXPMC_EDOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

/// Square CSR matrix, canonical as expmc::SparseMatrix stores it (sparse.hpp:21-75).
struct CsrView {
    int64_t n = 0;
    std::vector<int64_t> row_ptr{0};
    std::vector<int64_t> col;
    std::vector<double> val;
};

/// mlmc.hpp:18-31 (+ jumps).
struct LevelStats {
    int level = 0;
    double sum = 0.0;
    double sum_sq = 0.0;
    std::uint64_t samples = 0;
    std::uint64_t cost = 0;
    std::uint64_t jumps = 0;
    double mean() const { return samples ? sum / static_cast<double>(samples) : 0.0; }
    double variance() const {
        if (samples < 2) return 0.0;
        const double m = mean();
        const double v = sum_sq / static_cast<double>(samples) - m * m;
        return v > 0.0 ? v : 0.0;
    }
    double unit_cost() const { return samples ? static_cast<double>(cost) / static_cast<double>(samples) : 0.0; }
};

/// mlmc.hpp:59-67.
struct MlmcOptions {
    double epsilon = 1e-3;
    std::uint64_t seed = 0;
    int threads = 0;
    int l0_override = -1;
    std::uint64_t warmup = 1000;
    int max_levels_above_l0 = 30;
    int max_iterations = 200;
    double max_cost = 0.0;  // extension (0 = off): per-component budget in model units
    expmc_options c() const {
        return expmc_options{epsilon, seed, threads, l0_override, warmup, max_levels_above_l0, max_iterations, max_cost};
    }
};

/// mlmc.hpp:33-43 (+ totals of jumps and samples).
struct MlmcResult {
    double estimate = 0.0;
    double statistical_error = 0.0;
    double bias_estimate = 0.0;
    double quadrature_bound = 0.0;
    std::vector<LevelStats> levels;
    int l0 = 0;
    int L = 0;
    std::uint64_t total_cost = 0;
    bool converged = false;
    std::uint64_t total_jumps = 0;
    std::uint64_t total_samples = 0;
};

/// Device tables of A plus the bound vector u on one GPU (decompose + MlmcProblem::u).
class Context {
  public:
    Context(const CsrView& a, const std::vector<double>& u, int device = 0) {
        if (static_cast<int64_t>(u.size()) != a.n)
            throw std::invalid_argument("vector length does not match decomposition");
        const expmc_csr csr{a.n, a.row_ptr.empty() ? 0 : a.row_ptr.back(), a.row_ptr.data(), a.col.data(),
                            a.val.data()};
        check(expmc_ctx_create(&csr, u.data(), device, &ctx_));
        check(expmc_ctx_get_info(ctx_, &info_));
    }
    /// decompose_scaled (chain.cpp:80-85): the tables of diag(row_scale) A.
    Context(const CsrView& a, const std::vector<double>& row_scale, const std::vector<double>& u, int device) {
        if (static_cast<int64_t>(u.size()) != a.n)
            throw std::invalid_argument("vector length does not match decomposition");
        if (static_cast<int64_t>(row_scale.size()) != a.n)
            throw std::invalid_argument("row scale length does not match matrix dimension");
        const expmc_csr csr{a.n, a.row_ptr.empty() ? 0 : a.row_ptr.back(), a.row_ptr.data(), a.col.data(),
                            a.val.data()};
        check(expmc_ctx_create_scaled(&csr, row_scale.data(), u.data(), device, &ctx_));
        check(expmc_ctx_get_info(ctx_, &info_));
    }
    ~Context() { expmc_ctx_destroy(ctx_); }
    /// MlmcProblem::load for fem mode.
    void set_load(const std::vector<double>& load) {
        if (static_cast<int64_t>(load.size()) != info_.n)
            throw std::invalid_argument("load length does not match decomposition");
        check(expmc_ctx_set_load(ctx_, load.data()));
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    expmc_ctx* get() const { return ctx_; }
    const expmc_ctx_info& info() const { return info_; }

  private:
    expmc_ctx* ctx_ = nullptr;
    expmc_ctx_info info_{};
};

/// A^T in canonical CSR (SparseMatrix::transposed): forward mode runs on the tables of A^T.
inline CsrView transposed(const CsrView& a) {
    CsrView t;
    t.n = a.n;
    t.row_ptr.assign(static_cast<size_t>(a.n) + 1, 0);
    for (int64_t k = 0; k < static_cast<int64_t>(a.col.size()); ++k) ++t.row_ptr[static_cast<size_t>(a.col[k]) + 1];
    std::partial_sum(t.row_ptr.begin(), t.row_ptr.end(), t.row_ptr.begin());
    t.col.resize(a.col.size());
    t.val.resize(a.val.size());
    std::vector<int64_t> next(t.row_ptr.begin(), t.row_ptr.end() - 1);
    for (int64_t i = 0; i < a.n; ++i)  // rows ascending: each new row's columns come out sorted
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const int64_t at = next[static_cast<size_t>(a.col[k])]++;
            t.col[at] = i;
            t.val[at] = a.val[k];
        }
    return t;
}

/// mlmc.hpp:45.  fem is outside this build (the C-ABI answers EXPMC_ENOTIMPL).
enum class SampleMode { entry, forward, fem };

/// mlmc.hpp:47-57: entry mode on the context of A, forward mode on the context of A^T.
struct MlmcProblem {
    Context* ctx = nullptr;
    std::int64_t entry = 0;
    double beta = 1.0;
    SampleMode mode = SampleMode::entry;
};

/// spectral_scale (chain.cpp:98-102): 1 / d_max.
inline double spectral_scale(const Context& ctx) {
    if (!(ctx.info().d_max > 0.0)) throw std::domain_error("d_max <= 0: no spectral scale, supply beta explicitly");
    return 1.0 / ctx.info().d_max;
}

inline void check_mode(SampleMode) {}

inline int initial_level(double beta, double d_max) {
    int32_t l = 0;
    check(expmc_initial_level(beta, d_max, &l));
    return l;
}

inline std::vector<std::uint64_t> optimal_allocation(const std::vector<double>& v, const std::vector<double>& c,
                                                     double eps) {
    if (v.size() != c.size()) throw std::invalid_argument("variance and cost arrays differ in length");
    std::vector<std::uint64_t> m(v.size());
    check(expmc_optimal_allocation(static_cast<int64_t>(v.size()), v.data(), c.data(), eps, m.data()));
    return m;
}

inline double bias_estimate(const std::vector<double>& means) {
    double b = 0.0;
    check(expmc_bias_estimate(static_cast<int64_t>(means.size()), means.data(), &b));
    return b;
}

/// run_level (mlmc.hpp:86-88); `threads` is accepted for signature compatibility.
inline LevelStats run_level(const MlmcProblem& p, int level, bool base_level, std::uint64_t first_index,
                            std::uint64_t additional, std::uint64_t seed, int /*threads*/ = 0) {
    if (p.ctx == nullptr) throw std::invalid_argument("problem has no decomposition");
    check_mode(p.mode);
    expmc_level_stats s{};
    if (p.mode == SampleMode::forward)
        check(expmc_run_level_forward(p.ctx->get(), p.beta, level, base_level ? 1 : 0, first_index, additional, seed,
                                      &s));
    else if (p.mode == SampleMode::fem)
        check(expmc_run_level_fem(p.ctx->get(), p.entry, p.beta, level, base_level ? 1 : 0, first_index, additional,
                                  seed, &s));
    else
        check(expmc_run_level(p.ctx->get(), p.entry, p.beta, level, base_level ? 1 : 0, first_index, additional,
                              seed, &s));
    return LevelStats{level, s.sum, s.sum_sq, s.samples, s.cost, s.jumps};
}

inline MlmcResult to_result(const expmc_result& r, const expmc_level_record* lv) {
    MlmcResult o;
    o.estimate = r.estimate;
    o.statistical_error = r.statistical_error;
    o.bias_estimate = r.bias_estimate;
    o.quadrature_bound = r.quadrature_bound;
    o.l0 = r.l0;
    o.L = r.L;
    o.total_cost = r.total_cost;
    o.converged = r.converged != 0;
    o.total_jumps = r.total_jumps;
    o.total_samples = r.total_samples;
    for (int i = 0; i < r.nlevels && lv; ++i)
        o.levels.push_back(LevelStats{lv[i].level, lv[i].sum, lv[i].sum_sq, lv[i].samples, lv[i].cost, 0});
    return o;
}

/// mlmc_driver (mlmc.hpp:94).
inline MlmcResult mlmc_driver(const MlmcProblem& p, const MlmcOptions& opt) {
    if (p.ctx == nullptr) throw std::invalid_argument("problem has no decomposition");
    constexpr int kMax = 64;
    expmc_result r{};
    std::vector<expmc_level_record> lv(kMax);
    const expmc_options o = opt.c();
    check_mode(p.mode);
    if (p.mode == SampleMode::forward) {
        check(expmc_mlmc_driver_forward(p.ctx->get(), p.beta, &o, 1, nullptr, &r, lv.data(), kMax));
    } else if (p.mode == SampleMode::fem) {
        const std::int64_t row = p.entry;
        const std::uint64_t seed = opt.seed;
        check(expmc_mlmc_driver_fem(p.ctx->get(), p.beta, &o, 1, &row, &seed, &r, lv.data(), kMax));
    } else
        check(expmc_mlmc_driver(p.ctx->get(), p.entry, p.beta, &o, &r, lv.data(), kMax));
    return to_result(r, lv.data());
}

/// total_communicability (communicability.cpp:10-21): 1^T e^{beta A} 1 by forward-mode MLMC
/// on A^T; beta defaults to spectral_scale of A^T's decomposition.
inline MlmcResult total_communicability(const CsrView& a, std::optional<double> beta, const MlmcOptions& opt,
                                        int device = 0) {
    Context ctx(transposed(a), std::vector<double>(static_cast<size_t>(a.n), 1.0), device);
    MlmcProblem p{&ctx, 0, beta ? *beta : spectral_scale(ctx), SampleMode::forward};
    return mlmc_driver(p, opt);
}

/// fem.hpp FemSystem: lumped-mass system M u' = -K u + F, u(0) = u0.
struct FemSystem {
    std::vector<double> mass_diag;
    CsrView stiffness;
    std::vector<double> load;
    std::vector<double> u0;
    std::int64_t size() const { return stiffness.n; }
};

/// solve_convdiff_point (fem.cpp:51-73): u(node, t) by fem-mode MLMC on the chain of -M^{-1}K.
inline MlmcResult solve_convdiff_point(const FemSystem& sys, std::int64_t node, double t, const MlmcOptions& opt,
                                       int device = 0) {
    if (!(t > 0.0)) throw std::invalid_argument("time must be positive");
    if (node < 0 || node >= sys.size()) throw std::out_of_range("node index outside system");
    const size_t n = static_cast<size_t>(sys.size());
    std::vector<double> row_scale(n), scaled_load(n);
    for (size_t i = 0; i < n; ++i) {
        row_scale[i] = -1.0 / sys.mass_diag[i];
        scaled_load[i] = sys.load[i] / sys.mass_diag[i];
    }
    Context ctx(sys.stiffness, row_scale, sys.u0, device);
    ctx.set_load(scaled_load);
    return mlmc_driver(MlmcProblem{&ctx, node, t, SampleMode::fem}, opt);
}

/// node_communicability (communicability.cpp:23-35): (e^{beta A} 1)_node, entry mode.
inline MlmcResult node_communicability(const CsrView& a, std::int64_t node, std::optional<double> beta,
                                       const MlmcOptions& opt, int device = 0) {
    Context ctx(a, std::vector<double>(static_cast<size_t>(a.n), 1.0), device);
    MlmcProblem p{&ctx, node, beta ? *beta : spectral_scale(ctx), SampleMode::entry};
    return mlmc_driver(p, opt);
}

/// The all-components estimator: one reference decision sequence per row, batched on the GPU.
inline std::vector<MlmcResult> mlmc_driver_rows(Context& ctx, double beta, const std::vector<std::int64_t>& rows,
                                                const std::vector<std::uint64_t>& seeds, const MlmcOptions& opt) {
    if (rows.size() != seeds.size()) throw std::invalid_argument("one seed per row required");
    constexpr int kMax = 64;
    std::vector<expmc_result> r(rows.size());
    std::vector<expmc_level_record> lv(rows.size() * kMax);
    const expmc_options o = opt.c();
    check(expmc_mlmc_driver_rows(ctx.get(), beta, &o, static_cast<int64_t>(rows.size()), rows.data(), seeds.data(),
                                 r.data(), lv.data(), kMax));
    std::vector<MlmcResult> out;
    out.reserve(rows.size());
    for (size_t i = 0; i < rows.size(); ++i) out.push_back(to_result(r[i], lv.data() + i * kMax));
    return out;
}

}  // namespace expmc::b200
