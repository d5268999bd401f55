// Host C++ MLMC driver, batched over rows (the per-component estimator interface).
//
// Restates mlmc_driver (mlmc.cpp:170-260) for many entries at once.  Each row keeps its own
// copy of the reference's state (levels, top, iteration counter) and takes EXACTLY the
// reference's decision sequence: warm start at L = l0+4 with `warmup` samples per level,
// then per iteration the Lagrange allocation (optimal_allocation, mlmc.cpp:25-43), the
// extension of short levels, the stopping test sqrt(V_T) <= eps/sqrt2 and bias <= eps/sqrt2
// (mlmc.cpp:223-240) and, while the bias bound fails, one more level (mlmc.cpp:241-246).
// Rows advance in lock-step rounds: every row's pending extensions of one round go to the
// GPU as a single batched run_level pass (context.cu), so a round costs one sampler launch
// per 4M chunks no matter how many rows are active.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <type_traits>
#include <utility>
#include <string>
#include <vector>

#include <omp.h>

#include "internal.hpp"

using namespace expmc_b200;

namespace {

struct Level {
    double sum = 0.0, sum_sq = 0.0;
    double integ = 0.0;  // fem: Level::integ_sum (mlmc.cpp:184-198)
    uint64_t samples = 0, cost = 0, jumps = 0;
    double mean() const { return samples ? sum / static_cast<double>(samples) : 0.0; }
    double variance() const {  // LevelStats::variance, mlmc.cpp:13-17
        if (samples < 2) return 0.0;
        const double m = mean();
        return std::max(0.0, sum_sq / static_cast<double>(samples) - m * m);
    }
    double unit_cost() const {
        return samples ? static_cast<double>(cost) / static_cast<double>(samples) : 0.0;
    }
};

int initial_level_impl(double beta, double d_max) {  // mlmc.cpp:19-23
    if (!(beta > 0.0)) throw Status(EXPMC_EINVAL, "beta must be positive");
    if (!(d_max > 0.0)) return 0;
    return static_cast<int>(std::max<long>(0, std::lround(std::log2(2.0 * beta * d_max))));
}

void optimal_allocation_impl(size_t n, const double* v, const double* c, double eps, uint64_t* m) {
    if (!(eps > 0.0)) throw Status(EXPMC_EINVAL, "epsilon must be positive");  // mlmc.cpp:25-43
    double s = 0.0;
    for (size_t l = 0; l < n; ++l) {
        if (v[l] < 0.0 || !(c[l] > 0.0)) throw Status(EXPMC_EINVAL, "require V_l >= 0 and C_l > 0");
        s += std::sqrt(v[l] * c[l]);
    }
    const double scale = 2.0 / (eps * eps) * s;
    for (size_t l = 0; l < n; ++l) {
        const double raw = scale * std::sqrt(v[l] / c[l]);
        m[l] = std::max<uint64_t>(2, static_cast<uint64_t>(std::ceil(raw)));
    }
}

double bias_estimate_impl(size_t n, const double* means) {  // mlmc.cpp:45-51
    if (n < 2) throw Status(EXPMC_EINVAL, "bias estimate needs at least two coupled levels");
    const double last = std::abs(means[n - 1]);
    const double prev = std::abs(means[n - 2]);
    return std::max(last, prev / 4.0) / 3.0;
}

// A growable array of trivially copyable T whose new elements are left uninitialised.
template <class T>
struct RawArray {
    std::unique_ptr<T[]> p;
    size_t n = 0, cap = 0;
    void resize(size_t m) {
        if (m > cap) {
            std::unique_ptr<T[]> q(new T[m]);  // default-init: no zeroing pass
            if (n) std::memcpy(q.get(), p.get(), n * sizeof(T));
            p = std::move(q);
            cap = m;
        }
        n = m;
    }
    size_t size() const { return n; }
    T* data() { return p.get(); }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

// Per-row level and request lists live in bump arenas (one per OpenMP thread) whose 8 MB blocks
// come from a process-wide pool: a C2 job has 2^20 rows, and two small heap allocations per row
// cost ~60 ms to create and ~90 ms to free per job with the GPU idle.  Blocks go back to the
// pool, untouched, when the driver call ends.
struct BlockPool {
    std::mutex m;
    std::vector<char*> free_blocks;
    std::multimap<size_t, char*> row_buffers;
};
BlockPool& block_pool() {
    static BlockPool* p = new BlockPool;  // never destroyed: blocks live until process exit
    return *p;
}
constexpr size_t kArenaBlock = size_t{8} << 20;

struct Arena {
    std::vector<char*> blocks;
    char* cur = nullptr;
    size_t left = 0;
    void* get(size_t bytes) {
        bytes = (bytes + 15) & ~size_t{15};
        if (bytes > left) {
            if (bytes > kArenaBlock) throw Status(EXPMC_EINTERNAL, "driver arena request too large");
            char* b = nullptr;
            {
                BlockPool& pool = block_pool();
                std::lock_guard<std::mutex> g(pool.m);
                if (!pool.free_blocks.empty()) {
                    b = pool.free_blocks.back();
                    pool.free_blocks.pop_back();
                }
            }
            if (!b) b = new char[kArenaBlock];
            blocks.push_back(b);
            cur = b;
            left = kArenaBlock;
        }
        void* p = cur;
        cur += bytes;
        left -= bytes;
        return p;
    }
    ~Arena() {
        BlockPool& pool = block_pool();
        std::lock_guard<std::mutex> g(pool.m);
        pool.free_blocks.insert(pool.free_blocks.end(), blocks.begin(), blocks.end());
    }
};
thread_local Arena* tl_arena = nullptr;  // the calling OpenMP thread's arena

// The row-state array itself (~100 B x rows): a pooled buffer as well, kept for the next call.
struct RowBuffer {
    char* p = nullptr;
    size_t bytes = 0;
    explicit RowBuffer(size_t want) {
        BlockPool& pool = block_pool();
        std::lock_guard<std::mutex> g(pool.m);
        auto it = pool.row_buffers.lower_bound(want);
        if (it != pool.row_buffers.end()) {
            bytes = it->first;
            p = it->second;
            pool.row_buffers.erase(it);
        }
        if (!p) {
            bytes = std::max<size_t>(want, 1);
            p = new char[bytes];
        }
    }
    ~RowBuffer() {
        BlockPool& pool = block_pool();
        std::lock_guard<std::mutex> g(pool.m);
        pool.row_buffers.emplace(bytes, p);
    }
};

// A growable array of trivially copyable T in the calling thread's arena.
template <class T>
struct ArenaVec {
    T* p = nullptr;
    uint32_t n = 0, cap = 0;
    size_t size() const { return n; }
    bool empty() const { return n == 0; }
    void clear() { n = 0; }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
    T* begin() { return p; }
    T* end() { return p + n; }
    const T* begin() const { return p; }
    const T* end() const { return p + n; }
    void reserve(uint32_t want) {
        if (want <= cap) return;
        const uint32_t nc = std::max(want, cap * 2u);
        T* q = static_cast<T*>(tl_arena->get(nc * sizeof(T)));
        if (n) std::memcpy(static_cast<void*>(q), p, n * sizeof(T));
        p = q;
        cap = nc;
    }
    template <class... A>
    void emplace_back(A&&... a) {
        if (n == cap) reserve(n + 1);
        p[n++] = T{std::forward<A>(a)...};
    }
    void resize(uint32_t m) {
        reserve(m);
        for (uint32_t i = n; i < m; ++i) p[i] = T{};
        n = m;
    }
};

enum class Phase { waiting_warmup, waiting_extend, waiting_added, done };

struct RowState {
    int64_t entry = 0;
    uint64_t seed = 0;
    int l0 = 0, cap = 0, top = 0, iter = 0;
    Phase phase = Phase::waiting_warmup;
    ArenaVec<Level> lv;
    ArenaVec<std::pair<int, uint64_t>> pending;  // (level index, additional samples)
    double stat_error = 0.0, bias = 0.0, quad = 0.0;
    double projected = 0.0;
    bool converged = false;
    bool over_budget = false;
};

static_assert(std::is_trivially_destructible<RowState>::value, "row states are never destroyed");
static_assert(std::is_trivially_copyable<Level>::value, "levels are moved with memcpy");

struct DriverConfig {
    double eps, target;
    uint64_t warmup;
    int max_iterations;
    double max_cost;
    bool fem;
};

// Advance one row whose pending work has completed, up to its next GPU request or the end.
void advance(RowState& r, const DriverConfig& cfg, std::vector<double>& v, std::vector<double>& c,
             std::vector<uint64_t>& want, std::vector<double>& means) {
    bool eval = r.phase == Phase::waiting_extend;
    for (;;) {
        if (!eval) {
            // ---- top of the reference's for-iter loop (mlmc.cpp:212-221)
            if (r.iter >= cfg.max_iterations) {
                r.phase = Phase::done;
                return;
            }
            const size_t nl = r.lv.size();
            v.resize(nl);
            c.resize(nl);
            want.resize(nl);
            for (size_t i = 0; i < nl; ++i) {
                v[i] = r.lv[i].variance();
                c[i] = std::max(r.lv[i].unit_cost(), 1.0);
            }
            optimal_allocation_impl(nl, v.data(), c.data(), cfg.eps, want.data());
            double proj = 0.0;
            for (size_t i = 0; i < nl; ++i)
                proj += static_cast<double>(std::max(want[i], r.lv[i].samples)) * c[i];
            r.projected = proj;
            if (cfg.max_cost > 0.0 && proj > cfg.max_cost) {  // extension: infeasible component
                r.over_budget = true;
                r.phase = Phase::done;
                return;
            }
            for (size_t i = 0; i < nl; ++i)
                if (want[i] > r.lv[i].samples)
                    r.pending.emplace_back(static_cast<int>(i), want[i] - r.lv[i].samples);
            if (!r.pending.empty()) {
                r.phase = Phase::waiting_extend;
                return;
            }
        }
        eval = false;
        // ---- statistics after the extension (mlmc.cpp:223-240)
        double vt = 0.0;
        for (const Level& l : r.lv) vt += l.variance() / static_cast<double>(l.samples);
        r.stat_error = std::sqrt(vt);
        means.clear();
        for (size_t i = 1; i < r.lv.size(); ++i) means.push_back(r.lv[i].mean());
        r.bias = bias_estimate_impl(means.size(), means.data());
        if (cfg.fem) {  // quad = bias_estimate(integ_means), mlmc.cpp:226-235
            means.clear();
            for (size_t i = 1; i < r.lv.size(); ++i)
                means.push_back(r.lv[i].integ / static_cast<double>(r.lv[i].samples));
            r.quad = bias_estimate_impl(means.size(), means.data());
        }
        if (r.stat_error <= cfg.target && r.bias <= cfg.target) {
            r.converged = true;
            r.phase = Phase::done;
            return;
        }
        if (r.bias > cfg.target) {  // mlmc.cpp:241-246
            if (r.top == r.cap) {
                r.phase = Phase::done;
                return;
            }
            ++r.top;
            r.lv.emplace_back();
            r.pending.emplace_back(static_cast<int>(r.lv.size() - 1), cfg.warmup);
            ++r.iter;
            r.phase = Phase::waiting_added;
            return;
        }
        ++r.iter;
    }
}

// lane EXPMC_LANE_FORWARD: rows == nullptr, each "row" an independent run of the functional
// sum(e^{tA} u) with its own seed; validate_problem skips the entry check (mlmc.cpp:154).
// lane EXPMC_LANE_FEM: entry rows plus the load integrals; l0 >= 1 (mlmc.cpp:177).
void drive_rows(expmc_ctx* ctx, uint32_t lane, double beta, const expmc_options& opt, int64_t nrows,
                const int64_t* rows, const uint64_t* row_seed, expmc_result* out, expmc_level_record* levels,
                int32_t max_levels) {
    expmc_ctx_info info{};
    if (expmc_ctx_get_info(ctx, &info) != EXPMC_OK) throw Status(EXPMC_EINVAL, "null context");
    for (int64_t r = 0; rows && r < nrows; ++r)  // validate_problem, mlmc.cpp:150-159
        if (rows[r] < 0 || rows[r] >= info.n) throw Status(EXPMC_ERANGE, "entry index outside matrix");
    if (lane == EXPMC_LANE_FEM && !ctx_has_load(ctx))
        throw Status(EXPMC_EINVAL, "load length does not match decomposition");
    if (!(beta > 0.0)) throw Status(EXPMC_EINVAL, "beta must be positive");
    if (!(opt.epsilon > 0.0)) throw Status(EXPMC_EINVAL, "epsilon must be positive");
    int l0 = opt.l0_override >= 0 ? opt.l0_override : initial_level_impl(beta, info.d_max);
    if (lane == EXPMC_LANE_FEM) l0 = std::max(l0, 1);  // the coarse grid must carry a Simpson rule
    const int cap = l0 + opt.max_levels_above_l0;
    // fewer than two coupled levels: the reference's first iteration throws from bias_estimate
    // (mlmc.cpp:45-47, 201-235); checked here, before the per-row setup sizes arrays from it
    if (opt.max_iterations > 0 && nrows > 0 && opt.max_levels_above_l0 < 2)
        throw Status(EXPMC_EINVAL, "bias estimate needs at least two coupled levels");
    DriverConfig cfg{opt.epsilon, opt.epsilon / std::sqrt(2.0), opt.warmup, opt.max_iterations, opt.max_cost,
                     lane == EXPMC_LANE_FEM};

    const auto t_setup = std::chrono::steady_clock::now();
    std::vector<Arena> arenas(static_cast<size_t>(omp_get_max_threads()));
    RowBuffer st_mem(static_cast<size_t>(nrows) * sizeof(RowState));
    RowState* const st = reinterpret_cast<RowState*>(st_mem.p);  // constructed in place below
    int setup_failed = 0;
#pragma omp parallel
    {
        tl_arena = &arenas[static_cast<size_t>(omp_get_thread_num())];
#pragma omp for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        RowState& s = st[static_cast<size_t>(r)];
        new (&s) RowState();
        s.entry = rows ? rows[r] : 0;
        s.seed = row_seed[r];
        s.l0 = l0;
        s.cap = cap;
        s.top = std::min(l0 + 4, cap);  // mlmc.cpp:201-205
        try {  // nothing may escape an OpenMP region
            s.lv.reserve(8);  // one arena slice each for the common L - l0 < 8
            s.pending.reserve(8);
            s.lv.resize(static_cast<uint32_t>(s.top - l0 + 1));
            for (int i = 0; i <= s.top - l0; ++i) s.pending.emplace_back(i, opt.warmup);
        } catch (...) {
#pragma omp atomic write
            setup_failed = 1;
        }
    }
    }
    if (setup_failed) throw Status(EXPMC_EINTERNAL, "host allocation failed in the driver setup");

    // Per round: (1) every active row's pending extensions become one contiguous slice of a
    // batch, (2) one batched GPU pass, (3) each row applies its slice (extend(), mlmc.cpp:188-199)
    // and advances its state machine.  Rows are independent, so (1) and (3) run in parallel --
    // and large jobs split the rows into two cohorts whose rounds alternate on the GPU: while
    // one cohort's batch samples, the host consumes the other's results and stages its next
    // batch (two staging slots in the context), so the host work hides behind the kernels.
    // Every row still sees exactly its own sequence of requests and results.
    struct Cohort {
        std::vector<int64_t> active;
        // request / result arrays: grown without value-initialisation, first touched by the
        // parallel fill (round 0 stages ~5 requests per row: hundreds of MB at n = 2^20)
        RawArray<expmc_level_req> req;
        RawArray<expmc_level_stats> res;
        std::vector<size_t> off;
        std::vector<unsigned char> keep;
        bool inflight = false;
        int round = 0;
        double build_ms = 0.0;
    };
    const int ncoh = nrows >= 4096 ? 2 : 1;
    Cohort coh[2];
    for (int64_t r = 0; r < nrows; ++r) coh[r % ncoh].active.push_back(r);
    const bool trace = std::getenv("EXPMC_TRACE") != nullptr;  // per-round timeline on stderr
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };

    auto launch = [&](Cohort& co, int slot) {
        if (co.active.empty()) return;
        const auto t0 = clk::now();
        const size_t na = co.active.size();
        co.off.assign(na + 1, 0);
        for (size_t i = 0; i < na; ++i) co.off[i + 1] = co.off[i] + st[static_cast<size_t>(co.active[i])].pending.size();
        co.req.resize(co.off[na]);
        co.res.resize(co.off[na]);  // batch_launch writes every element
#pragma omp parallel for schedule(static)
        for (size_t i = 0; i < na; ++i) {
            const RowState& s = st[static_cast<size_t>(co.active[i])];
            size_t k = co.off[i];
            for (const auto& p : s.pending) {
                const Level& l = s.lv[static_cast<size_t>(p.first)];
                const int level = s.l0 + p.first;
                co.req[k++] = expmc_level_req{s.entry, s.seed, l.samples, p.second, level, level == s.l0 ? 1 : 0};
            }
        }
        batch_launch(ctx, slot, beta, lane, co.req.data(), static_cast<int64_t>(co.req.size()), co.res.data());
        co.inflight = true;
        co.build_ms = ms(t0, clk::now());
    };

    auto consume = [&](Cohort& co, int slot) {
        const auto t0 = clk::now();
        batch_finish(ctx, slot, co.req.data(), co.res.data());
        co.inflight = false;
        const auto t1 = clk::now();
        const size_t na = co.active.size();
        co.keep.assign(na, 0);
        int err_code = 0;
        std::string err_msg;
#pragma omp parallel
        {
            tl_arena = &arenas[static_cast<size_t>(omp_get_thread_num())];
            std::vector<double> v, c, means;
            std::vector<uint64_t> want;
#pragma omp for schedule(dynamic, 256)
            for (size_t i = 0; i < na; ++i) {
                RowState& s = st[static_cast<size_t>(co.active[i])];
                for (size_t j = 0; j < s.pending.size(); ++j) {  // extend(): mlmc.cpp:188-199
                    const expmc_level_stats& d = co.res[co.off[i] + j];
                    Level& l = s.lv[static_cast<size_t>(s.pending[j].first)];
                    l.sum += d.sum;
                    l.sum_sq += d.sum_sq;
                    l.samples += d.samples;
                    l.cost += d.cost;
                    l.jumps += d.jumps;
                    l.integ += d.integ_sum;
                }
                s.pending.clear();
                try {
                    advance(s, cfg, v, c, want, means);
                } catch (const Status& e) {
#pragma omp critical(expmc_driver_error)
                    if (err_code == 0) {
                        err_code = e.code;
                        err_msg = e.what();
                    }
                    s.phase = Phase::done;
                } catch (const std::exception& e) {  // nothing may escape an OpenMP region
#pragma omp critical(expmc_driver_error)
                    if (err_code == 0) {
                        err_code = EXPMC_EINTERNAL;
                        err_msg = e.what();
                    }
                    s.phase = Phase::done;
                }
                co.keep[i] = s.phase != Phase::done;
            }
        }
        if (err_code) throw Status(err_code, err_msg);
        size_t m = 0;
        for (size_t i = 0; i < na; ++i)
            if (co.keep[i]) co.active[m++] = co.active[i];
        if (trace) {
            uint64_t smp = 0;
            for (size_t q = 0; q < co.req.size(); ++q) smp += co.req[q].count;
            std::fprintf(stderr, "[expmc] cohort %d round %d rows %zu reqs %zu samples %llu | build %.2f ms wait %.2f ms "
                         "advance %.2f ms\n",
                         slot, co.round, na, co.req.size(), static_cast<unsigned long long>(smp), co.build_ms,
                         ms(t0, t1), ms(t1, clk::now()));
        }
        ++co.round;
        co.active.resize(m);
    };

    const auto t_rounds = clk::now();
    try {
        for (int k = 0; k < ncoh; ++k) launch(coh[k], k);
        for (;;) {
            bool any = false;
            for (int k = 0; k < ncoh; ++k) {
                if (!coh[k].inflight) continue;
                any = true;
                consume(coh[k], k);
                launch(coh[k], k);  // queued behind the other cohort's batch
            }
            if (!any) break;
        }
    } catch (...) {
        batch_drain(ctx);  // no batch may outlive its staging arrays
        throw;
    }

    const auto t_out = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {  // mlmc.cpp:249-259
        const RowState& s = st[static_cast<size_t>(r)];
        expmc_result& o = out[r];
        std::memset(&o, 0, sizeof o);
        o.l0 = s.l0;
        o.L = s.top;
        o.statistical_error = s.stat_error;
        o.bias_estimate = s.bias;
        o.quadrature_bound = s.quad;
        o.converged = s.converged ? 1 : 0;
        o.projected_cost = s.projected;
        o.over_budget = s.over_budget ? 1 : 0;
        o.nlevels = static_cast<int32_t>(s.lv.size());
        for (size_t i = 0; i < s.lv.size(); ++i) {
            const Level& l = s.lv[i];
            o.estimate += l.mean();
            o.total_cost += l.cost;
            o.total_jumps += l.jumps;
            o.total_samples += l.samples;
            if (levels && static_cast<int32_t>(i) < max_levels) {
                expmc_level_record& rec = levels[r * max_levels + static_cast<int64_t>(i)];
                rec.level = s.l0 + static_cast<int32_t>(i);
                rec.pad = 0;
                rec.sum = l.sum;
                rec.sum_sq = l.sum_sq;
                rec.samples = l.samples;
                rec.cost = l.cost;
            }
        }
    }
    if (trace) {
        const auto t_end = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[expmc] driver rows %lld | setup %.2f ms rounds %.2f ms output %.2f ms\n",
                     static_cast<long long>(nrows), ms(t_setup, t_rounds), ms(t_rounds, t_out), ms(t_out, t_end));
    }
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EXPMC_OK;
    } catch (const Status& s) {
        set_error(s.what());
        return s.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return EXPMC_EINTERNAL;
    }
}

}  // namespace

extern "C" {

int expmc_mlmc_driver_rows(expmc_ctx* ctx, double beta, const expmc_options* opt, int64_t nrows, const int64_t* rows,
                           const uint64_t* row_seed, expmc_result* out, expmc_level_record* levels,
                           int32_t max_levels) {
    return guarded([&] {
        if (!ctx || !opt || (nrows > 0 && (!rows || !row_seed || !out)))
            throw Status(EXPMC_EINVAL, "null argument");
        drive_rows(ctx, EXPMC_LANE_ENTRY, beta, *opt, nrows, rows, row_seed, out, levels, max_levels);
    });
}

int expmc_mlmc_driver(expmc_ctx* ctx, int64_t entry, double beta, const expmc_options* opt, expmc_result* out,
                      expmc_level_record* levels, int32_t max_levels) {
    return guarded([&] {
        if (!ctx || !opt || !out) throw Status(EXPMC_EINVAL, "null argument");
        const uint64_t seed = opt->seed;
        drive_rows(ctx, EXPMC_LANE_ENTRY, beta, *opt, 1, &entry, &seed, out, levels, max_levels);
    });
}

int expmc_mlmc_driver_forward(expmc_ctx* ctx, double beta, const expmc_options* opt, int64_t nruns,
                              const uint64_t* seeds, expmc_result* out, expmc_level_record* levels,
                              int32_t max_levels) {
    return guarded([&] {
        if (!ctx || !opt || (nruns > 0 && !out)) throw Status(EXPMC_EINVAL, "null argument");
        const uint64_t one = opt->seed;
        if (!seeds) {
            if (nruns != 1) throw Status(EXPMC_EINVAL, "null argument");
            seeds = &one;
        }
        drive_rows(ctx, EXPMC_LANE_FORWARD, beta, *opt, nruns, nullptr, seeds, out, levels, max_levels);
    });
}

int expmc_mlmc_driver_fem(expmc_ctx* ctx, double beta, const expmc_options* opt, int64_t nrows, const int64_t* rows,
                          const uint64_t* row_seed, expmc_result* out, expmc_level_record* levels,
                          int32_t max_levels) {
    return guarded([&] {
        if (!ctx || !opt || (nrows > 0 && (!rows || !row_seed || !out)))
            throw Status(EXPMC_EINVAL, "null argument");
        drive_rows(ctx, EXPMC_LANE_FEM, beta, *opt, nrows, rows, row_seed, out, levels, max_levels);
    });
}

int expmc_initial_level(double beta, double d_max, int32_t* out) {
    return guarded([&] { *out = initial_level_impl(beta, d_max); });
}

int expmc_optimal_allocation(int64_t n, const double* v, const double* c, double eps, uint64_t* out) {
    return guarded([&] { optimal_allocation_impl(static_cast<size_t>(n), v, c, eps, out); });
}

int expmc_bias_estimate(int64_t n, const double* means, double* out) {
    return guarded([&] { *out = bias_estimate_impl(static_cast<size_t>(n), means); });
}

}  // extern "C"
