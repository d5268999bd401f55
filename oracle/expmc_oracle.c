/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the MLMC random-walk estimator.
 *
 * Plain-C restatement of the reference (arXiv 1904.12754 `expmc`, /root/reference/proj/core);
 * see expmc_oracle.h for the contract.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline/reference legs may load this library, and only as the checker.
 *
 * Compile with -ffp-contract=off (oracle/Makefile): every expression below is evaluated in
 * the same order and with the same roundings as the reference's C++.
 */
#include "expmc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- Philox4x32-10
 * rng.hpp:21-73.  key = (seed_lo, seed_hi); counter = (block, sample_lo, sample_hi,
 * level&0xFFFFFF | lane<<24); each block yields two 64-bit words, consumed (c2,c3) first,
 * then (c0,c1); uniform = (bits >> 11) * 2^-53.                                        */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_stream_init(orc_stream* s, uint64_t seed, uint32_t level, uint64_t sample, uint32_t lane) {
    s->key[0] = (uint32_t)seed;
    s->key[1] = (uint32_t)(seed >> 32);
    s->base[0] = 0u;
    s->base[1] = (uint32_t)sample;
    s->base[2] = (uint32_t)(sample >> 32);
    s->base[3] = (level & 0xFFFFFFu) | (lane << 24);
    s->block = 0;
    s->buf[0] = s->buf[1] = 0;
    s->cached = 0;
}

static void philox_refill(orc_stream* s) { /* rng.hpp:54-66 */
    uint32_t c[4] = {s->block++, s->base[1], s->base[2], s->base[3]};
    uint32_t k0 = s->key[0], k1 = s->key[1];
    for (int r = 0; r < 10; ++r) { /* round(): rng.hpp:44-52 */
        const uint64_t p0 = (uint64_t)PHILOX_M0 * c[0];
        const uint64_t p1 = (uint64_t)PHILOX_M1 * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += PHILOX_W0;
        k1 += PHILOX_W1;
    }
    s->buf[0] = ((uint64_t)c[0] << 32) | c[1];
    s->buf[1] = ((uint64_t)c[2] << 32) | c[3];
    s->cached = 2;
}

double orc_next_uniform(orc_stream* s) { /* rng.hpp:32-36 */
    if (s->cached == 0) philox_refill(s);
    const uint64_t bits = s->buf[--s->cached];
    return (double)(bits >> 11) * 0x1.0p-53;
}

void orc_uniforms(uint64_t seed, uint32_t level, uint64_t sample, uint32_t lane, int64_t count,
                  double* out) {
    orc_stream s;
    orc_stream_init(&s, seed, level, sample, lane);
    for (int64_t i = 0; i < count; ++i) out[i] = orc_next_uniform(&s);
}

/* ---------------------------------------------------------------- decomposition
 * decompose_impl, chain.cpp:15-71 (row_scale empty).  Input is a canonical CSR
 * (sorted columns, no duplicates) as SparseMatrix stores it (sparse.hpp:23-26).        */
int orc_decompose(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                  orc_chain** out) {
    if (n < 0) return fail(1, "matrix dimension must be nonnegative");
    const int64_t nnz = row_ptr[n];
    orc_chain* c = (orc_chain*)calloc(1, sizeof *c);
    c->n = n;
    c->d = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    c->rate = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    c->row_ptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    c->cdf = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    c->target = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    c->sign = (uint8_t*)malloc((size_t)(nnz > 0 ? nnz : 1));
    c->weight = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    int64_t e = 0;
    double d_sum = 0.0;
    double d_max = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        double diag = 0.0, rate = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            const double v = 1.0 * val[k]; /* scale * vals[k], scale = 1 (chain.cpp:34) */
            if (!isfinite(v)) {
                orc_chain_free(c);
                return fail(1, "matrix entry is NaN or Inf");
            }
            if (col[k] == i) {
                diag = v;
                continue;
            }
            if (v == 0.0) continue;
            const double w = fabs(v);
            rate += w;
            c->weight[e] = w;
            c->cdf[e] = rate;
            c->target[e] = col[k];
            c->sign[e] = v < 0.0 ? 1 : 0;
            ++e;
        }
        c->rate[i] = rate;
        const double di = diag + rate;
        c->d[i] = di;
        c->row_ptr[i + 1] = e;
        d_sum += di;
        if (di > d_max) d_max = di; /* std::max(d_max, di) */
        if (rate > 0.0) {
            const int64_t b = c->row_ptr[i], end = c->row_ptr[i + 1];
            for (int64_t k = b; k < end - 1; ++k) c->cdf[k] /= rate;
            c->cdf[end - 1] = 1.0;
        }
    }
    c->nedges = e;
    c->d_max = n > 0 ? d_max : 0.0;
    c->d_bar = n > 0 ? d_sum / (double)n : 0.0;
    *out = c;
    return 0;
}

void orc_chain_free(orc_chain* c) {
    if (!c) return;
    free(c->d); free(c->rate); free(c->row_ptr); free(c->cdf);
    free(c->target); free(c->sign); free(c->weight); free(c);
}

int64_t orc_chain_n(const orc_chain* c) { return c->n; }
int64_t orc_chain_edges(const orc_chain* c) { return c->nedges; }

void orc_chain_export(const orc_chain* c, double* d, double* rate, int64_t* row_ptr, double* cdf,
                      int64_t* target, uint8_t* sign, double* weight, double* d_max, double* d_bar) {
    const size_t n = (size_t)c->n, e = (size_t)c->nedges;
    memcpy(d, c->d, n * sizeof(double));
    memcpy(rate, c->rate, n * sizeof(double));
    memcpy(row_ptr, c->row_ptr, (n + 1) * sizeof(int64_t));
    memcpy(cdf, c->cdf, e * sizeof(double));
    memcpy(target, c->target, e * sizeof(int64_t));
    memcpy(sign, c->sign, e);
    memcpy(weight, c->weight, e * sizeof(double));
    *d_max = c->d_max;
    *d_bar = c->d_bar;
}

/* ---------------------------------------------------------------- path sampler */

/* evolve_common, paths.cpp:44-71 */
static int64_t evolve_common(const orc_chain* c, int64_t state, int* sign, uint64_t* draws,
                             uint64_t* jumps, double remaining, double first_q, orc_stream* s) {
    double q = first_q;
    for (;;) {
        const double rate = c->rate[state];
        if (rate == 0.0) break;
        const double u = orc_next_uniform(s);
        ++*draws;
        if (u >= q) break;
        remaining -= -log1p(-u) / rate;
        ++*jumps;
        const double v = orc_next_uniform(s);
        /* std::upper_bound(cdf + begin, cdf + end, v) */
        int64_t lo = c->row_ptr[state], count = c->row_ptr[state + 1] - lo;
        const int64_t end = c->row_ptr[state + 1];
        while (count > 0) {
            const int64_t step = count / 2;
            const int64_t it = lo + step;
            if (!(v < c->cdf[it])) {
                lo = it + 1;
                count -= step + 1;
            } else {
                count = step;
            }
        }
        const int64_t kk = lo < end ? lo : end - 1;
        if (c->sign[kk]) *sign = -*sign;
        state = c->target[kk];
        if (remaining <= 0.0) break;
        q = -expm1(-c->rate[state] * remaining);
    }
    return state;
}

typedef struct {
    double fine, coarse;
    uint64_t cost, jumps;
    int64_t end_state;
} orc_sample;

/* make_initial_distribution, paths.cpp:12-28: forward mode's start-state CDF over u. */
typedef struct {
    double* cdf;
    int64_t n;
    double total;
} orc_init;

static int init_build(const double* u, int64_t n, orc_init* init) {
    init->cdf = NULL;
    init->n = n;
    init->total = 0.0;
    if (n <= 0) return fail(1, "forward sampling requires sum(u) > 0");
    init->cdf = (double*)malloc((size_t)n * sizeof(double));
    double total = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        if (u[j] < 0.0) {
            free(init->cdf);
            init->cdf = NULL;
            return fail(1, "forward sampling requires a nonnegative vector");
        }
        total += u[j];
        init->cdf[j] = total;
    }
    if (!(total > 0.0)) {
        free(init->cdf);
        init->cdf = NULL;
        return fail(1, "forward sampling requires sum(u) > 0");
    }
    for (int64_t j = 0; j < n; ++j) init->cdf[j] /= total;
    init->cdf[n - 1] = 1.0;
    init->total = total;
    return 0;
}

/* sample_initial, paths.cpp:32-36: upper_bound of one uniform in the CDF. */
static int64_t sample_initial(const orc_init* init, orc_stream* s) {
    const double v = orc_next_uniform(s);
    int64_t lo = 0, count = init->n;
    while (count > 0) {
        const int64_t step = count / 2;
        if (!(v < init->cdf[lo + step])) {
            lo += step + 1;
            count -= step + 1;
        } else {
            count = step;
        }
    }
    return lo;
}

/* LevelSampler::single, paths.cpp:99-114 (nojump_ from the ctor, paths.cpp:88-90); with
 * init != NULL LevelSampler::forward_single, paths.cpp:144-157 (start drawn from u, the
 * terminal factor sum(u) instead of u[end]). */
static orc_sample sample_single(const orc_chain* c, const double* u, int64_t entry, double dt,
                                int64_t steps, orc_stream* s, const orc_init* init) {
    int64_t state = init ? sample_initial(init, s) : entry;
    int sign = 1;
    uint64_t draws = 0, jumps = 0;
    double expo = 0.0;
    for (int64_t n = 0; n < steps; ++n) {
        const int64_t s0 = state;
        const double q = -expm1(-c->rate[state] * dt);
        state = evolve_common(c, state, &sign, &draws, &jumps, dt, q, s);
        expo += dt * 0.5 * (c->d[s0] + c->d[state]);
    }
    orc_sample r;
    r.fine = sign * exp(expo) * (init ? init->total : u[state]);
    r.coarse = 0.0;
    r.cost = draws + (uint64_t)steps;
    r.jumps = jumps;
    r.end_state = state;
    return r;
}

/* LevelSampler::coupled, paths.cpp:116-141; forward_coupled with init, paths.cpp:159-181 */
static orc_sample sample_coupled(const orc_chain* c, const double* u, int64_t entry, double dt,
                                 int64_t steps, orc_stream* s, const orc_init* init) {
    int64_t state = init ? sample_initial(init, s) : entry;
    int sign = 1;
    uint64_t draws = 0, jumps = 0;
    double coarse = 0.0, delta = 0.0;
    for (int64_t m = 0; m < steps / 2; ++m) {
        const int64_t s0 = state;
        state = evolve_common(c, state, &sign, &draws, &jumps, dt, -expm1(-c->rate[state] * dt), s);
        const int64_t s1 = state;
        state = evolve_common(c, state, &sign, &draws, &jumps, dt, -expm1(-c->rate[state] * dt), s);
        const double half_ends = 0.5 * (c->d[s0] + c->d[state]);
        coarse += dt * (c->d[s0] + c->d[state]);
        delta += dt * (c->d[s1] - half_ends);
    }
    const double uf = sign * (init ? init->total : u[state]);
    orc_sample r;
    r.fine = uf * exp(coarse + delta);
    r.coarse = uf * exp(coarse);
    r.cost = draws + (uint64_t)steps;
    r.jumps = jumps;
    r.end_state = state;
    return r;
}

static int check_level(int level);

/* scaled_simpson (mlmc.cpp:66-75): composite Simpson weight of node j of `panels`, scaled by
 * the step through h = step / 3. */
static double simpson_w(int64_t j, int64_t panels, double h) {
    const int end = (j == 0 || j == panels);
    return h * (end ? 1.0 : (j % 2 == 1 ? 4.0 : 2.0));
}

typedef struct {
    double value, eta_f, eta_c, integ_f, integ_c;
    uint64_t cost, jumps;
    int64_t end_state;
} orc_fem_sample;

/* LevelSampler::fem_single, paths.cpp:183-203 (weights: run_level_ex, mlmc.cpp:89-90) */
static orc_fem_sample fem_single(const orc_chain* c, const double* u, const double* load, int64_t entry,
                                 double dt, int64_t steps, orc_stream* s) {
    const double h = dt / 3.0;
    int64_t state = entry;
    int sign = 1;
    uint64_t draws = 0, jumps = 0;
    double expo = 0.0;
    double integ = simpson_w(0, steps, h) * load[entry];
    for (int64_t n = 0; n < steps; ++n) {
        const int64_t s0 = state;
        state = evolve_common(c, state, &sign, &draws, &jumps, dt, -expm1(-c->rate[state] * dt), s);
        expo += dt * 0.5 * (c->d[s0] + c->d[state]);
        integ += simpson_w(n + 1, steps, h) * sign * exp(expo) * load[state];
    }
    orc_fem_sample r;
    r.value = sign * exp(expo) * u[state] + integ;
    r.eta_f = r.eta_c = r.integ_f = r.integ_c = 0.0;
    r.cost = draws + (uint64_t)steps;
    r.jumps = jumps;
    r.end_state = state;
    return r;
}

/* LevelSampler::fem_coupled, paths.cpp:205-245; the run_level sample
 * u[terminal] (eta_f - eta_c) + (integ_f - integ_c), mlmc.cpp:126-133 */
static orc_fem_sample fem_coupled(const orc_chain* c, const double* u, const double* load, int64_t entry,
                                  double dt, int64_t steps, orc_stream* s) {
    const double hf = dt / 3.0, hc = (2.0 * dt) / 3.0;
    const int64_t half = steps / 2;
    int64_t state = entry;
    int sign = 1;
    uint64_t draws = 0, jumps = 0;
    double coarse = 0.0, delta = 0.0, eta_f = 1.0, eta_c = 1.0;
    double integ_f = simpson_w(0, steps, hf) * load[entry];
    double integ_c = simpson_w(0, half, hc) * load[entry];
    for (int64_t m = 0; m < half; ++m) {
        const int64_t s0 = state;
        state = evolve_common(c, state, &sign, &draws, &jumps, dt, -expm1(-c->rate[state] * dt), s);
        const int64_t s1 = state;
        const double mid = coarse + delta + dt * 0.5 * (c->d[s0] + c->d[s1]);
        integ_f += simpson_w(2 * m + 1, steps, hf) * sign * exp(mid) * load[s1];
        state = evolve_common(c, state, &sign, &draws, &jumps, dt, -expm1(-c->rate[state] * dt), s);
        const double half_ends = 0.5 * (c->d[s0] + c->d[state]);
        coarse += dt * (c->d[s0] + c->d[state]);
        delta += dt * (c->d[s1] - half_ends);
        eta_f = sign * exp(coarse + delta);
        eta_c = sign * exp(coarse);
        integ_f += simpson_w(2 * m + 2, steps, hf) * eta_f * load[state];
        integ_c += simpson_w(m + 1, half, hc) * eta_c * load[state];
    }
    orc_fem_sample r;
    const double du = u[state] * (eta_f - eta_c);
    const double di = integ_f - integ_c;
    r.value = du + di;
    r.eta_f = eta_f;
    r.eta_c = eta_c;
    r.integ_f = integ_f;
    r.integ_c = integ_c;
    r.cost = draws + (uint64_t)steps;
    r.jumps = jumps;
    r.end_state = state;
    return r;
}

static int check_fem(const orc_chain* c, const double* load, int64_t entry, int level, int base) {
    if (entry < 0 || entry >= c->n) return fail(2, "entry index outside matrix");
    if (!load) return fail(1, "load length does not match decomposition");
    if (!base && level < 2) return fail(1, "coupled quadrature needs a step count divisible by 4");
    return 0;
}

int orc_fem_samples(const orc_chain* c, const double* u, const double* load, int64_t entry, double beta,
                    int level, int base, uint64_t seed, int64_t count, const uint64_t* sample_idx,
                    double* value, double* eta_f, double* eta_c, double* integ_f, double* integ_c,
                    int64_t* end_state, uint64_t* cost, uint64_t* jumps) {
    int rc = check_level(level);
    if (rc || (rc = check_fem(c, load, entry, level, base))) return rc;
    const int64_t steps = (int64_t)1 << level;
    const double dt = beta / (double)steps;
    if (!(dt > 0.0)) return fail(1, "step size must be positive");
    for (int64_t i = 0; i < count; ++i) {
        orc_stream s;
        orc_stream_init(&s, seed, (uint32_t)level, sample_idx[i], ORC_LANE_FEM);
        const orc_fem_sample r = base ? fem_single(c, u, load, entry, dt, steps, &s)
                                      : fem_coupled(c, u, load, entry, dt, steps, &s);
        value[i] = r.value;
        if (eta_f) eta_f[i] = r.eta_f;
        if (eta_c) eta_c[i] = r.eta_c;
        if (integ_f) integ_f[i] = r.integ_f;
        if (integ_c) integ_c[i] = r.integ_c;
        if (end_state) end_state[i] = base ? -1 : r.end_state;
        if (cost) cost[i] = r.cost;
        if (jumps) jumps[i] = r.jumps;
    }
    return 0;
}

static int check_level(int level) {
    if (level < 0 || level > 62) return fail(1, "level outside [0, 62]");
    return 0;
}

int orc_samples(const orc_chain* c, const double* u, int64_t entry, double beta, int level,
                int base, uint64_t seed, uint32_t lane, int64_t count, const uint64_t* sample_idx,
                double* fine, double* coarse, uint64_t* cost, uint64_t* jumps, int64_t* end_state) {
    int rc = check_level(level);
    if (rc) return rc;
    const int forward = lane == ORC_LANE_FORWARD;
    if (!forward && (entry < 0 || entry >= c->n)) return fail(2, "entry index outside matrix");
    const int64_t steps = (int64_t)1 << level;
    const double dt = beta / (double)steps;
    if (!(dt > 0.0)) return fail(1, "step size must be positive");
    if (!base && steps % 2 != 0) return fail(1, "coupled sampling needs an even step count");
    orc_init init = {NULL, 0, 0.0};
    if (forward && (rc = init_build(u, c->n, &init))) return rc;
    const orc_init* ip = forward ? &init : NULL;
    for (int64_t i = 0; i < count; ++i) {
        orc_stream s;
        orc_stream_init(&s, seed, (uint32_t)level, sample_idx[i], lane);
        const orc_sample r = base ? sample_single(c, u, entry, dt, steps, &s, ip)
                                  : sample_coupled(c, u, entry, dt, steps, &s, ip);
        fine[i] = r.fine;
        coarse[i] = r.coarse;
        cost[i] = r.cost;
        if (jumps) jumps[i] = r.jumps;
        if (end_state) end_state[i] = r.end_state;
    }
    free(init.cdf);
    return 0;
}

/* run_level_ex, mlmc.cpp:76-148 with parallel_samples<SumAcc>, parallel.hpp:20-76:
 * 512-sample chunks by absolute index, sequential sums inside a chunk, chunk partials
 * combined in ascending order from a zero accumulator.                                 */
#define ORC_CHUNK 512u

int orc_run_level(const orc_chain* c, const double* u, int64_t entry, double beta, int level,
                  int base, uint64_t first, uint64_t count, uint64_t seed, uint32_t lane,
                  int threads, orc_level_stats* out) {
    int rc = check_level(level);
    if (rc) return rc;
    const int forward = lane == ORC_LANE_FORWARD;
    if (!forward && (entry < 0 || entry >= c->n)) return fail(2, "entry index outside matrix");
    if (!(beta > 0.0)) return fail(1, "beta must be positive");
    const int64_t steps = (int64_t)1 << level;
    const double dt = beta / (double)steps;
    if (!base && steps % 2 != 0) return fail(1, "coupled sampling needs an even step count");
    memset(out, 0, sizeof *out);
    if (count == 0) return 0;
    orc_init init = {NULL, 0, 0.0};
    if (forward && (rc = init_build(u, c->n, &init))) return rc;  /* mlmc.cpp:86 */
    const orc_init* ip = forward ? &init : NULL;
    const uint64_t first_chunk = first / ORC_CHUNK;
    const uint64_t last_chunk = (first + count - 1) / ORC_CHUNK;
    const int64_t nch = (int64_t)(last_chunk - first_chunk + 1);
    orc_level_stats* part = (orc_level_stats*)calloc((size_t)nch, sizeof *part);
    if (threads <= 0) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t ci = 0; ci < nch; ++ci) {
        const uint64_t chunk = first_chunk + (uint64_t)ci;
        const uint64_t lo = first > chunk * ORC_CHUNK ? first : chunk * ORC_CHUNK;
        const uint64_t hi = (first + count) < (chunk + 1) * ORC_CHUNK ? (first + count) : (chunk + 1) * ORC_CHUNK;
        orc_level_stats a = {0.0, 0.0, 0, 0, 0};
        for (uint64_t smp = lo; smp < hi; ++smp) {
            orc_stream s;
            orc_stream_init(&s, seed, (uint32_t)level, smp, lane);
            double x;
            orc_sample r;
            if (base) {
                r = sample_single(c, u, entry, dt, steps, &s, ip);
                x = r.fine;
            } else {
                r = sample_coupled(c, u, entry, dt, steps, &s, ip);
                x = r.fine - r.coarse;
            }
            a.sum += x; /* SumAcc::add, parallel.hpp:64-69 */
            a.sum_sq += x * x;
            a.cost += r.cost;
            a.jumps += r.jumps;
            ++a.samples;
        }
        part[ci] = a;
    }
    for (int64_t ci = 0; ci < nch; ++ci) { /* SumAcc::combine in chunk order, parallel.hpp:52 */
        out->sum += part[ci].sum;
        out->sum_sq += part[ci].sum_sq;
        out->cost += part[ci].cost;
        out->jumps += part[ci].jumps;
        out->samples += part[ci].samples;
    }
    free(part);
    free(init.cdf);
    return 0;
}

/* run_level_ex in fem mode (mlmc.cpp:76-148): the same 512-sample chunking, plus the SumAcc
 * side channel `extra` = sum of (integ_f - integ_c) of the coupled samples (parallel.hpp:60). */
int orc_fem_run_level(const orc_chain* c, const double* u, const double* load, int64_t entry, double beta,
                      int level, int base, uint64_t first, uint64_t count, uint64_t seed, int threads,
                      orc_level_stats* out, double* integ_sum) {
    int rc = check_level(level);
    if (rc) return rc;
    if (entry < 0 || entry >= c->n) return fail(2, "entry index outside matrix");
    if (!load) return fail(1, "load length does not match decomposition");
    if (!(beta > 0.0)) return fail(1, "beta must be positive");
    const int64_t steps = (int64_t)1 << level;
    const double dt = beta / (double)steps;
    memset(out, 0, sizeof *out);
    *integ_sum = 0.0;
    if (count == 0) return 0;
    if (!base && level < 2) return fail(1, "coupled quadrature needs a step count divisible by 4");
    const uint64_t first_chunk = first / ORC_CHUNK;
    const uint64_t last_chunk = (first + count - 1) / ORC_CHUNK;
    const int64_t nch = (int64_t)(last_chunk - first_chunk + 1);
    orc_level_stats* part = (orc_level_stats*)calloc((size_t)nch, sizeof *part);
    double* extra = (double*)calloc((size_t)nch, sizeof *extra);
    if (threads <= 0) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t ci = 0; ci < nch; ++ci) {
        const uint64_t chunk = first_chunk + (uint64_t)ci;
        const uint64_t lo = first > chunk * ORC_CHUNK ? first : chunk * ORC_CHUNK;
        const uint64_t hi = (first + count) < (chunk + 1) * ORC_CHUNK ? (first + count) : (chunk + 1) * ORC_CHUNK;
        orc_level_stats a = {0.0, 0.0, 0, 0, 0};
        double ex = 0.0;
        for (uint64_t smp = lo; smp < hi; ++smp) {
            orc_stream s;
            orc_stream_init(&s, seed, (uint32_t)level, smp, ORC_LANE_FEM);
            const orc_fem_sample r = base ? fem_single(c, u, load, entry, dt, steps, &s)
                                          : fem_coupled(c, u, load, entry, dt, steps, &s);
            a.sum += r.value;
            a.sum_sq += r.value * r.value;
            a.cost += r.cost;
            a.jumps += r.jumps;
            ++a.samples;
            if (!base) ex += r.integ_f - r.integ_c;
        }
        part[ci] = a;
        extra[ci] = ex;
    }
    for (int64_t ci = 0; ci < nch; ++ci) {
        out->sum += part[ci].sum;
        out->sum_sq += part[ci].sum_sq;
        out->cost += part[ci].cost;
        out->jumps += part[ci].jumps;
        out->samples += part[ci].samples;
        *integ_sum += extra[ci];
    }
    free(part);
    free(extra);
    return 0;
}

/* ---------------------------------------------------------------- classical MC
 * mc_single_entry / mc_forward_scalar (mc.cpp:42-76): samples [0, m) at dt with
 * steps = round(beta / dt), key level = bit_width(steps); WelfordAcc per 512-sample chunk
 * (parallel.hpp:80-92), chunks merged in order by Chan's formula (parallel.hpp:93-104). */
typedef struct {
    uint64_t n;
    double mean, m2;
    uint64_t cost, jumps;
} orc_welford;

static void welford_merge(orc_welford* a, const orc_welford* o) {
    if (o->n == 0) return;
    if (a->n == 0) {
        *a = *o;
        return;
    }
    const double delta = o->mean - a->mean;
    const double total = (double)(a->n + o->n);
    a->mean += delta * ((double)o->n / total);
    a->m2 += o->m2 + delta * delta * ((double)a->n * (double)o->n / total);
    a->n += o->n;
    a->cost += o->cost;
    a->jumps += o->jumps;
}

int orc_mc(const orc_chain* c, const double* u, int64_t entry, double beta, double dt, uint64_t samples,
           uint64_t seed, uint32_t lane, int threads, orc_mc_result* out) {
    if (samples < 2) return fail(1, "at least 2 samples required");
    const int forward = lane == ORC_LANE_FORWARD;
    if (!forward && (entry < 0 || entry >= c->n)) return fail(2, "entry index outside matrix");
    if (!(dt > 0.0) || !(beta > 0.0)) return fail(1, "beta and dt must be positive");
    const double ratio = beta / dt;
    const double rounded = round(ratio);
    if (fabs(ratio - rounded) > 1e-9 * ratio || rounded < 1.0)
        return fail(1, "beta/dt must be a positive integer step count");
    const int64_t steps = (int64_t)rounded;
    const uint32_t key = (uint32_t)(64 - __builtin_clzll((unsigned long long)steps));
    orc_init init = {NULL, 0, 0.0};
    int rc;
    if (forward && (rc = init_build(u, c->n, &init))) return rc;
    const orc_init* ip = forward ? &init : NULL;
    const int64_t nch = (int64_t)((samples - 1) / ORC_CHUNK + 1);
    orc_welford* part = (orc_welford*)calloc((size_t)nch, sizeof *part);
    if (threads <= 0) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t ci = 0; ci < nch; ++ci) {
        const uint64_t lo = (uint64_t)ci * ORC_CHUNK;
        const uint64_t hi = samples < lo + ORC_CHUNK ? samples : lo + ORC_CHUNK;
        orc_welford a = {0, 0.0, 0.0, 0, 0};
        for (uint64_t smp = lo; smp < hi; ++smp) {
            orc_stream s;
            orc_stream_init(&s, seed, key, smp, lane);
            const orc_sample r = sample_single(c, u, entry, dt, steps, &s, ip);
            ++a.n; /* WelfordAcc::add */
            const double delta = r.fine - a.mean;
            a.mean += delta / (double)a.n;
            a.m2 += delta * (r.fine - a.mean);
            a.cost += r.cost;
            a.jumps += r.jumps;
        }
        part[ci] = a;
    }
    orc_welford t = {0, 0.0, 0.0, 0, 0};
    for (int64_t ci = 0; ci < nch; ++ci) welford_merge(&t, &part[ci]);
    free(part);
    free(init.cdf);
    out->estimate = t.mean;
    const double var = t.n > 1 ? (t.m2 / (double)(t.n - 1) > 0.0 ? t.m2 / (double)(t.n - 1) : 0.0) : 0.0;
    out->std_error = t.n > 1 ? sqrt(var / (double)t.n) : 0.0;
    out->samples = t.n;
    out->dt = dt;
    out->steps = steps;
    out->wall_cost = t.cost;
    out->jumps = t.jumps;
    return 0;
}

/* ---------------------------------------------------------------- driver helpers */

int orc_initial_level(double beta, double d_max, int* out) { /* mlmc.cpp:19-23 */
    if (!(beta > 0.0)) return fail(1, "beta must be positive");
    if (!(d_max > 0.0)) {
        *out = 0;
        return 0;
    }
    const long r = lround(log2(2.0 * beta * d_max));
    *out = (int)(r > 0 ? r : 0);
    return 0;
}

int orc_optimal_allocation(int64_t n, const double* v, const double* c, double eps, uint64_t* out) {
    /* mlmc.cpp:25-43 */
    if (!(eps > 0.0)) return fail(1, "epsilon must be positive");
    double s = 0.0;
    for (int64_t l = 0; l < n; ++l) {
        if (v[l] < 0.0 || !(c[l] > 0.0)) return fail(1, "require V_l >= 0 and C_l > 0");
        s += sqrt(v[l] * c[l]);
    }
    const double scale = 2.0 / (eps * eps) * s;
    for (int64_t l = 0; l < n; ++l) {
        const double raw = scale * sqrt(v[l] / c[l]);
        const uint64_t m = (uint64_t)ceil(raw);
        out[l] = m > 2 ? m : 2;
    }
    return 0;
}

int orc_bias_estimate(int64_t n, const double* means, double* out) { /* mlmc.cpp:45-51 */
    if (n < 2) return fail(1, "bias estimate needs at least two coupled levels");
    const double last = fabs(means[n - 1]);
    const double prev = fabs(means[n - 2]);
    const double p4 = prev / 4.0;
    *out = (last > p4 ? last : p4) / 3.0;
    return 0;
}

typedef struct {
    double sum, sum_sq;
    uint64_t samples, cost, jumps;
    double integ; /* fem: Level::integ_sum, mlmc.cpp:184-198 */
} lvl_t;

static double lvl_mean(const lvl_t* l) { return l->samples ? l->sum / (double)l->samples : 0.0; }
static double lvl_var(const lvl_t* l) { /* LevelStats::variance, mlmc.cpp:13-17 */
    if (l->samples < 2) return 0.0;
    const double m = lvl_mean(l);
    const double v = l->sum_sq / (double)l->samples - m * m;
    return v > 0.0 ? v : 0.0;
}
static double lvl_unit_cost(const lvl_t* l) {
    return l->samples ? (double)l->cost / (double)l->samples : 0.0;
}

#define ORC_MAX_LEVELS 64

/* mlmc_driver, mlmc.cpp:170-260, entry (lane 0), forward (lane 1) or fem (lane 2, with load;
 * quad = the result's quadrature_bound) mode, one run at a time */
static int driver_one(const orc_chain* c, const double* u, int64_t entry, double beta,
                      const orc_options* o, uint64_t seed, uint32_t lane, const double* load,
                      orc_result* res, double* quad_out, orc_level_record* rec, int32_t max_levels) {
    if (lane != ORC_LANE_FORWARD && (entry < 0 || entry >= c->n)) return fail(2, "entry index outside matrix");
    if (!(beta > 0.0)) return fail(1, "beta must be positive");
    if (!(o->epsilon > 0.0)) return fail(1, "epsilon must be positive");
    int l0;
    if (o->l0_override >= 0) {
        l0 = o->l0_override;
    } else {
        int rc = orc_initial_level(beta, c->d_max, &l0);
        if (rc) return rc;
    }
    if (lane == ORC_LANE_FEM && l0 < 1) l0 = 1; /* mlmc.cpp:177 */
    const int cap = l0 + o->max_levels_above_l0;
    const double target = o->epsilon / sqrt(2.0);
    lvl_t lv[ORC_MAX_LEVELS];
    memset(lv, 0, sizeof lv);
    int nlv = 0;
#define EXTEND(level, add)                                                                 \
    do {                                                                                   \
        orc_level_stats d_;                                                                \
        double ig_ = 0.0;                                                                  \
        lvl_t* e_ = &lv[(level)-l0];                                                       \
        int rc_ = lane == ORC_LANE_FEM                                                     \
                      ? orc_fem_run_level(c, u, load, entry, beta, (level), (level) == l0,  \
                                          e_->samples, (add), seed, o->threads, &d_, &ig_) \
                      : orc_run_level(c, u, entry, beta, (level), (level) == l0,           \
                                      e_->samples, (add), seed, lane, o->threads, &d_);    \
        if (rc_) return rc_;                                                               \
        e_->integ += ig_;                                                                  \
        e_->sum += d_.sum;                                                                 \
        e_->sum_sq += d_.sum_sq;                                                           \
        e_->samples += d_.samples;                                                         \
        e_->cost += d_.cost;                                                               \
        e_->jumps += d_.jumps;                                                             \
    } while (0)

    int top = l0 + 4 < cap ? l0 + 4 : cap;
    for (int l = l0; l <= top; ++l) {
        if (nlv >= ORC_MAX_LEVELS) return fail(1, "too many levels");
        ++nlv;
        EXTEND(l, o->warmup);
    }
    double stat_error = 0.0, bias = 0.0, quad = 0.0;
    int converged = 0;
    for (int iter = 0; iter < o->max_iterations; ++iter) {
        double v[ORC_MAX_LEVELS], cc[ORC_MAX_LEVELS];
        uint64_t want[ORC_MAX_LEVELS];
        for (int i = 0; i < nlv; ++i) {
            v[i] = lvl_var(&lv[i]);
            const double uc = lvl_unit_cost(&lv[i]);
            cc[i] = uc > 1.0 ? uc : 1.0;
        }
        int rc = orc_optimal_allocation(nlv, v, cc, o->epsilon, want);
        if (rc) return rc;
        for (int i = 0; i < nlv; ++i)
            if (want[i] > lv[i].samples) EXTEND(l0 + i, want[i] - lv[i].samples);
        double vt = 0.0;
        for (int i = 0; i < nlv; ++i) vt += lvl_var(&lv[i]) / (double)lv[i].samples;
        stat_error = sqrt(vt);
        double means[ORC_MAX_LEVELS];
        for (int i = 1; i < nlv; ++i) means[i - 1] = lvl_mean(&lv[i]);
        rc = orc_bias_estimate(nlv - 1, means, &bias);
        if (rc) return rc;
        if (lane == ORC_LANE_FEM) { /* quad = bias_estimate(integ_means), mlmc.cpp:226-235 */
            double im[ORC_MAX_LEVELS];
            for (int i = 1; i < nlv; ++i) im[i - 1] = lv[i].integ / (double)lv[i].samples;
            rc = orc_bias_estimate(nlv - 1, im, &quad);
            if (rc) return rc;
        }
        if (stat_error <= target && bias <= target) {
            converged = 1;
            break;
        }
        if (bias > target) {
            if (top == cap) break;
            ++top;
            if (nlv >= ORC_MAX_LEVELS) return fail(1, "too many levels");
            ++nlv;
            EXTEND(top, o->warmup);
        }
    }
#undef EXTEND
    memset(res, 0, sizeof *res);
    res->l0 = l0;
    res->L = top;
    res->statistical_error = stat_error;
    res->bias_estimate = bias;
    res->converged = converged;
    res->nlevels = nlv;
    if (quad_out) *quad_out = quad;
    for (int i = 0; i < nlv; ++i) {
        res->estimate += lvl_mean(&lv[i]);
        res->total_cost += lv[i].cost;
        res->total_jumps += lv[i].jumps;
        res->total_samples += lv[i].samples;
        if (rec && i < max_levels) {
            rec[i].level = l0 + i;
            rec[i].pad = 0;
            rec[i].sum = lv[i].sum;
            rec[i].sum_sq = lv[i].sum_sq;
            rec[i].samples = lv[i].samples;
            rec[i].cost = lv[i].cost;
        }
    }
    return 0;
}

int orc_mlmc_driver_rows(const orc_chain* c, const double* u, double beta, const orc_options* o,
                         int64_t nrows, const int64_t* rows, const uint64_t* row_seed,
                         orc_result* out, orc_level_record* levels, int32_t max_levels) {
    for (int64_t r = 0; r < nrows; ++r) {
        int rc = driver_one(c, u, rows[r], beta, o, row_seed[r], ORC_LANE_ENTRY, NULL, &out[r], NULL,
                            levels ? levels + r * max_levels : NULL, max_levels);
        if (rc) return rc;
    }
    return 0;
}

int orc_mlmc_driver_forward(const orc_chain* c, const double* u, double beta, const orc_options* o,
                            int64_t nruns, const uint64_t* seeds, orc_result* out,
                            orc_level_record* levels, int32_t max_levels) {
    for (int64_t r = 0; r < nruns; ++r) {
        int rc = driver_one(c, u, 0, beta, o, seeds[r], ORC_LANE_FORWARD, NULL, &out[r], NULL,
                            levels ? levels + r * max_levels : NULL, max_levels);
        if (rc) return rc;
    }
    return 0;
}

int orc_mlmc_driver_fem(const orc_chain* c, const double* u, const double* load, double beta,
                        const orc_options* o, int64_t nrows, const int64_t* rows, const uint64_t* row_seed,
                        orc_result* out, double* quad, orc_level_record* levels, int32_t max_levels) {
    for (int64_t r = 0; r < nrows; ++r) {
        int rc = driver_one(c, u, rows[r], beta, o, row_seed[r], ORC_LANE_FEM, load, &out[r], &quad[r],
                            levels ? levels + r * max_levels : NULL, max_levels);
        if (rc) return rc;
    }
    return 0;
}

/* ---------------------------------------------------------------- deterministic oracle
 * dense_expmv, oracle.cpp:31-60, without the n <= 5000 guard; SpMV rows are independent
 * so the OpenMP split does not change any rounding.                                   */
static double max_abs(const double* v, int64_t n) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs(v[i]);
        if (a > m) m = a; /* std::max(m, |x|) */
    }
    return m;
}

int orc_dense_expmv(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                    const double* u, double beta, int threads, double* out) {
    if (threads <= 0) threads = 1;
    double* colsum = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    const int64_t nnz = row_ptr[n];
    for (int64_t k = 0; k < nnz; ++k) colsum[col[k]] += fabs(val[k]); /* one_norm, oracle.cpp:20-29 */
    double one = 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (colsum[i] > one) one = colsum[i];
    free(colsum);
    const double norm = fabs(beta) * one;
    int64_t stages = (int64_t)ceil(norm);
    if (stages < 1) stages = 1;
    const double h = beta / (double)stages;
    double* x = out;
    memcpy(x, u, (size_t)n * sizeof(double));
    double* term = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double* next = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int64_t s = 0; s < stages; ++s) {
        memcpy(term, x, (size_t)n * sizeof(double));
        double ref = max_abs(x, n);
        for (int k = 1; k <= 64; ++k) {
#pragma omp parallel for schedule(static) num_threads(threads)
            for (int64_t i = 0; i < n; ++i) { /* SparseMatrix::multiply, sparse.cpp:100-109 */
                double acc = 0.0;
                for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) acc += val[j] * term[col[j]];
                next[i] = acc;
            }
            const double cf = h / (double)k;
            for (int64_t i = 0; i < n; ++i) term[i] = cf * next[i];
            for (int64_t i = 0; i < n; ++i) x[i] += term[i];
            const double t = max_abs(term, n);
            const double mx = max_abs(x, n);
            if (mx > ref) ref = mx;
            if (t <= 1e-17 * ref) break;
        }
    }
    free(term);
    free(next);
    return 0;
}

/* ---------------------------------------------------------------- config inputs
 * C1/C2 (BASELINE.json configs[0..1]): 2D 5-point Laplacian on g x g interior
 * nodes, row = y*g + x, diag -4, off-diagonal +1, Dirichlet boundary eliminated; columns
 * ascending.  v_i = stream_for(seed, 0, i, lane 6) (lanes 0-3, 7 are taken by the reference). */
int64_t orc_grid_nnz(int64_t g) { return 5 * g * g - 4 * g; }

void orc_grid_laplacian(int64_t g, int64_t* row_ptr, int64_t* col, double* val) {
    int64_t k = 0;
    row_ptr[0] = 0;
    for (int64_t y = 0; y < g; ++y)
        for (int64_t x = 0; x < g; ++x) {
            const int64_t r = y * g + x;
            if (y > 0) { col[k] = r - g; val[k++] = 1.0; }
            if (x > 0) { col[k] = r - 1; val[k++] = 1.0; }
            col[k] = r; val[k++] = -4.0;
            if (x + 1 < g) { col[k] = r + 1; val[k++] = 1.0; }
            if (y + 1 < g) { col[k] = r + g; val[k++] = 1.0; }
            row_ptr[r + 1] = k;
        }
}

void orc_grid_vector(uint64_t seed, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) {
        orc_stream s;
        orc_stream_init(&s, seed, 0u, (uint64_t)i, 6u);
        out[i] = orc_next_uniform(&s);
    }
}
