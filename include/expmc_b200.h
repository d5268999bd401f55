/* expmc_b200 -- C-ABI of the B200-native MLMC random-walk estimator for e^{tA}v.
 *
 * Drop-in boundary for the hot path of arXiv 1904.12754's reference (`expmc`,
 * /root/reference/proj/core): everything the reference does between "a decomposed matrix
 * and a vector are ready" and "LevelStats / MlmcResult come back" runs behind these entry
 * points on one GPU.  Plain pointers and sizes only; all buffers passed in are caller-owned
 * HOST memory, read or written during the call.  A context owns all device memory of one
 * GPU (one context per process per GPU; multi-GPU = one process per GPU).
 *
 * Error convention: every int-returning call returns EXPMC_OK (0) or a status whose value
 * names the C++ exception type the reference throws for the same input, so the C++ shim
 * (expmc_b200.hpp) can rethrow it.  expmc_last_error() gives the message (thread-local).
 *
 * Thread safety: a context is driven by one host thread at a time (the reference driver is
 * sequential too).  Results are a pure function of (matrix, vector, level,
 * entry, seed, sample-index range): independent of launch geometry and GPU count.
 */
#ifndef EXPMC_B200_H
#define EXPMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EXPMC_OK 0
#define EXPMC_EINVAL 1    /* std::invalid_argument */
#define EXPMC_ERANGE 2    /* std::out_of_range     */
#define EXPMC_EDOMAIN 3   /* std::domain_error     */
#define EXPMC_ECUDA 4     /* CUDA runtime failure (no CPU fallback exists) */
#define EXPMC_ENOTIMPL 5  /* unknown sampling lane                          */
#define EXPMC_EIO 6       /* std::runtime_error: file / parse errors (io.cpp), "path:line: what" */
#define EXPMC_EOVERFLOW 7 /* std::overflow_error (mc_auto: step count beyond 64 bits)            */
#define EXPMC_EINTERNAL 9

/* Path samplers.  REFERENCE: draw-for-draw the reference's evolve_common / single / coupled
 * (paths.cpp:44-141) -- same jump chain, same values, exact parity (default).  EVENT: one
 * exponential clock per jump, fine-step boundaries crossed in closed form: the same path law
 * at O(jumps) instead of O(2^level) events per path; statistical parity. */
#define EXPMC_SAMPLER_REFERENCE 0
#define EXPMC_SAMPLER_EVENT 1
/* Sampler flags (expmc_ctx_set_sampler_flags).  FULL_HOLD: the event-driven sampler evaluates
 * every sample's first holding interval in full instead of deciding "never leaves the entry"
 * from the first draw against a per-item threshold (same outcomes; A/B testing only). */
#define EXPMC_SAMPLER_FLAG_FULL_HOLD 1u
/* LOG_HOLD: the reference-order sampler runs every holding test in time space (E = -log1p(-u)
 * against rate * remaining) instead of probability space (1 - u against e^{-rate*remaining},
 * no logarithm); same draws and outcomes up to ulp ties (A/B testing only). */
#define EXPMC_SAMPLER_FLAG_LOG_HOLD 2u
/* SCREEN_EACH: the event-driven sampler's chunk kernel tests every sample's first draw for
 * "never leaves the entry" (one Philox block per sample) instead of locating the chunk's
 * jumpers by geometric gaps between them (same law; A/B testing only). */
#define EXPMC_SAMPLER_FLAG_SCREEN_EACH 4u
/* ROW_GATHER: the event-driven sampler reads the target's row record with a second gather after
 * the edge's target word instead of the per-edge record that carries the target row's payload
 * (same draws and outcomes; A/B testing only). */
#define EXPMC_SAMPLER_FLAG_ROW_GATHER 8u

/* Sampling lanes of the reference's Philox key (mlmc.cpp:94-96).  ENTRY estimates
 * (e^{tA}u)_entry; FORWARD estimates sum_i (e^{tA}u)_i from paths started at a state drawn
 * with probability u_i / sum(u) (SampleMode::forward, paths.cpp:12-36, 144-181) and runs on
 * a context built from A^T (mlmc.hpp:47-49). */
#define EXPMC_LANE_ENTRY 0u
#define EXPMC_LANE_FORWARD 1u
/* FEM (SampleMode::fem, paths.cpp:183-245): entry mode plus the Duhamel integral of a load
 * vector along the path with composite-Simpson weights; runs on a context built with
 * expmc_ctx_create_scaled (the chain of -M^{-1}K) and a load set by expmc_ctx_set_load. */
#define EXPMC_LANE_FEM 2u

typedef struct expmc_ctx expmc_ctx;

/* Square sparse matrix in canonical CSR, exactly what expmc::SparseMatrix stores
 * (sparse.hpp:21-75): row_ptr[0]=0, non-decreasing, row_ptr[n]=nnz; columns strictly
 * increasing inside a row and in [0,n); finite values. */
typedef struct {
    int64_t n;
    int64_t nnz;
    const int64_t* row_ptr;
    const int64_t* col;
    const double* val;
} expmc_csr;

typedef struct {
    int64_t n;
    int64_t n_edges;      /* off-diagonal chain edges (ChainDecomposition::jump_target.size()) */
    double d_max;         /* ChainDecomposition::d_max (exact) */
    double d_bar;         /* ChainDecomposition::d_bar (device tree sum; ~1 ulp from the reference) */
    int32_t device;
    int32_t num_sms;
    uint64_t table_bytes; /* device bytes of the packed row + edge tables */
} expmc_ctx_info;

/* One run_level request (mlmc.hpp:86-88): extend level `level` of the entry-mode problem
 * for row `entry` by sample indices [first_index, first_index + count) under `seed`. */
typedef struct {
    int64_t entry;
    uint64_t seed;
    uint64_t first_index;
    uint64_t count;
    int32_t level;
    int32_t base_level; /* nonzero: plain fine functional P_l (l == l0); zero: P_l - P_{l-1} */
} expmc_level_req;

/* LevelStats (mlmc.hpp:18-31) increment, plus the number of CTMC jumps (transitions). */
typedef struct {
    double sum;
    double sum_sq;
    uint64_t samples;
    uint64_t cost; /* model units: exponential draws + fine steps (paths.hpp:22-23) */
    uint64_t jumps;
    double integ_sum; /* fem: sum of integ_fine - integ_coarse (LevelDelta::integ_sum, mlmc.cpp:61) */
} expmc_level_stats;

/* MlmcOptions (mlmc.hpp:59-67); `seed` is used by expmc_mlmc_driver only (the row API takes
 * one seed per row); `threads` is accepted and ignored. */
typedef struct {
    double epsilon;
    uint64_t seed;
    int32_t threads;
    int32_t l0_override;
    uint64_t warmup;
    int32_t max_levels_above_l0;
    int32_t max_iterations;
    /* Extension (0 = off = the reference's behaviour): stop a component, unconverged, as soon
     * as the Lagrange allocation projects more than max_cost model units for it (hub rows of
     * C3/C4 need ~1e17 at eps = 1e-3); its projection is reported. */
    double max_cost;
} expmc_options;

/* MlmcResult (mlmc.hpp:33-43) without the per-level vector (returned separately). */
typedef struct {
    double estimate;
    double statistical_error;
    double bias_estimate;
    int32_t l0;
    int32_t L;
    uint64_t total_cost;
    int32_t converged;
    int32_t nlevels;
    uint64_t total_jumps;
    uint64_t total_samples;
    double projected_cost; /* model units the last allocation asked for (sum_l M_l C_l) */
    int32_t over_budget;   /* 1: stopped by max_cost */
    int32_t pad;
    double quadrature_bound; /* fem: bias_estimate of the load-integral means (mlmc.hpp:37) */
} expmc_result;

/* One entry of MlmcResult::levels (LevelStats, mlmc.hpp:18-24). */
typedef struct {
    int32_t level;
    int32_t pad;
    double sum;
    double sum_sq;
    uint64_t samples;
    uint64_t cost;
} expmc_level_record;

/* Counters since context creation (or the last reset). */
typedef struct {
    uint64_t kernel_launches;  /* every kernel this library launched */
    uint64_t sampler_launches; /* launches of the path-sampler kernel */
    double sampler_ms;         /* summed CUDA-event duration of the sampler launches */
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t samples;
    uint64_t jumps;
    uint64_t fine_steps;
    uint64_t rounds;           /* batched driver rounds (kernel batches) */
    uint64_t nccl_bytes;       /* chunk-partial bytes all-reduced (sample-sharded mode) */
} expmc_counters;

const char* expmc_last_error(void);
const char* expmc_version(void);
int expmc_device_count(int* out);

/* Build the sampling tables of A on `device` and bind the vector u (length n).
 * Replaces: decompose(A) (chain.cpp:75, decompose_impl chain.cpp:15-71) + the per-level
 * LevelSampler threshold table (paths.cpp:84-91) + MlmcProblem{dec, u} (mlmc.hpp:50-57).
 * Errors as decompose / SparseMatrix: non-finite entry -> EXPMC_EINVAL, column outside
 * [0,n) -> EXPMC_ERANGE, non-canonical CSR -> EXPMC_EINVAL. */
int expmc_ctx_create(const expmc_csr* A, const double* u, int device, expmc_ctx** out);
void expmc_ctx_destroy(expmc_ctx* ctx);
int expmc_ctx_get_info(const expmc_ctx* ctx, expmc_ctx_info* out);
/* decompose_scaled (chain.cpp:80-85): the tables of diag(row_scale) A -- the generator
 * -M^{-1}K of a lumped-mass FEM system (fem.cpp:62-66) without materialising it.  Errors as
 * the reference, row by row: non-finite row_scale[i] -> EXPMC_EINVAL "row scale is NaN or
 * Inf", non-finite scaled entry -> EXPMC_EINVAL; entries scaled to zero vanish. */
int expmc_ctx_create_scaled(const expmc_csr* A, const double* row_scale, const double* u, int device,
                            expmc_ctx** out);
/* Rebind u (MlmcProblem::u): length n. */
int expmc_ctx_set_vector(expmc_ctx* ctx, const double* u);
/* Bind the fem load vector (MlmcProblem::load, mlmc.hpp:53; length n).  Until it is set,
 * fem requests fail with EXPMC_EINVAL "load length does not match decomposition". */
int expmc_ctx_set_load(expmc_ctx* ctx, const double* load);
/* Export the decomposition (ChainDecomposition, chain.hpp:27-40): d, rate [n], row_ptr [n+1],
 * jump_cdf, jump_target [n_edges], sign [n_edges]; any pointer may be NULL. */
int expmc_ctx_export_tables(const expmc_ctx* ctx, double* d, double* rate, int64_t* row_ptr,
                            double* jump_cdf, int64_t* jump_target, uint8_t* sign);
/* Alias records of the event-driven sampler (built when EXPMC_SAMPLER_EVENT is selected on a
 * matrix with non-uniform rows; none otherwise): per edge slot e, prob[e] and the two target
 * words self[e] / alias[e] (column, or -(column + 1) for a negative entry).  `rows` receives the
 * number of non-uniform rows; the array pointers may be null.  Test / inspection only; no
 * reference counterpart (the reference samples from the CDF, chain.cpp:49-58, paths.cpp:57-63). */
int expmc_ctx_export_alias(const expmc_ctx* ctx, double* prob, int64_t* self, int64_t* alias, uint64_t* rows);
int expmc_ctx_get_counters(const expmc_ctx* ctx, expmc_counters* out);
/* Select the path sampler (EXPMC_SAMPLER_REFERENCE / EXPMC_SAMPLER_EVENT) for all later calls. */
int expmc_ctx_set_sampler(expmc_ctx* ctx, int32_t mode);
int expmc_ctx_get_sampler(const expmc_ctx* ctx, int32_t* mode);
int expmc_ctx_set_sampler_flags(expmc_ctx* ctx, uint32_t flags);
/* The context's CUDA stream (cudaStream_t as void*), for timing with events on the stream
 * the sampler kernels are launched on. */
int expmc_ctx_get_stream(const expmc_ctx* ctx, void** stream);
int expmc_ctx_reset_counters(expmc_ctx* ctx);

/* Sample sharding over GPUs (one process per GPU).  Every rank runs the SAME rows
 * and requests; a batch's 512-sample chunk g is sampled on rank g % world only, and the chunk
 * partials are summed across ranks with an NCCL all-reduce before the ordered combine.  Each
 * chunk is non-zero on exactly one rank, so the sums are exact: results are bit-for-bit those
 * of one GPU, on every rank (hence identical driver decisions everywhere).
 *   expmc_nccl_unique_id      on one rank; broadcast the 128 bytes to the others
 *   expmc_ctx_shard_samples   collective: ncclCommInitRank + enable sharding
 *   expmc_ctx_set_shard       the chunk filter alone, no exchange (single-GPU emulation, tests)
 *   expmc_ctx_last_partials   the last sampler window's chunk partials (for the emulation) */
#define EXPMC_NCCL_ID_BYTES 128
int expmc_nccl_unique_id(uint8_t* id);
int expmc_ctx_shard_samples(expmc_ctx* ctx, const uint8_t* id, int32_t rank, int32_t world);
int expmc_ctx_set_shard(expmc_ctx* ctx, int32_t rank, int32_t world);
int expmc_ctx_last_partials(const expmc_ctx* ctx, int64_t* count, double* sum, double* sum_sq, uint64_t* cost,
                            uint64_t* jumps);

/* run_level (mlmc.hpp:86-88; run_level_ex mlmc.cpp:76-148), entry mode, ONE request.
 * Errors as the reference: level outside [0,62] or beta <= 0 -> EXPMC_EINVAL; entry outside
 * [0,n) -> EXPMC_ERANGE; coupled (base_level == 0) at level 0 -> EXPMC_EINVAL. */
int expmc_run_level(expmc_ctx* ctx, int64_t entry, double beta, int32_t level, int32_t base_level,
                    uint64_t first_index, uint64_t additional, uint64_t seed,
                    expmc_level_stats* out);

/* run_level in forward mode (mlmc.cpp:86, 112-120): ONE request on lane 1.  The context must
 * hold A^T; its vector u is the initial distribution, with the reference's errors: a negative
 * u_i -> EXPMC_EINVAL "forward sampling requires a nonnegative vector"; sum(u) <= 0 ->
 * EXPMC_EINVAL "forward sampling requires sum(u) > 0" (make_initial_distribution,
 * paths.cpp:12-28). */
int expmc_run_level_forward(expmc_ctx* ctx, double beta, int32_t level, int32_t base_level,
                            uint64_t first_index, uint64_t additional, uint64_t seed,
                            expmc_level_stats* out);

/* Batched run_level: nreq independent requests (any mix of rows/levels/ranges) in one GPU
 * pass; out[i] is bit-for-bit what expmc_run_level would return for req[i].  lane is
 * EXPMC_LANE_ENTRY or EXPMC_LANE_FORWARD (req[i].entry ignored); others -> EXPMC_ENOTIMPL. */
int expmc_run_level_batch(expmc_ctx* ctx, double beta, uint32_t lane, int64_t nreq,
                          const expmc_level_req* req, expmc_level_stats* out);

/* Per-sample functionals (LevelSampler::single / ::coupled, paths.cpp:99-141) for golden
 * parity: sample i uses stream_for(req[i].seed, req[i].level, req[i].first_index, lane).
 * base_level != 0 -> eta_fine = value, eta_coarse = 0.  req[i].count is ignored. */
int expmc_sample_debug(expmc_ctx* ctx, double beta, uint32_t lane, int64_t nreq,
                       const expmc_level_req* req, double* eta_fine, double* eta_coarse,
                       uint64_t* cost, uint64_t* jumps, int64_t* end_state);

/* Per-sample record of any lane: value = the run_level sample x (mlmc.cpp:103-133); fem also
 * reports the load integrals (FemCoupledSample, paths.hpp). */
typedef struct {
    double eta_fine;    /* base: the value */
    double eta_coarse;
    double value;
    double integ_fine;
    double integ_coarse;
    uint64_t cost;
    uint64_t jumps;
    int64_t end_state;
} expmc_sample_record;
int expmc_sample_debug_ex(expmc_ctx* ctx, double beta, uint32_t lane, int64_t nreq,
                          const expmc_level_req* req, expmc_sample_record* out);

/* run_level in fem mode (mlmc.cpp:76-148, lane 2), ONE request; out->integ_sum carries the
 * load-integral side channel.  Errors: load not set -> EXPMC_EINVAL; coupled at level < 2 ->
 * EXPMC_EINVAL "coupled quadrature needs a step count divisible by 4" (paths.cpp:212-213). */
int expmc_run_level_fem(expmc_ctx* ctx, int64_t entry, double beta, int32_t level, int32_t base_level,
                        uint64_t first_index, uint64_t additional, uint64_t seed, expmc_level_stats* out);

/* mlmc_driver in fem mode for nrows entries (l0 >= 1, mlmc.cpp:177; result.quadrature_bound,
 * mlmc.cpp:226-241). */
int expmc_mlmc_driver_fem(expmc_ctx* ctx, double beta, const expmc_options* options, int64_t nrows,
                          const int64_t* rows, const uint64_t* row_seed, expmc_result* out,
                          expmc_level_record* levels, int32_t max_levels);

/* mlmc_driver (mlmc.hpp:94; mlmc.cpp:170-260) for ONE entry, options->seed as the seed. */
int expmc_mlmc_driver(expmc_ctx* ctx, int64_t entry, double beta, const expmc_options* options,
                      expmc_result* out, expmc_level_record* levels, int32_t max_levels);

/* mlmc_driver for nrows entries at once: row r runs the reference's Algorithm-1 decision
 * sequence with seed row_seed[r]; all rows advance in lock-step rounds, each round one
 * batched GPU pass.  levels: nrows x max_levels records (nullable). */
int expmc_mlmc_driver_rows(expmc_ctx* ctx, double beta, const expmc_options* options,
                           int64_t nrows, const int64_t* rows, const uint64_t* row_seed,
                           expmc_result* out, expmc_level_record* levels, int32_t max_levels);

/* mlmc_driver in forward mode (MlmcProblem.mode = forward): nruns independent runs of the
 * reference's driver on lane 1, run r seeded seeds[r] (seeds == NULL with nruns == 1: the
 * reference's single call, seeded options->seed), advanced in lock-step batched rounds like
 * expmc_mlmc_driver_rows.  levels: nruns x max_levels records (nullable). */
int expmc_mlmc_driver_forward(expmc_ctx* ctx, double beta, const expmc_options* options, int64_t nruns,
                              const uint64_t* seeds, expmc_result* out, expmc_level_record* levels,
                              int32_t max_levels);

/* Classical (single-level) Monte Carlo on the same sampler (mc.hpp, mc.cpp:42-113): samples
 * [0, samples) of one step size dt = beta / steps, steps = round(beta / dt) (must be a positive
 * integer, 1e-9 relative), stream_for(seed, bit_width(steps), s, lane) and the reference's
 * Welford accumulator per 512-sample chunk merged in chunk order (parallel.hpp:80-104). */
typedef struct {
    double estimate;
    double std_error;
    uint64_t samples;
    double dt;
    int64_t steps;
    uint64_t wall_cost; /* model units: exponential draws + fine steps */
    uint64_t jumps;
} expmc_mc_result;

typedef struct {
    int64_t entry;    /* ignored on the forward lane */
    uint64_t seed;
    uint64_t samples; /* >= 2 */
    double beta;
    double dt;
} expmc_mc_req;

/* mc_single_entry (mc.cpp:42-58): lane 0 on the context of A. */
int expmc_mc_single_entry(expmc_ctx* ctx, int64_t entry, double beta, double dt, uint64_t samples, uint64_t seed,
                          expmc_mc_result* out);
/* mc_forward_scalar (mc.cpp:60-76): lane 1 on the context of A^T (u: the start weights). */
int expmc_mc_forward_scalar(expmc_ctx* ctx, double beta, double dt, uint64_t samples, uint64_t seed,
                            expmc_mc_result* out);
/* nreq independent classical-MC runs in one GPU pass (lane 0 or 1). */
int expmc_mc_batch(expmc_ctx* ctx, uint32_t lane, int64_t nreq, const expmc_mc_req* req, expmc_mc_result* out);
/* mc_auto (mc.cpp:78-113): two 1000-sample pilots at dt_a = beta / 2^max(2, l0) and dt_a / 2
 * (seeds seed+1, seed+2; one batched pass), the Richardson bias constant, the step count and the
 * sample count of the final run; wall_cost includes the pilots. */
int expmc_mc_auto(expmc_ctx* ctx, int64_t entry, double beta, double epsilon, uint64_t seed, expmc_mc_result* out);

/* Roofline denominator: random 32-B-sector gather throughput of `device` over a buffer of
 * `bytes` (L2-resident or HBM-sized), `loads_per_thread` independent sector loads per thread,
 * best of `reps` launches.  Writes achieved GB/s (32 B per load / kernel time). */
/* Self-test: out[2i] = the sampler's exp (constant-memory coefficients), out[2i+1] = the
 * toolkit's exp, for n arguments x (tests: the two must agree bit for bit). */
int expmc_selftest_exp(int device, int64_t n, const double* x, double* out);
int expmc_bench_gather(int device, uint64_t bytes, int32_t loads_per_thread, int32_t reps, double* gbps);

/* Host input generators for the BASELINE configs (no GPU needed; csrc/gen.cpp).
 * Results are canonical CSR matrices owned by the library until expmc_matrix_destroy. */
typedef struct expmc_matrix expmc_matrix;

/* Host input pipeline (multi-threaded, bit-identical results and the same messages):
 *   expmc_read_matrix_market  read_matrix_market (io.cpp:69-128): coordinate real
 *                             general|symmetric; errors EXPMC_EIO "path:line: what"
 *   expmc_read_vector         read_vector (io.cpp:154-167): *n = entries; copies min(cap, n)
 *   expmc_csr_from_triplets   SparseMatrix::from_triplets (sparse.cpp:12-49): sorted,
 *                             duplicates summed, zero sums dropped; EXPMC_ERANGE / EXPMC_EINVAL */
int expmc_read_matrix_market(const char* path, expmc_matrix** out);
int expmc_read_vector(const char* path, int64_t cap, double* out, int64_t* n);
int expmc_csr_from_triplets(int64_t n, int64_t count, const int64_t* rows, const int64_t* cols,
                            const double* vals, expmc_matrix** out);
/* Barabasi-Albert, the reference's pref(n, d, seed) algorithm (netgen.cpp:61-107). */
int expmc_gen_ba(int64_t n, int64_t d, uint64_t seed, expmc_matrix** out);
/* R-MAT: 2^scale nodes, edge_factor * 2^scale directed draws, symmetrised, unit weights. */
int expmc_gen_rmat(int32_t scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                   expmc_matrix** out);
/* 3-D 7-point convection-diffusion on g^3 nodes, cell Peclet `peclet` along `axis` (0=x). */
int expmc_gen_convdiff3d(int64_t g, double peclet, int32_t axis, expmc_matrix** out);
int expmc_matrix_info(const expmc_matrix* m, int64_t* n, int64_t* nnz);
int expmc_matrix_copy(const expmc_matrix* m, int64_t* row_ptr, int64_t* col, double* val);
void expmc_matrix_destroy(expmc_matrix* m);
/* lambda_max estimate by `iters` power iterations from the all-ones vector. */
int expmc_power_iteration(const expmc_csr* A, int32_t iters, double* lambda);

/* Host-side driver helpers, identical to the reference (no GPU needed). */
int expmc_initial_level(double beta, double d_max, int32_t* out);             /* mlmc.cpp:19-23 */
int expmc_optimal_allocation(int64_t nlevels, const double* variances,        /* mlmc.cpp:25-43 */
                             const double* unit_costs, double epsilon, uint64_t* out);
int expmc_bias_estimate(int64_t n, const double* coupled_means, double* out); /* mlmc.cpp:45-51 */

#ifdef __cplusplus
}
#endif
#endif /* EXPMC_B200_H */
