/* TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Never linked into the product path.
 *
 * A plain-C restatement of the reference's MLMC random-walk estimator (arXiv 1904.12754,
 * `expmc`, /root/reference/proj/core), entry mode.  Every function cites the reference
 * file:line it follows.  It is pinned against the reference itself (oracle/_ref, built by
 * oracle/Makefile from the unmodified sources) and against the golden vectors in
 * tests/golden/ (see tests/test_oracle_golden.py): uniforms, decompositions, per-sample
 * functionals, run_level sums and driver results are required to be BITWISE equal to the
 * reference (same glibc libm, same operation order, no FP contraction).
 *
 * Status codes (mirroring the reference's exception types):
 *   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 std::domain_error.
 */
#ifndef EXPMC_ORACLE_H
#define EXPMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t key[2];
    uint32_t base[4];
    uint32_t block;
    uint64_t buf[2];
    int cached;
} orc_stream;

void orc_stream_init(orc_stream* s, uint64_t seed, uint32_t level, uint64_t sample, uint32_t lane);
double orc_next_uniform(orc_stream* s);
void orc_uniforms(uint64_t seed, uint32_t level, uint64_t sample, uint32_t lane, int64_t count,
                  double* out);

typedef struct {
    int64_t n;
    int64_t nedges;
    double* d;
    double* rate;
    int64_t* row_ptr;
    double* cdf;
    int64_t* target;
    uint8_t* sign;
    double* weight;
    double d_max;
    double d_bar;
} orc_chain;

const char* orc_last_error(void);

int orc_decompose(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                  orc_chain** out);
void orc_chain_free(orc_chain* c);
void orc_chain_export(const orc_chain* c, double* d, double* rate, int64_t* row_ptr, double* cdf,
                      int64_t* target, uint8_t* sign, double* weight, double* d_max, double* d_bar);
int64_t orc_chain_n(const orc_chain* c);
int64_t orc_chain_edges(const orc_chain* c);

/* Sampling lanes (mlmc.cpp:94-96).  lane ORC_LANE_FORWARD selects forward mode
 * (LevelSampler::forward_single/coupled, paths.cpp:144-181): entry is ignored, the start
 * state is drawn from u / sum(u), and the chain must be the decomposition of A^T. */
#define ORC_LANE_ENTRY 0u
#define ORC_LANE_FORWARD 1u
#define ORC_LANE_FEM 2u

int orc_samples(const orc_chain* c, const double* u, int64_t entry, double beta, int level,
                int base, uint64_t seed, uint32_t lane, int64_t count, const uint64_t* sample_idx,
                double* fine, double* coarse, uint64_t* cost, uint64_t* jumps, int64_t* end_state);

typedef struct {
    double sum;
    double sum_sq;
    uint64_t samples;
    uint64_t cost;
    uint64_t jumps;
} orc_level_stats;

int orc_run_level(const orc_chain* c, const double* u, int64_t entry, double beta, int level,
                  int base, uint64_t first, uint64_t count, uint64_t seed, uint32_t lane,
                  int threads, orc_level_stats* out);

typedef struct {
    double epsilon;
    uint64_t seed;
    int32_t threads;
    int32_t l0_override;
    uint64_t warmup;
    int32_t max_levels_above_l0;
    int32_t max_iterations;
} orc_options;

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
} orc_result;

typedef struct {
    int32_t level;
    int32_t pad;
    double sum;
    double sum_sq;
    uint64_t samples;
    uint64_t cost;
} orc_level_record;

int orc_mlmc_driver_rows(const orc_chain* c, const double* u, double beta, const orc_options* o,
                         int64_t nrows, const int64_t* rows, const uint64_t* row_seed,
                         orc_result* out, orc_level_record* levels, int32_t max_levels);

/* mlmc_driver in forward mode: nruns independent runs, run r seeded seeds[r]. */
int orc_mlmc_driver_forward(const orc_chain* c, const double* u, double beta, const orc_options* o,
                            int64_t nruns, const uint64_t* seeds, orc_result* out,
                            orc_level_record* levels, int32_t max_levels);

/* fem mode (lane 2; LevelSampler::fem_single / fem_coupled, paths.cpp:183-245, on the chain of
 * -M^{-1}K with load = M^{-1}F).  value = the run_level sample; for coupled samples also
 * eta_f/eta_c/integ_f/integ_c and the terminal state (base: -1). */
int orc_fem_samples(const orc_chain* c, const double* u, const double* load, int64_t entry, double beta,
                    int level, int base, uint64_t seed, int64_t count, const uint64_t* sample_idx,
                    double* value, double* eta_f, double* eta_c, double* integ_f, double* integ_c,
                    int64_t* end_state, uint64_t* cost, uint64_t* jumps);
int orc_fem_run_level(const orc_chain* c, const double* u, const double* load, int64_t entry, double beta,
                      int level, int base, uint64_t first, uint64_t count, uint64_t seed, int threads,
                      orc_level_stats* out, double* integ_sum);
int orc_mlmc_driver_fem(const orc_chain* c, const double* u, const double* load, double beta,
                        const orc_options* o, int64_t nrows, const int64_t* rows, const uint64_t* row_seed,
                        orc_result* out, double* quad, orc_level_record* levels, int32_t max_levels);

/* classical MC (mc.cpp:42-76): lane 0 = mc_single_entry, lane 1 = mc_forward_scalar. */
typedef struct {
    double estimate, std_error;
    uint64_t samples;
    double dt;
    int64_t steps;
    uint64_t wall_cost, jumps;
} orc_mc_result;
int orc_mc(const orc_chain* c, const double* u, int64_t entry, double beta, double dt, uint64_t samples,
           uint64_t seed, uint32_t lane, int threads, orc_mc_result* out);

int orc_initial_level(double beta, double d_max, int* out);
int orc_optimal_allocation(int64_t n, const double* v, const double* c, double eps, uint64_t* out);
int orc_bias_estimate(int64_t n, const double* means, double* out);

int orc_dense_expmv(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                    const double* u, double beta, int threads, double* out);

int64_t orc_grid_nnz(int64_t g);
void orc_grid_laplacian(int64_t g, int64_t* row_ptr, int64_t* col, double* val);
void orc_grid_vector(uint64_t seed, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
