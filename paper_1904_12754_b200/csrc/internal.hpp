// Internal (non-ABI) declarations shared by the CUDA translation units and the host driver.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "expmc_b200.h"

// Host canonical CSR owned by the library (generators, readers; expmc_matrix_* accessors).
struct expmc_matrix {
    int64_t n = 0;
    std::vector<int64_t> row_ptr{0};
    std::vector<int64_t> col;
    std::vector<double> val;
};

namespace expmc_b200 {

// ----------------------------------------------------------------------------- HBM layout
// Packed row record: everything a walker needs when it lands on a row, in ONE 32-B sector
// (the reference reads rate/d/row_ptr/u from four SoA arrays, chain.hpp:31-35), as two 16-B
// halves: what a JUMP needs (rate, begin, deg: one 128-bit load) and what the END of a fine step
// or of the path needs (d, u: one 128-bit load).  The level-0 walker reads exactly one half per
// event; the others read the first half and d (load_row, walker.cuh).
struct alignas(32) RowRec {
    double rate;     // sum_{j != i} |a_ij|               (chain.cpp:39-46)
    uint32_t begin;  // first edge of the row
    uint32_t deg;    // bits 0-30: number of chain edges; bit 31: kUniformRow
    double d;        // a_ii + rate_i                     (chain.cpp:47-48)
    double u;        // u_i, the terminal factor           (paths.cpp:112,138)
};
static_assert(sizeof(RowRec) == 32, "row record must be one 32-B sector");

// Edges, structure of arrays (chain.hpp:33-35):
//   tgt[e] = column j | kSignBit where a_ij < 0          (4 B, read on every jump)
//   cdf[e] = cumulative |a_ij| / rate_i, last entry of a row exactly 1   (8 B, read only for
//            rows without kUniformRow)
// kUniformRow marks rows whose stored CDF is exactly fl((j+1)/deg) for every j -- every row
// whose off-diagonal magnitudes are equal (Laplacians, adjacency matrices).  Their
// upper_bound(cdf, v) is computed exactly from v's 53-bit integer (walker.cuh), so a jump
// reads one 4-B target word instead of the row's CDF.
constexpr uint32_t kUniformRow = 0x80000000u;
constexpr uint32_t kDegMask = 0x7FFFFFFFu;
constexpr uint32_t kSignBit = 0x80000000u;
constexpr uint32_t kTargetMask = 0x7FFFFFFFu;

// Per-edge-slot alias record of a non-uniform row (Walker / Vose alias method), built on the
// device for the event-driven sampler (csrc/kernels.cu k_build_alias).  A jump in a row of
// degree deg draws slot j = floor(v deg) and keeps the slot's own target when the fraction
// v deg - j is below prob, else takes its alias: one 16-B load instead of a binary search
// over the row's CDF.  Both target words carry the sign bit like tgt[].
struct alignas(16) AliasRec {
    double prob;     // probability of keeping the slot's own target
    uint32_t self;   // tgt[begin + j]
    uint32_t alias;  // tgt[begin + alias(j)]
};
static_assert(sizeof(AliasRec) == 16, "alias record must be one 128-bit load");

// Per-edge record with the target row's payload (event-driven sampler): a jump reads ONE
// 32-B sector -- the chosen edge's target word plus everything the walker needs of the row it
// lands on -- instead of the 4-B target and then the target's row record (two dependent
// random gathers; tables beyond L2 on C3/C4).  u is not copied: it is read once per sample.
struct alignas(32) EdgeRec {
    uint32_t tgt;    // target | sign bit (tgt[])
    uint32_t begin;  // the target row's RowRec::begin
    uint32_t deg;    // the target row's RowRec::deg (with kUniformRow)
    uint32_t pad;
    double rate;     // the target row's rate
    double d;        // the target row's d
};
static_assert(sizeof(EdgeRec) == 32, "edge record must be one 32-B sector");

struct EdgeTables {
    const double* cdf;
    const uint32_t* tgt;
    const AliasRec* alias;  // per edge slot, non-uniform rows only (nullptr: none built)
    const EdgeRec* erec;    // per edge slot, event sampler (nullptr: none / separate row gathers)
};

// One device work item = one run_level request with count > 0.
struct alignas(16) DevItem {
    uint64_t seed;
    uint64_t first;
    uint64_t count;
    double dt;        // beta / 2^level (mlmc.cpp:81)
    uint64_t nsteps;  // 2^level
    uint32_t entry;
    uint32_t key3;    // (level & 0xFFFFFF) | lane << 24   (rng.hpp:29)
    uint32_t base;
    uint32_t mode;    // lane: 0 entry, 1 forward, 2 fem (the kernel instantiation is chosen per batch)
};

// Per-context data of the non-entry lanes: forward mode's initial distribution
// (InitialDistribution, paths.hpp; make_initial_distribution paths.cpp:12-28) and fem mode's
// load vector (MlmcProblem::load, mlmc.hpp:53).
struct LaneData {
    const double* cdf;
    double total;
    uint32_t n;
    const double* load;
    const uint32_t* guide;  // forward: guide[k] = upper_bound(cdf, k / 2^gbits), k = 0..2^gbits
    uint32_t gbits;
};

// Per-chunk partial and per-item running total (SumAcc, parallel.hpp:57-78, + jumps).
struct alignas(16) Partial {
    double sum;
    double sum_sq;
    unsigned long long cost;
    unsigned long long jumps;
    double extra;  // fem: sum of integ_f - integ_c (SumAcc::extra, parallel.hpp:60)
};

// Chunk partials of one sampler window, structure of arrays so that a sample-sharded run can
// sum them across GPUs with two all-reduces (fp64 sums, u64 counts).  Every chunk is sampled
// by exactly one rank and is zero elsewhere, so the cross-rank sum is exact (x + 0 = x).
struct ChunkPartials {
    double* sum;     // [W]
    double* sum_sq;  // [W]  (contiguous after sum)
    double* extra;   // [W]  (contiguous after sum_sq; written by fem batches only)
    unsigned long long* cost;   // [W]
    unsigned long long* jumps;  // [W]  (contiguous after cost)
};

// Per-sample debug output.
struct SampleOut {
    double fine;      // single: value; coupled: eta_fine (fem: sign e^{coarse+delta})
    double coarse;    // coupled: eta_coarse
    double value;     // the run_level sample x (mlmc.cpp:103-133)
    double integ_f;   // fem: fine / coarse load integrals
    double integ_c;
    unsigned long long cost;
    unsigned long long jumps;
    long long end_state;
};

constexpr uint64_t kChunk = 512;  // parallel.hpp:20 -- samples per chunk, by absolute index

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);

// ----------------------------------------------------------------------------- launchers
struct SamplerArgs {
    const RowRec* rows;
    EdgeTables edges;
    const DevItem* items;
    const uint64_t* chunk0;  // nitems + 1, exclusive prefix of chunk counts
    uint32_t nitems;
    uint64_t g_begin, g_end;  // global chunk range of this launch
    uint64_t part_base;       // chunk g's partial is partials[g - part_base] (the window's first chunk)
    ChunkPartials partials;   // one per chunk of the window
    LaneData init;
    unsigned int* counter;    // dynamic chunk counter, zeroed before launch
    uint32_t shard_rank;      // sample sharding: this launch samples the chunks g with
    uint32_t shard_world;     //   g % shard_world == shard_rank (the others stay zero)
    uint32_t flags;           // EXPMC_SAMPLER_FLAG_*
};

// level0: every item of the launch is an entry-lane base level with one fine step (RefPolicy0)
void launch_sampler(const SamplerArgs& a, int grid, int mode, uint32_t lane, cudaStream_t s, bool level0 = false);
void launch_sampler_welford(const SamplerArgs& a, int grid, int mode, uint32_t lane, cudaStream_t s);
void launch_combine_welford(const uint64_t* chunk0, const DevItem* items, uint32_t nitems, uint64_t g_begin,
                            uint64_t g_end, const ChunkPartials& partials, Partial* totals, cudaStream_t s);
void launch_combine(const uint64_t* chunk0, uint32_t nitems, uint64_t g_begin, uint64_t g_end,
                    const ChunkPartials& partials, bool with_extra, bool ordered, Partial* totals, cudaStream_t s);
void launch_debug(const RowRec* rows, EdgeTables edges, const DevItem* items, uint32_t n,
                  const LaneData& init, SampleOut* out, int mode, uint32_t lane, uint32_t flags, cudaStream_t s);
constexpr int kSamplerFem = 2;  // sampler_blocks_per_sm: the fem instantiation
int sampler_blocks_per_sm(int mode);
int sampler_threads();

void math_check(const double* x, int64_t n, double* out /* 2n: dexp, exp */, cudaStream_t s);
float bench_gather(uint64_t bytes, int loads_per_thread, int reps, int num_sms, uint64_t* total_loads);

// table builder
void launch_count_edges(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                        uint64_t* deg, unsigned int* err, uint32_t* heavy, unsigned int* nheavy, int num_sms,
                        cudaStream_t s);
void launch_fill_tables(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                        const double* u, const uint64_t* begin, RowRec* rows, double* cdf, uint32_t* tgt,
                        const uint32_t* heavy, const unsigned int* nheavy, int num_sms, cudaStream_t s);
void launch_set_vector(int64_t n, const double* u, RowRec* rows, cudaStream_t s);
void launch_export(int64_t n, const RowRec* rows, double* d, double* rate, int64_t* row_ptr,
                   cudaStream_t s);
void launch_export_edges(uint64_t e, EdgeTables edges, double* cdf, int64_t* target,
                         uint8_t* sign, cudaStream_t s);
// alias tables of the non-uniform rows: count them, then build (scratch: one u32 per edge)
void launch_count_nonuniform(int64_t n, const RowRec* rows, unsigned long long* count, cudaStream_t s);
void launch_build_alias(int64_t n, const RowRec* rows, EdgeTables edges, AliasRec* alias, uint32_t* scratch,
                        cudaStream_t s);
void launch_build_erec(uint64_t e, const RowRec* rows, const uint32_t* tgt, EdgeRec* erec, cudaStream_t s);
void launch_export_alias(uint64_t e, const AliasRec* alias, double* prob, int64_t* self, int64_t* alias_target,
                         cudaStream_t s);
// scans / reductions (CUB): exclusive sum of n u64, max / sum of RowRec::d
size_t scan_temp_bytes(int64_t n);
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, void* tmp, size_t tmp_bytes,
                        cudaStream_t s);
size_t dstat_temp_bytes(int64_t n);
void d_stats(const RowRec* rows, int64_t n, double* out2 /* device: max, sum */, void* tmp,
             size_t tmp_bytes, cudaStream_t s);

}  // namespace expmc_b200

// Host-side batched run_level used by the driver (context.cu).
struct expmc_ctx;
namespace expmc_b200 {
void run_level_batch(expmc_ctx* ctx, double beta, uint32_t lane, const expmc_level_req* req,
                     int64_t nreq, expmc_level_stats* out);
void set_error(const std::string& m);
bool ctx_has_load(const expmc_ctx* c);
// Pipelined batches (two staging slots, s = 0 or 1): launch queues the device pass and returns;
// finish waits for it and writes the totals; drain synchronises after an error.
void batch_launch(expmc_ctx* c, int s, double beta, uint32_t lane, const expmc_level_req* req, int64_t nreq,
                  expmc_level_stats* out);
void batch_finish(expmc_ctx* c, int s, const expmc_level_req* req, expmc_level_stats* out);
void batch_drain(expmc_ctx* c);
// Classical MC batch (csrc/mc.cpp front end): validated requests, Welford reduction.
void mc_batch(expmc_ctx* c, uint32_t lane, const expmc_mc_req* req, int64_t nreq, expmc_mc_result* out);
}  // namespace expmc_b200
