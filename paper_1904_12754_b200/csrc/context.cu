// C-ABI: device context (tables), batched run_level, per-sample debug path.
//
// expmc_ctx_create      <- decompose (chain.cpp:75) + LevelSampler tables (paths.cpp:84-91)
// expmc_run_level[_batch] <- run_level / run_level_ex (mlmc.hpp:86-88, mlmc.cpp:76-168)
// expmc_sample_debug    <- LevelSampler::single / ::coupled per sample (paths.cpp:99-141)
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <omp.h>

#include "internal.hpp"

using namespace expmc_b200;

// One batch's staging: pinned host arrays and their device twins (grown on demand), the request
// -> item map of the batch in flight, and its events.
struct Staging {
    DevItem* d_items = nullptr;
    uint64_t* d_chunk0 = nullptr;
    Partial* d_totals = nullptr;
    size_t cap_items = 0;
    DevItem* h_items = nullptr;  // pinned
    uint64_t* h_chunk0 = nullptr;
    Partial* h_totals = nullptr;
    size_t cap_h = 0;
    std::vector<int64_t> slot;        // request index of each item (count > 0), unless identity
    bool identity = false;            // every request has count > 0: item k is request k
    size_t n0 = 0;                    // items [0, n0) are level-0 entry items (RefPolicy0 launches)
    size_t nitems = 0;
    bool inflight = false;
    std::vector<cudaEvent_t> ev;      // sampler launch brackets (timing)
    size_t nev = 0;
    cudaEvent_t done = nullptr;       // totals are on the host
};

struct expmc_ctx {
    int device = 0;
    int num_sms = 0;
    int sampler_grid = 0;       // persistent grid of the active sampler
    int sampler_grid_ref = 0;
    int sampler_grid_ed = 0;
    int sampler_grid_fem = 0;
    int sampler = EXPMC_SAMPLER_REFERENCE;
    uint32_t sampler_flags = 0;  // EXPMC_SAMPLER_FLAG_*
    cudaStream_t stream = nullptr;
    int64_t n = 0;
    uint64_t nedges = 0;
    double d_max = 0.0, d_bar = 0.0;
    RowRec* rows = nullptr;
    double* cdf = nullptr;     // per edge, read only for non-uniform rows
    uint32_t* tgt = nullptr;   // per edge: target | sign bit
    AliasRec* alias = nullptr; // per edge, event sampler: alias records of the non-uniform rows
    bool alias_checked = false;
    uint64_t alias_rows = 0;   // non-uniform rows (0: every row picks exactly from its degree)
    EdgeRec* erec = nullptr;   // per edge, event sampler: target word + the target row's payload
    EdgeTables edges() const {
        const bool row_gather = sampler != EXPMC_SAMPLER_EVENT || (sampler_flags & EXPMC_SAMPLER_FLAG_ROW_GATHER);
        return EdgeTables{cdf, tgt, alias, row_gather ? nullptr : erec};
    }

    // batch staging, two slots so that one batch can be prepared / consumed on the host while
    // the other samples (expmc_b200::batch_launch / batch_finish; the driver's row cohorts)
    Staging stage[2];
    double* d_pf = nullptr;          // chunk partials window: sum | sum_sq | extra
    unsigned long long* d_pu = nullptr;  //                    cost | jumps
    uint64_t cap_partials = 0;
    uint64_t last_window = 0;
    // sample sharding across GPUs (one process per GPU): chunk g is sampled on rank g % world
    int shard_rank = 0;
    int shard_world = 1;
    ncclComm_t nccl = nullptr;
    unsigned* d_counter = nullptr;
    // forward mode: CDF of u and sum(u) (make_initial_distribution, paths.cpp:12-28), built on
    // the first forward request and dropped by set_vector
    double* d_init_cdf = nullptr;
    uint32_t* d_init_guide = nullptr;  // bucket guide over the CDF (exact upper_bound ranges)
    uint32_t guide_bits = 0;
    double init_total = 0.0;
    bool init_valid = false;
    double* d_load = nullptr;  // fem: MlmcProblem::load (mlmc.hpp:53), set by expmc_ctx_set_load
    SampleOut* d_dbg = nullptr;
    size_t cap_dbg = 0;

    expmc_counters ctr{};
};

namespace {

thread_local std::string g_err;

constexpr uint64_t kWindowChunks = uint64_t{1} << 22;  // chunk partials per sampler launch (128 MB)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EXPMC_OK;
    } catch (const Status& s) {
        g_err = s.what();
        return s.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return EXPMC_EINTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return EXPMC_EINTERNAL;
    }
}

void need(bool ok, int code, const char* msg) {
    if (!ok) throw Status(code, msg);
}

// Device buffers come from the device's stream-ordered memory pool (cudaMallocAsync /
// cudaFreeAsync on the context's stream) with the release threshold raised, so a context
// created after another one was destroyed reuses its blocks: no cudaMalloc / cudaFree (each a
// device-wide synchronisation, hundreds of ms for GB-sized tables) per context.
void keep_pool_memory(int device) {
    static std::mutex m;
    static std::vector<int> done;
    std::lock_guard<std::mutex> g(m);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    cudaMemPool_t pool;
    cuda_check(cudaDeviceGetDefaultMemPool(&pool, device), "cudaDeviceGetDefaultMemPool");
    uint64_t threshold = ~uint64_t{0};
    cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold), "cudaMemPoolSetAttribute");
    done.push_back(device);
}

void dev_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

template <class T>
void dev_alloc(T** p, size_t count, cudaStream_t s) {
    dev_free(*p, s);
    *p = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T), s), "cudaMallocAsync");
}

// Process-wide pool of pinned staging blocks.  Page-locking hundreds of MB (the C2 warm-up round
// stages 5M requests) costs far more than the transfer, so blocks of destroyed contexts are kept
// and handed to the next context that needs one at least as large.
struct PinnedPool {
    std::mutex m;
    std::multimap<size_t, void*> free_blocks;
};

PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // never destroyed: blocks live until process exit
    return *p;
}

void* pinned_get(size_t bytes) {
    {
        PinnedPool& pool = pinned_pool();
        std::lock_guard<std::mutex> g(pool.m);
        auto it = pool.free_blocks.lower_bound(bytes);
        if (it != pool.free_blocks.end() && it->first <= 2 * bytes + (size_t{64} << 20)) {
            void* p = it->second;
            pool.free_blocks.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    cuda_check(cudaHostAlloc(&p, bytes, cudaHostAllocPortable), "cudaHostAlloc");
    return p;
}

void pinned_put(void* p, size_t bytes) {
    if (!p) return;
    PinnedPool& pool = pinned_pool();
    std::lock_guard<std::mutex> g(pool.m);
    pool.free_blocks.emplace(bytes, p);
}

template <class T>
void host_alloc(T** p, size_t count, size_t old_count) {
    pinned_put(*p, std::max<size_t>(old_count, 1) * sizeof(T));
    *p = static_cast<T*>(pinned_get(std::max<size_t>(count, 1) * sizeof(T)));
}

void ensure_items(Staging& S, size_t nitems, cudaStream_t st) {
    if (nitems + 1 > S.cap_items) {
        const size_t cap = std::max<size_t>(nitems + 1, S.cap_items * 2);
        dev_alloc(&S.d_items, cap, st);
        dev_alloc(&S.d_chunk0, cap, st);
        dev_alloc(&S.d_totals, cap, st);
        S.cap_items = cap;
    }
    if (nitems + 1 > S.cap_h) {
        const size_t cap = std::max<size_t>(nitems + 1, S.cap_h * 2);
        host_alloc(&S.h_items, cap, S.cap_h);
        host_alloc(&S.h_chunk0, cap, S.cap_h);
        host_alloc(&S.h_totals, cap, S.cap_h);
        S.cap_h = cap;
    }
}

void bind(const expmc_ctx* c) { cuda_check(cudaSetDevice(c->device), "cudaSetDevice"); }

// Tables of the event-driven sampler, built once per context on first selecting it: alias
// records of the non-uniform rows (AliasRec, k_build_alias; uniform rows -- Laplacians,
// adjacency matrices -- pick exactly from their degree and need none) and the per-edge records
// carrying the target row's payload (EdgeRec, k_build_erec).
void ensure_event_tables(expmc_ctx* c) {
    if (c->alias_checked) return;
    bind(c);
    unsigned long long* d_count = nullptr;
    dev_alloc(&d_count, 1, c->stream);
    launch_count_nonuniform(c->n, c->rows, d_count, c->stream);
    unsigned long long count = 0;
    cuda_check(cudaMemcpyAsync(&count, d_count, sizeof count, cudaMemcpyDeviceToHost, c->stream), "D2H count");
    cuda_check(cudaStreamSynchronize(c->stream), "count non-uniform rows");
    dev_free(d_count, c->stream);
    c->alias_rows = count;
    if (count > 0 && c->nedges > 0) {
        uint32_t* scratch = nullptr;
        dev_alloc(&c->alias, c->nedges, c->stream);
        dev_alloc(&scratch, c->nedges, c->stream);
        cuda_check(cudaMemsetAsync(c->alias, 0, c->nedges * sizeof(AliasRec), c->stream), "memset alias");  // uniform rows
        launch_build_alias(c->n, c->rows, c->edges(), c->alias, scratch, c->stream);
        c->ctr.kernel_launches += 1;
        cudaError_t e = cudaStreamSynchronize(c->stream);
        dev_free(scratch, c->stream);
        cuda_check(e, "build alias tables");
    }
    c->ctr.kernel_launches += 1;
    if (c->nedges > 0) {  // EdgeRec: one sector per jump instead of the target word + its row record
        dev_alloc(&c->erec, c->nedges, c->stream);
        launch_build_erec(c->nedges, c->rows, c->tgt, c->erec, c->stream);
        c->ctr.kernel_launches += 1;
        cuda_check(cudaStreamSynchronize(c->stream), "build edge records");
    }
    c->alias_checked = true;
}

// NCCL is resolved at run time, only when sample sharding is requested: the process may already
// hold a libnccl.so.2 (PyTorch ships its own), and a link-time dependency would bind whichever
// copy the loader met first for everybody.  dlopen returns the already-loaded one if present.
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
    static Nccl api = [] {
        Nccl a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.all_reduce || !api.comm_init_rank || !api.get_unique_id)
        throw Status(EXPMC_ECUDA, "libnccl.so.2 not loadable: sample sharding unavailable");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Status(EXPMC_ECUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

// Sum the window's chunk partials across the ranks.  Each chunk was sampled by exactly one
// rank and is +0 on the others, so every element's sum is exact and rank-order independent:
// the combined totals are bit-for-bit those of a single GPU.
void nccl_allreduce_partials(ncclComm_t comm, const ChunkPartials& p, uint64_t w, uint64_t, cudaStream_t s) {
    const Nccl& n = nccl();
    nccl_check(n.group_start(), "ncclGroupStart");
    nccl_check(n.all_reduce(p.sum, p.sum, w, ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
    nccl_check(n.all_reduce(p.sum_sq, p.sum_sq, w, ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
    nccl_check(n.all_reduce(p.extra, p.extra, w, ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
    nccl_check(n.all_reduce(p.cost, p.cost, w, ncclUint64, ncclSum, comm, s), "ncclAllReduce");
    nccl_check(n.all_reduce(p.jumps, p.jumps, w, ncclUint64, ncclSum, comm, s), "ncclAllReduce");
    nccl_check(n.group_end(), "ncclGroupEnd");
}

// make_initial_distribution (paths.cpp:12-28) over the u held in the row records: the same
// sequential running sum, division by the total and last entry pinned to 1, so the device
// upper_bound sees the reference's CDF bit for bit.  Errors carry the reference's messages.
void ensure_forward_init(expmc_ctx* c) {
    if (c->init_valid) return;
    need(c->n > 0, EXPMC_EINVAL, "forward sampling requires sum(u) > 0");
    const size_t n = static_cast<size_t>(c->n);
    std::vector<double> cdf(n);
    cuda_check(cudaMemcpy2DAsync(cdf.data(), sizeof(double), reinterpret_cast<const char*>(c->rows) + offsetof(RowRec, u),
                                 sizeof(RowRec), sizeof(double), n, cudaMemcpyDeviceToHost, c->stream),
               "D2H u");
    cuda_check(cudaStreamSynchronize(c->stream), "D2H u");
    c->ctr.d2h_bytes += n * sizeof(double);
    double total = 0.0;
    for (size_t j = 0; j < n; ++j) {
        need(!(cdf[j] < 0.0), EXPMC_EINVAL, "forward sampling requires a nonnegative vector");
        total += cdf[j];
        cdf[j] = total;
    }
    need(total > 0.0, EXPMC_EINVAL, "forward sampling requires sum(u) > 0");
    for (double& x : cdf) x /= total;
    cdf.back() = 1.0;
    // Guide table: 2^b buckets (b = ceil(log2 n), 4..24), guide[k] = upper_bound(cdf, k 2^-b).
    // A draw v = K 2^-53 lies in bucket k = K >> (53 - b), i.e. k 2^-b <= v < (k+1) 2^-b exactly,
    // so upper_bound(v) lies in [guide[k], guide[k+1]]: the device searches that range only.
    uint32_t bits = 4;
    while (bits < 24 && (size_t{1} << bits) < n) ++bits;
    const size_t nb = (size_t{1} << bits) + 1;
    std::vector<uint32_t> guide(nb);
#pragma omp parallel for schedule(static)
    for (size_t k = 0; k < nb; ++k) {
        const double edge = std::ldexp(static_cast<double>(k), -static_cast<int>(bits));
        guide[k] = static_cast<uint32_t>(std::upper_bound(cdf.begin(), cdf.end(), edge) - cdf.begin());
    }
    if (!c->d_init_guide || bits != c->guide_bits) dev_alloc(&c->d_init_guide, nb, c->stream);
    c->guide_bits = bits;
    cuda_check(cudaMemcpyAsync(c->d_init_guide, guide.data(), nb * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               c->stream),
               "H2D guide");
    c->ctr.h2d_bytes += nb * sizeof(uint32_t);
    if (!c->d_init_cdf) dev_alloc(&c->d_init_cdf, n, c->stream);
    cuda_check(cudaMemcpyAsync(c->d_init_cdf, cdf.data(), n * sizeof(double), cudaMemcpyHostToDevice, c->stream),
               "H2D initial CDF");
    cuda_check(cudaStreamSynchronize(c->stream), "H2D initial CDF");
    c->ctr.h2d_bytes += n * sizeof(double);
    c->init_total = total;
    c->init_valid = true;
}

LaneData lane_data(const expmc_ctx* c) {
    LaneData ld = c->init_valid ? LaneData{c->d_init_cdf, c->init_total, static_cast<uint32_t>(c->n), nullptr,
                                           c->d_init_guide, c->guide_bits}
                                : LaneData{nullptr, 0.0, 0u, nullptr, nullptr, 0u};
    ld.load = c->d_load;
    return ld;
}

// Samples parallel_samples actually draws for [first, first + count) (parallel.hpp:39-50): all
// of them, except that a chunk whose end (chunk + 1) * 512 wraps to 0 at 2^64 contributes none.
uint64_t sampled_count(uint64_t first, uint64_t count) {
    if (count == 0) return 0;
    const uint64_t last_chunk = (first + count - 1) / kChunk;
    if ((last_chunk + 1) * kChunk != 0) return count;
    const uint64_t lo = first > last_chunk * kChunk ? first : last_chunk * kChunk;
    return count - ((first + count) - lo);
}

DevItem make_item(const expmc_level_req& r, double beta, uint32_t lane) {
    DevItem it{};
    const uint64_t steps = uint64_t{1} << r.level;
    it.seed = r.seed;
    it.first = r.first_index;
    it.count = r.count;
    it.dt = beta / static_cast<double>(steps);  // mlmc.cpp:81
    it.nsteps = steps;
    it.entry = lane == EXPMC_LANE_FORWARD ? 0u : static_cast<uint32_t>(r.entry);  // fem: entry mode's entry
    it.key3 = (static_cast<uint32_t>(r.level) & 0xFFFFFFu) | (lane << 24);  // rng.hpp:29
    it.base = r.base_level ? 1u : 0u;
    it.mode = lane;
    return it;
}

// validate_problem (mlmc.cpp:150-159) + run_level_ex's level check (mlmc.cpp:79) + the
// coupled even-step check (paths.cpp:119).
// Forward requests carry no entry (the start state is drawn from u).  fem requests need the
// load (validate_problem, mlmc.cpp:156-157) and, when coupled, a step count divisible by 4
// (fem_coupled, paths.cpp:212-213; raised per sample, so only for count > 0).
void validate_req(const expmc_ctx* c, const expmc_level_req& r, double beta, uint32_t lane) {
    if (lane != EXPMC_LANE_FORWARD) need(r.entry >= 0 && r.entry < c->n, EXPMC_ERANGE, "entry index outside matrix");
    if (lane == EXPMC_LANE_FEM)
        need(c->d_load != nullptr, EXPMC_EINVAL, "load length does not match decomposition");
    need(beta > 0.0, EXPMC_EINVAL, "beta must be positive");
    need(r.level >= 0 && r.level <= 62, EXPMC_EINVAL, "level outside [0, 62]");
    need(beta / static_cast<double>(uint64_t{1} << r.level) > 0.0, EXPMC_EINVAL, "step size must be positive");
    if (lane == EXPMC_LANE_FEM && !r.base_level && r.level < 2 && r.count > 0)
        throw Status(EXPMC_EINVAL, "coupled quadrature needs a step count divisible by 4");
    if (!r.base_level && r.level == 0 && r.count > 0)
        throw Status(EXPMC_EINVAL, "coupled sampling needs an even step count");
}

}  // namespace

namespace expmc_b200 {

void set_error(const std::string& m) { g_err = m; }

bool ctx_has_load(const expmc_ctx* c) { return c->d_load != nullptr; }

// The device pass over prepared items (S.h_items, S.h_chunk0 = per-item chunk counts):
// upload, sampler windows of up to kWindowChunks chunks (+ the NCCL exchange when sample-
// sharded), ordered combine, totals back to S.h_totals -- all queued on the context's stream;
// sample_wait collects them.  welford: the classical-MC reduction.
void sample_launch(expmc_ctx* c, Staging& S, size_t nitems, uint32_t lane, bool welford) {
    // exclusive prefix of the chunk counts: per-thread block sums, then the blocks' offsets
    uint64_t total = 0;
    if (nitems < (size_t{1} << 16)) {
        for (size_t k = 0; k < nitems; ++k) {
            const uint64_t n = S.h_chunk0[k];
            S.h_chunk0[k] = total;
            total += n;
        }
    } else {
        std::vector<uint64_t> part(static_cast<size_t>(omp_get_max_threads()) + 1, 0);
        size_t used = 1;
#pragma omp parallel
        {
            const size_t nt = static_cast<size_t>(omp_get_num_threads()), t = static_cast<size_t>(omp_get_thread_num());
            const size_t b = nitems * t / nt, e = nitems * (t + 1) / nt;
            uint64_t acc = 0;
            for (size_t k = b; k < e; ++k) acc += S.h_chunk0[k];
            part[t + 1] = acc;
#pragma omp barrier
#pragma omp single
            {
                for (size_t q = 1; q <= nt; ++q) part[q] += part[q - 1];
                used = nt;
            }  // implicit barrier
            acc = part[t];
            for (size_t k = b; k < e; ++k) {
                const uint64_t n = S.h_chunk0[k];
                S.h_chunk0[k] = acc;
                acc += n;
            }
        }
        total = part[used];
    }
    S.h_chunk0[nitems] = total;
    cuda_check(cudaMemcpyAsync(S.d_items, S.h_items, nitems * sizeof(DevItem), cudaMemcpyHostToDevice, c->stream),
               "H2D items");
    cuda_check(cudaMemcpyAsync(S.d_chunk0, S.h_chunk0, (nitems + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                               c->stream),
               "H2D chunk0");
    c->ctr.h2d_bytes += nitems * sizeof(DevItem) + (nitems + 1) * sizeof(uint64_t);
    cuda_check(cudaMemsetAsync(S.d_totals, 0, nitems * sizeof(Partial), c->stream), "memset totals");
    if (!c->d_pf) {
        // EXPMC_WINDOW_CHUNKS (tests): a small window exercises the multi-launch path
        const char* wenv = std::getenv("EXPMC_WINDOW_CHUNKS");
        const uint64_t wreq = wenv ? std::strtoull(wenv, nullptr, 10) : 0;
        c->cap_partials = wreq > 0 && wreq <= (kWindowChunks << 4) ? wreq : kWindowChunks;
        dev_alloc(&c->d_pf, 3 * c->cap_partials, c->stream);
        dev_alloc(&c->d_pu, 2 * c->cap_partials, c->stream);
        dev_alloc(&c->d_counter, 1, c->stream);
    }
    const ChunkPartials cp{c->d_pf, c->d_pf + c->cap_partials, c->d_pf + 2 * c->cap_partials, c->d_pu,
                           c->d_pu + c->cap_partials};
    const bool fem = lane == EXPMC_LANE_FEM && !welford;
    const int sampler_grid = fem ? c->sampler_grid_fem : c->sampler_grid;
    const uint32_t world = static_cast<uint32_t>(c->shard_world);
    const int warps_per_block = sampler_threads() / 32;
    size_t nev = 0;
    // chunks [0, g_split) belong to the leading level-0 items (RefPolicy0), the rest to RefPolicy
    const uint64_t g_split = welford ? 0 : S.h_chunk0[std::min(S.n0, nitems)];
    for (uint64_t g0 = 0; g0 < total; g0 += c->cap_partials) {
        const uint64_t g1 = std::min(total, g0 + c->cap_partials);
        const uint64_t w = g1 - g0;
        if (world > 1) {  // chunks sampled by the other ranks stay exactly zero here
            cuda_check(cudaMemsetAsync(cp.sum, 0, w * sizeof(double), c->stream), "memset partials");
            cuda_check(cudaMemsetAsync(cp.sum_sq, 0, w * sizeof(double), c->stream), "memset partials");
            cuda_check(cudaMemsetAsync(cp.extra, 0, w * sizeof(double), c->stream), "memset partials");
            cuda_check(cudaMemsetAsync(cp.cost, 0, w * sizeof(uint64_t), c->stream), "memset partials");
            cuda_check(cudaMemsetAsync(cp.jumps, 0, w * sizeof(uint64_t), c->stream), "memset partials");
        }
        // one launch per policy part of the window: [g0, g_split) level-0, [g_split, g1) the rest
        const uint64_t cut[3] = {g0, std::min(std::max(g_split, g0), g1), g1};
        for (int part = 0; part < 2; ++part) {
            const uint64_t b0 = cut[part], b1 = cut[part + 1];
            if (b0 >= b1) continue;
            cuda_check(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned), c->stream), "memset counter");
            SamplerArgs a;
            a.rows = c->rows;
            a.edges = c->edges();
            a.items = S.d_items;
            a.chunk0 = S.d_chunk0;
            a.nitems = static_cast<uint32_t>(nitems);
            a.g_begin = b0;
            a.g_end = b1;
            a.part_base = g0;
            a.partials = cp;
            a.counter = c->d_counter;
            a.shard_rank = static_cast<uint32_t>(c->shard_rank);
            a.shard_world = world;
            a.flags = c->sampler_flags;
            a.init = lane_data(c);
            const uint64_t own = (b1 - b0 + world - 1) / world;
            const uint64_t want_blocks = (own + warps_per_block - 1) / warps_per_block;
            const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(sampler_grid, want_blocks)));
            while (S.ev.size() < 2 * (nev + 1)) {
                cudaEvent_t e;
                cuda_check(cudaEventCreate(&e), "cudaEventCreate");
                S.ev.push_back(e);
            }
            cuda_check(cudaEventRecord(S.ev[2 * nev], c->stream), "event");
            if (welford) launch_sampler_welford(a, grid, c->sampler, lane, c->stream);
            else launch_sampler(a, grid, c->sampler, lane, c->stream, part == 0 && S.n0 > 0);
            cuda_check(cudaEventRecord(S.ev[2 * nev + 1], c->stream), "event");
            ++nev;
            c->ctr.kernel_launches += 1;
            c->ctr.sampler_launches += 1;
        }
        if (c->nccl) {  // exact cross-GPU sum of the window's chunk partials (one rank non-zero per chunk)
            nccl_allreduce_partials(c->nccl, cp, w, c->cap_partials, c->stream);
            c->ctr.nccl_bytes += w * (3 * sizeof(double) + 2 * sizeof(uint64_t));
        }
        if (welford)
            launch_combine_welford(S.d_chunk0, S.d_items, static_cast<uint32_t>(nitems), g0, g1, cp, S.d_totals,
                                   c->stream);
        else
            launch_combine(S.d_chunk0, static_cast<uint32_t>(nitems), g0, g1, cp, fem,
                           fem || c->sampler != EXPMC_SAMPLER_EVENT, S.d_totals, c->stream);
        c->ctr.kernel_launches += 1;  // the combine
        c->last_window = w;
    }
    cuda_check(cudaMemcpyAsync(S.h_totals, S.d_totals, nitems * sizeof(Partial), cudaMemcpyDeviceToHost, c->stream),
               "D2H totals");
    c->ctr.d2h_bytes += nitems * sizeof(Partial);
    if (!S.done) cuda_check(cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventRecord(S.done, c->stream), "event");
    S.nev = nev;
    S.nitems = nitems;
    S.inflight = true;
}

// Wait for a launched batch's totals and account its sampler time.
void sample_wait(expmc_ctx* c, Staging& S) {
    if (!S.inflight) return;
    S.inflight = false;
    cuda_check(cudaEventSynchronize(S.done), "sampler");
    for (size_t k = 0; k < S.nev; ++k) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, S.ev[2 * k], S.ev[2 * k + 1]), "event time");
        c->ctr.sampler_ms += ms;
    }
}

// checked_steps (mc.cpp:16-23) and level_key = bit_width(steps) (mc.cpp:25-27).
int64_t mc_steps(double beta, double dt) {
    need(dt > 0.0 && beta > 0.0, EXPMC_EINVAL, "beta and dt must be positive");
    const double ratio = beta / dt;
    const double rounded = std::round(ratio);
    need(!(std::abs(ratio - rounded) > 1e-9 * ratio || rounded < 1.0), EXPMC_EINVAL,
         "beta/dt must be a positive integer step count");
    return static_cast<int64_t>(rounded);
}

void mc_batch(expmc_ctx* c, uint32_t lane, const expmc_mc_req* req, int64_t nreq, expmc_mc_result* out) {
    need(lane == EXPMC_LANE_ENTRY || lane == EXPMC_LANE_FORWARD, EXPMC_ENOTIMPL,
         "classical MC runs on the entry (0) or forward (1) lane");
    bind(c);
    std::vector<int64_t> steps(static_cast<size_t>(nreq));
    for (int64_t i = 0; i < nreq; ++i) {  // mc_single_entry / mc_forward_scalar checks, in order
        need(req[i].samples >= 2, EXPMC_EINVAL, "at least 2 samples required");
        if (lane == EXPMC_LANE_ENTRY)
            need(req[i].entry >= 0 && req[i].entry < c->n, EXPMC_ERANGE, "entry index outside matrix");
        steps[static_cast<size_t>(i)] = mc_steps(req[i].beta, req[i].dt);
    }
    if (nreq == 0) return;
    if (lane == EXPMC_LANE_FORWARD) ensure_forward_init(c);
    need(static_cast<uint64_t>(nreq) < (uint64_t{1} << 31), EXPMC_EINVAL, "too many MC requests in one batch");
    const size_t nitems = static_cast<size_t>(nreq);
    Staging& S = c->stage[0];
    sample_wait(c, S);
    ensure_items(S, nitems, c->stream);
    for (size_t k = 0; k < nitems; ++k) {
        const expmc_mc_req& r = req[k];
        DevItem it{};
        const uint64_t st = static_cast<uint64_t>(steps[k]);
        it.seed = r.seed;
        it.first = 0;
        it.count = r.samples;
        it.dt = r.dt;  // LevelSampler(dec, dt, steps): the given dt, not beta / steps
        it.nsteps = st;
        it.entry = lane == EXPMC_LANE_FORWARD ? 0u : static_cast<uint32_t>(r.entry);
        const uint32_t key = static_cast<uint32_t>(64 - __builtin_clzll(st));  // std::bit_width
        it.key3 = (key & 0xFFFFFFu) | (lane << 24);
        it.base = 1u;
        it.mode = lane;
        S.h_items[k] = it;
        S.h_chunk0[k] = (r.samples - 1) / kChunk + 1;
    }
    c->ctr.rounds += 1;
    sample_launch(c, S, nitems, lane, true);
    sample_wait(c, S);
    for (size_t k = 0; k < nitems; ++k) {  // finish (mc.cpp:29-38)
        const Partial& t = S.h_totals[k];
        const uint64_t n = static_cast<uint64_t>(t.extra);
        expmc_mc_result& o = out[k];
        o.samples = n;
        o.estimate = t.sum;
        const double var = n > 1 ? std::max(0.0, t.sum_sq / static_cast<double>(n - 1)) : 0.0;
        o.std_error = n > 1 ? std::sqrt(var / static_cast<double>(n)) : 0.0;
        o.dt = req[k].dt;
        o.steps = steps[k];
        o.wall_cost = t.cost;
        o.jumps = t.jumps;
        c->ctr.samples += n;
        c->ctr.jumps += t.jumps;
        c->ctr.fine_steps += n * static_cast<uint64_t>(steps[k]);
    }
}

// Validate a batch, stage its items in slot `s` and queue the device pass; out[] gets zeros for
// every request now and its totals from batch_finish.  The slot's previous batch, if any, must
// have been finished.
void batch_launch(expmc_ctx* c, int s, double beta, uint32_t lane, const expmc_level_req* req, int64_t nreq,
                  expmc_level_stats* out) {
    bind(c);
    Staging& S = c->stage[s];
    need(!S.inflight, EXPMC_EINTERNAL, "staging slot busy");
    S.nitems = 0;
    // validate (first failing request wins, as a sequential loop would report it)
    int64_t bad = nreq, empty = 0;
#pragma omp parallel for schedule(static) reduction(min : bad) reduction(+ : empty)
    for (int64_t i = 0; i < nreq; ++i) {
        out[i] = expmc_level_stats{0.0, 0.0, 0, 0, 0, 0.0};
        empty += req[i].count == 0;
        try {
            validate_req(c, req[i], beta, lane);
        } catch (const Status&) {
            bad = std::min(bad, i);
        }
    }
    if (bad < nreq) validate_req(c, req[bad], beta, lane);  // rethrows with the right code
    S.slot.clear();
    S.identity = empty == 0;  // the driver's batches: no empty requests, no index list to build
    S.n0 = 0;
    // Reference-order entry batches: the level-0 items (base level, one fine step) go first and
    // are sampled by the step-free walker (RefPolicy0, ~11 % faster per trip); the item order
    // changes no result (items are independent, each one's chunks keep their order).
    size_t nlev0 = 0;
    if (c->sampler == EXPMC_SAMPLER_REFERENCE && lane == EXPMC_LANE_ENTRY) {
#pragma omp parallel for schedule(static) reduction(+ : nlev0)
        for (int64_t i = 0; i < nreq; ++i) nlev0 += req[i].count > 0 && req[i].level == 0 && req[i].base_level != 0;
    }
    const size_t nnonempty = static_cast<size_t>(nreq - empty);
    if (nlev0 > 0 && nlev0 < nnonempty) {
        S.identity = false;
        S.slot.resize(nnonempty);
        size_t a0 = 0, a1 = nlev0;
        for (int64_t i = 0; i < nreq; ++i) {
            if (req[i].count == 0) continue;
            if (req[i].level == 0 && req[i].base_level != 0) S.slot[a0++] = i;
            else S.slot[a1++] = i;
        }
    } else if (!S.identity) {
        S.slot.reserve(static_cast<size_t>(nreq));
        for (int64_t i = 0; i < nreq; ++i)
            if (req[i].count > 0) S.slot.push_back(i);
    }
    S.n0 = nlev0;
    const size_t nitems = S.identity ? static_cast<size_t>(nreq) : S.slot.size();
    if (nitems == 0) return;
    const bool forward = lane == EXPMC_LANE_FORWARD;
    if (forward) ensure_forward_init(c);  // run_level builds it before sampling (mlmc.cpp)
    c->ctr.rounds += 1;
    need(nitems < (size_t{1} << 31), EXPMC_EINVAL, "too many run_level requests in one batch");
    ensure_items(S, nitems, c->stream);
#pragma omp parallel for schedule(static)
    for (size_t k = 0; k < nitems; ++k) {
        const expmc_level_req& r = req[S.identity ? static_cast<int64_t>(k) : S.slot[k]];
        S.h_items[k] = make_item(r, beta, lane);
        const uint64_t first_chunk = r.first_index / kChunk;
        const uint64_t last_chunk = (r.first_index + r.count - 1) / kChunk;  // parallel.hpp:36-38
        S.h_chunk0[k] = last_chunk - first_chunk + 1;
    }
    sample_launch(c, S, nitems, lane, false);
}

// Wait for slot `s`'s batch and write its per-request totals (the same req / out as the launch).
void batch_finish(expmc_ctx* c, int s, const expmc_level_req* req, expmc_level_stats* out) {
    Staging& S = c->stage[s];
    if (!S.inflight) return;  // nothing was queued (all counts 0)
    bind(c);
    sample_wait(c, S);
    const size_t nitems = S.nitems;
    uint64_t samples = 0, jumps = 0, steps = 0;
#pragma omp parallel for schedule(static) reduction(+ : samples, jumps, steps)
    for (size_t k = 0; k < nitems; ++k) {
        const int64_t i = S.identity ? static_cast<int64_t>(k) : S.slot[k];
        const expmc_level_req& r = req[i];
        expmc_level_stats& o = out[i];
        o.sum = S.h_totals[k].sum;
        o.sum_sq = S.h_totals[k].sum_sq;
        o.samples = sampled_count(r.first_index, r.count);
        o.cost = S.h_totals[k].cost;
        o.jumps = S.h_totals[k].jumps;
        o.integ_sum = S.h_totals[k].extra;
        samples += o.samples;
        jumps += o.jumps;
        steps += o.samples << r.level;
    }
    c->ctr.samples += samples;
    c->ctr.jumps += jumps;
    c->ctr.fine_steps += steps;
}

// Drain every staging slot (error paths of pipelined callers).
void batch_drain(expmc_ctx* c) {
    bind(c);
    cudaStreamSynchronize(c->stream);
    for (Staging& S : c->stage) S.inflight = false;
}

void run_level_batch(expmc_ctx* c, double beta, uint32_t lane, const expmc_level_req* req, int64_t nreq,
                     expmc_level_stats* out) {
    sample_wait(c, c->stage[0]);  // a previous pipelined caller may have left slot 0 queued
    batch_launch(c, 0, beta, lane, req, nreq, out);
    batch_finish(c, 0, req, out);
}

// Per-sample records of any lane (one debug launch): the shared body of expmc_sample_debug[_ex].
std::vector<SampleOut> sample_debug(expmc_ctx* c, double beta, uint32_t lane, int64_t nreq,
                                    const expmc_level_req* req) {
    need(lane <= EXPMC_LANE_FEM, EXPMC_ENOTIMPL, "unknown sampling lane (0 entry, 1 forward, 2 fem)");
    std::vector<SampleOut> o(static_cast<size_t>(nreq > 0 ? nreq : 0));
    if (nreq == 0) return o;
    bind(c);
    std::vector<DevItem> items(static_cast<size_t>(nreq));
    for (int64_t i = 0; i < nreq; ++i) {
        expmc_level_req r = req[i];
        r.count = 1;
        validate_req(c, r, beta, lane);
        items[i] = make_item(r, beta, lane);
    }
    if (lane == EXPMC_LANE_FORWARD) ensure_forward_init(c);
    Staging& S = c->stage[0];
    sample_wait(c, S);
    ensure_items(S, static_cast<size_t>(nreq), c->stream);
    if (static_cast<size_t>(nreq) > c->cap_dbg) {
        dev_alloc(&c->d_dbg, nreq, c->stream);
        c->cap_dbg = nreq;
    }
    cuda_check(cudaMemcpyAsync(S.d_items, items.data(), nreq * sizeof(DevItem), cudaMemcpyHostToDevice, c->stream),
               "H2D");
    launch_debug(c->rows, c->edges(), S.d_items, static_cast<uint32_t>(nreq), lane_data(c), c->d_dbg, c->sampler,
                 lane, c->sampler_flags, c->stream);
    c->ctr.kernel_launches += 1;
    cuda_check(cudaMemcpyAsync(o.data(), c->d_dbg, nreq * sizeof(SampleOut), cudaMemcpyDeviceToHost, c->stream),
               "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sample debug");
    return o;
}

}  // namespace expmc_b200

extern "C" {

const char* expmc_last_error(void) { return g_err.c_str(); }

const char* expmc_version(void) { return "expmc_b200 0.1.0 (sm_100a, reference-order sampler)"; }

int expmc_device_count(int* out) {
    return guarded([&] {
        const cudaError_t e = cudaGetDeviceCount(out);
        if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {  // CPU-only host: zero devices
            cudaGetLastError();
            *out = 0;
            return;
        }
        cuda_check(e, "cudaGetDeviceCount");
    });
}

int expmc_ctx_create(const expmc_csr* A, const double* u, int device, expmc_ctx** out) {
    return guarded([&] {
        need(A != nullptr && out != nullptr, EXPMC_EINVAL, "null argument");
        const int64_t n = A->n;
        need(n >= 0, EXPMC_EINVAL, "matrix dimension must be nonnegative");
        need(n < (int64_t{1} << 31), EXPMC_EINVAL, "matrix dimension must be < 2^31");
        need(n == 0 || (A->row_ptr && u), EXPMC_EINVAL, "null CSR or vector");
        if (n > 0) {
            need(A->row_ptr[0] == 0 && A->row_ptr[n] == A->nnz && A->nnz >= 0, EXPMC_EINVAL,
                 "CSR row_ptr must start at 0 and end at nnz");
            need(A->nnz == 0 || (A->col && A->val), EXPMC_EINVAL, "null CSR arrays");
        }
        auto* c = new expmc_ctx;
        try {
            c->device = device;
            bind(c);
            keep_pool_memory(device);
            cuda_check(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
            cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
            c->sampler_grid_ref = c->num_sms * sampler_blocks_per_sm(EXPMC_SAMPLER_REFERENCE);
            c->sampler_grid_ed = c->num_sms * sampler_blocks_per_sm(EXPMC_SAMPLER_EVENT);
            c->sampler_grid_fem = c->num_sms * sampler_blocks_per_sm(kSamplerFem);
            c->sampler_grid = c->sampler_grid_ref;
            c->n = n;
            if (n > 0) {
                const int64_t nnz = A->nnz;
                int64_t *d_rp = nullptr, *d_col = nullptr;
                double *d_val = nullptr, *d_u = nullptr, *d_st = nullptr;
                uint64_t *d_deg = nullptr, *d_begin = nullptr;
                unsigned* d_err = nullptr;  // [0] error bits, [1] heavy-row count
                uint32_t* d_heavy = nullptr;
                void* tmp = nullptr;
                auto cleanup = [&] {
                    for (void* p : {static_cast<void*>(d_rp), static_cast<void*>(d_col), static_cast<void*>(d_val),
                                    static_cast<void*>(d_u), static_cast<void*>(d_deg), static_cast<void*>(d_begin),
                                    static_cast<void*>(d_err), tmp, static_cast<void*>(d_st), static_cast<void*>(d_heavy)})
                        dev_free(p, c->stream);
                };
                try {
                    dev_alloc(&d_rp, n + 1, c->stream);
                    dev_alloc(&d_col, nnz, c->stream);
                    dev_alloc(&d_val, nnz, c->stream);
                    dev_alloc(&d_u, n, c->stream);
                    dev_alloc(&d_deg, n, c->stream);
                    dev_alloc(&d_begin, n, c->stream);
                    dev_alloc(&d_err, 2, c->stream);
                    dev_alloc(&d_heavy, static_cast<size_t>(std::min<int64_t>(n, nnz / 128 + 1)), c->stream);
                    dev_alloc(&d_st, 2, c->stream);
                    cuda_check(cudaMemcpyAsync(d_rp, A->row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream), "H2D");
                    if (nnz) {
                        cuda_check(cudaMemcpyAsync(d_col, A->col, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream), "H2D");
                        cuda_check(cudaMemcpyAsync(d_val, A->val, nnz * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
                    }
                    cuda_check(cudaMemcpyAsync(d_u, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
                    c->ctr.h2d_bytes += (n + 1) * 8 + nnz * 16 + n * 8;
                    cuda_check(cudaMemsetAsync(d_err, 0, 2 * sizeof(unsigned), c->stream), "memset");
                    launch_count_edges(n, d_rp, d_col, d_val, d_deg, d_err, d_heavy, d_err + 1, c->num_sms, c->stream);
                    unsigned err = 0;
                    cuda_check(cudaMemcpyAsync(&err, d_err, sizeof err, cudaMemcpyDeviceToHost, c->stream), "D2H");
                    cuda_check(cudaStreamSynchronize(c->stream), "count edges");
                    need(!(err & 2u), EXPMC_ERANGE, "triplet index outside [0, n)");
                    need(!(err & 1u), EXPMC_EINVAL, "matrix entry is NaN or Inf");
                    need(!(err & 4u), EXPMC_EINVAL, "CSR is not canonical (sorted, duplicate-free columns)");
                    const size_t tb = std::max(scan_temp_bytes(n), dstat_temp_bytes(n));
                    cuda_check(cudaMallocAsync(&tmp, tb, c->stream), "cudaMallocAsync");
                    exclusive_scan_u64(d_deg, d_begin, n, tmp, tb, c->stream);
                    uint64_t last[2];
                    cuda_check(cudaMemcpyAsync(&last[0], d_begin + (n - 1), 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
                    cuda_check(cudaMemcpyAsync(&last[1], d_deg + (n - 1), 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
                    cuda_check(cudaStreamSynchronize(c->stream), "scan");
                    c->nedges = last[0] + last[1];
                    need(c->nedges < (uint64_t{1} << 32), EXPMC_EINVAL, "more than 2^32 chain edges");
                    dev_alloc(&c->rows, n, c->stream);
                    dev_alloc(&c->cdf, c->nedges, c->stream);
                    dev_alloc(&c->tgt, c->nedges, c->stream);
                    launch_fill_tables(n, d_rp, d_col, d_val, d_u, d_begin, c->rows, c->cdf, c->tgt, d_heavy, d_err + 1,
                                       c->num_sms, c->stream);
                    d_stats(c->rows, n, d_st, tmp, tb, c->stream);
                    double st[2];
                    cuda_check(cudaMemcpyAsync(st, d_st, sizeof st, cudaMemcpyDeviceToHost, c->stream), "D2H");
                    c->ctr.d2h_bytes += 32;
                    c->ctr.kernel_launches += 7;
                    cuda_check(cudaStreamSynchronize(c->stream), "build tables");
                    c->d_max = st[0];                            // chain.cpp:70
                    c->d_bar = st[1] / static_cast<double>(n);   // chain.cpp:71 (tree-summed)
                } catch (...) {
                    cleanup();
                    throw;
                }
                cleanup();
            }
        } catch (...) {
            expmc_ctx_destroy(c);
            throw;
        }
        *out = c;
    });
}

void expmc_ctx_destroy(expmc_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStream_t st = c->stream;
    for (Staging& S : c->stage) {
        dev_free(S.d_items, st);
        dev_free(S.d_chunk0, st);
        dev_free(S.d_totals, st);
        if (S.cap_h) {  // staging blocks go back to the process-wide pool
            pinned_put(S.h_items, S.cap_h * sizeof(DevItem));
            pinned_put(S.h_chunk0, S.cap_h * sizeof(uint64_t));
            pinned_put(S.h_totals, S.cap_h * sizeof(Partial));
        }
    }
    for (void* p : {static_cast<void*>(c->rows), static_cast<void*>(c->cdf), static_cast<void*>(c->tgt),
                    static_cast<void*>(c->alias), static_cast<void*>(c->erec), static_cast<void*>(c->d_pf), static_cast<void*>(c->d_pu), static_cast<void*>(c->d_counter),
                    static_cast<void*>(c->d_init_cdf), static_cast<void*>(c->d_init_guide),
                    static_cast<void*>(c->d_load), static_cast<void*>(c->d_dbg)})
        dev_free(p, st);  // back to the device pool, in stream order
    if (st) cudaStreamSynchronize(st);
    for (Staging& S : c->stage) {
        for (cudaEvent_t e : S.ev) cudaEventDestroy(e);
        if (S.done) cudaEventDestroy(S.done);
    }
    if (c->nccl) nccl().comm_destroy(c->nccl);
    if (st) cudaStreamDestroy(st);
    delete c;
}

int expmc_ctx_get_info(const expmc_ctx* c, expmc_ctx_info* out) {
    return guarded([&] {
        need(c && out, EXPMC_EINVAL, "null argument");
        out->n = c->n;
        out->n_edges = static_cast<int64_t>(c->nedges);
        out->d_max = c->d_max;
        out->d_bar = c->d_bar;
        out->device = c->device;
        out->num_sms = c->num_sms;
        out->table_bytes = static_cast<uint64_t>(c->n) * sizeof(RowRec) + c->nedges * (sizeof(double) + sizeof(uint32_t)) +
                           (c->alias ? c->nedges * sizeof(AliasRec) : 0) + (c->erec ? c->nedges * sizeof(EdgeRec) : 0);
    });
}

int expmc_ctx_set_vector(expmc_ctx* c, const double* u) {
    return guarded([&] {
        need(c && (u || c->n == 0), EXPMC_EINVAL, "null argument");
        if (c->n == 0) return;
        bind(c);
        double* d_u = nullptr;
        dev_alloc(&d_u, c->n, c->stream);
        cuda_check(cudaMemcpyAsync(d_u, u, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
        launch_set_vector(c->n, d_u, c->rows, c->stream);
        c->ctr.h2d_bytes += c->n * 8;
        c->ctr.kernel_launches += 1;
        cudaError_t e = cudaStreamSynchronize(c->stream);
        dev_free(d_u, c->stream);
        c->init_valid = false;  // the forward CDF follows u
        cuda_check(e, "set vector");
    });
}

int expmc_ctx_export_tables(const expmc_ctx* c, double* d, double* rate, int64_t* row_ptr, double* cdf,
                            int64_t* target, uint8_t* sign) {
    return guarded([&] {
        need(c != nullptr, EXPMC_EINVAL, "null context");
        bind(c);
        const int64_t n = c->n;
        const uint64_t m = c->nedges;
        double *dd = nullptr, *dr = nullptr, *dc = nullptr;
        int64_t *drp = nullptr, *dt = nullptr;
        uint8_t* ds = nullptr;
        dev_alloc(&dd, n, c->stream); dev_alloc(&dr, n, c->stream); dev_alloc(&drp, n + 1, c->stream);
        dev_alloc(&dc, m, c->stream); dev_alloc(&dt, m, c->stream); dev_alloc(&ds, m, c->stream);
        launch_export(n, c->rows, dd, dr, drp, c->stream);
        launch_export_edges(m, c->edges(), dc, dt, ds, c->stream);
        cudaError_t e = cudaStreamSynchronize(c->stream);
        if (e == cudaSuccess && d) e = cudaMemcpy(d, dd, n * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && rate) e = cudaMemcpy(rate, dr, n * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && row_ptr) {
            e = cudaMemcpy(row_ptr, drp, n * 8, cudaMemcpyDeviceToHost);
            row_ptr[n] = static_cast<int64_t>(m);
        }
        if (e == cudaSuccess && cdf) e = cudaMemcpy(cdf, dc, m * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && target) e = cudaMemcpy(target, dt, m * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && sign) e = cudaMemcpy(sign, ds, m, cudaMemcpyDeviceToHost);
        for (void* p : {static_cast<void*>(dd), static_cast<void*>(dr), static_cast<void*>(drp), static_cast<void*>(dc),
                        static_cast<void*>(dt), static_cast<void*>(ds)})
            dev_free(p, c->stream);
        cuda_check(e, "export tables");
    });
}

int expmc_ctx_export_alias(const expmc_ctx* c, double* prob, int64_t* self, int64_t* alias, uint64_t* rows) {
    return guarded([&] {
        need(c != nullptr, EXPMC_EINVAL, "null context");
        if (rows) *rows = c->alias_rows;
        if (!prob && !self && !alias) return;
        need(c->alias != nullptr, EXPMC_EINVAL, "no alias table (select the event sampler on a matrix with non-uniform rows)");
        bind(c);
        const uint64_t m = c->nedges;
        double* dp = nullptr;
        int64_t *ds = nullptr, *da = nullptr;
        dev_alloc(&dp, m, c->stream); dev_alloc(&ds, m, c->stream); dev_alloc(&da, m, c->stream);
        launch_export_alias(m, c->alias, dp, ds, da, c->stream);
        cudaError_t e = cudaStreamSynchronize(c->stream);
        if (e == cudaSuccess && prob) e = cudaMemcpy(prob, dp, m * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && self) e = cudaMemcpy(self, ds, m * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && alias) e = cudaMemcpy(alias, da, m * 8, cudaMemcpyDeviceToHost);
        for (void* p : {static_cast<void*>(dp), static_cast<void*>(ds), static_cast<void*>(da)}) dev_free(p, c->stream);
        cuda_check(e, "export alias");
    });
}

int expmc_ctx_get_counters(const expmc_ctx* c, expmc_counters* out) {
    return guarded([&] {
        need(c && out, EXPMC_EINVAL, "null argument");
        *out = c->ctr;
    });
}

int expmc_ctx_set_sampler(expmc_ctx* c, int32_t mode) {
    return guarded([&] {
        need(c != nullptr, EXPMC_EINVAL, "null context");
        need(mode == EXPMC_SAMPLER_REFERENCE || mode == EXPMC_SAMPLER_EVENT, EXPMC_EINVAL, "unknown sampler mode");
        c->sampler = mode;
        c->sampler_grid = mode == EXPMC_SAMPLER_EVENT ? c->sampler_grid_ed : c->sampler_grid_ref;
        if (mode == EXPMC_SAMPLER_EVENT) ensure_event_tables(c);
    });
}

int expmc_ctx_set_sampler_flags(expmc_ctx* c, uint32_t flags) {
    return guarded([&] {
        need(c != nullptr, EXPMC_EINVAL, "null context");
        need((flags & ~(EXPMC_SAMPLER_FLAG_FULL_HOLD | EXPMC_SAMPLER_FLAG_LOG_HOLD | EXPMC_SAMPLER_FLAG_SCREEN_EACH |
                        EXPMC_SAMPLER_FLAG_ROW_GATHER)) == 0u,
             EXPMC_EINVAL,
             "unknown sampler flag");
        c->sampler_flags = flags;
    });
}

int expmc_ctx_get_sampler(const expmc_ctx* c, int32_t* mode) {
    return guarded([&] {
        need(c && mode, EXPMC_EINVAL, "null argument");
        *mode = c->sampler;
    });
}

int expmc_nccl_unique_id(uint8_t* id) {
    return guarded([&] {
        need(id != nullptr, EXPMC_EINVAL, "null argument");
        static_assert(sizeof(ncclUniqueId) == EXPMC_NCCL_ID_BYTES, "NCCL id size");
        ncclUniqueId u;
        nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof u);
    });
}

int expmc_ctx_shard_samples(expmc_ctx* c, const uint8_t* id, int32_t rank, int32_t world) {
    return guarded([&] {
        need(c && id, EXPMC_EINVAL, "null argument");
        need(world >= 1 && rank >= 0 && rank < world, EXPMC_EINVAL, "bad rank / world");
        bind(c);
        if (c->nccl) {
            nccl().comm_destroy(c->nccl);
            c->nccl = nullptr;
        }
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        nccl_check(nccl().comm_init_rank(&c->nccl, world, u, rank), "ncclCommInitRank");
        c->shard_rank = rank;
        c->shard_world = world;
    });
}

int expmc_ctx_set_shard(expmc_ctx* c, int32_t rank, int32_t world) {
    return guarded([&] {
        need(c != nullptr, EXPMC_EINVAL, "null context");
        need(world >= 1 && rank >= 0 && rank < world, EXPMC_EINVAL, "bad rank / world");
        need(c->nccl == nullptr || world == c->shard_world, EXPMC_EINVAL, "context is attached to an NCCL group");
        c->shard_rank = rank;
        c->shard_world = world;
    });
}

int expmc_ctx_last_partials(const expmc_ctx* c, int64_t* count, double* sum, double* sum_sq, uint64_t* cost,
                            uint64_t* jumps) {
    return guarded([&] {
        need(c && count, EXPMC_EINVAL, "null argument");
        bind(c);
        const uint64_t w = c->last_window;
        *count = static_cast<int64_t>(w);
        if (w == 0) return;
        cudaError_t e = cudaSuccess;
        if (sum) e = cudaMemcpy(sum, c->d_pf, w * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && sum_sq) e = cudaMemcpy(sum_sq, c->d_pf + c->cap_partials, w * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && cost) e = cudaMemcpy(cost, c->d_pu, w * 8, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && jumps) e = cudaMemcpy(jumps, c->d_pu + c->cap_partials, w * 8, cudaMemcpyDeviceToHost);
        cuda_check(e, "copy partials");
    });
}

int expmc_ctx_get_stream(const expmc_ctx* c, void** stream) {
    return guarded([&] {
        need(c && stream, EXPMC_EINVAL, "null argument");
        *stream = static_cast<void*>(c->stream);
    });
}

int expmc_selftest_exp(int device, int64_t n, const double* x, double* out) {
    return guarded([&] {
        need(n >= 0 && (n == 0 || (x && out)), EXPMC_EINVAL, "null argument");
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        double* d = nullptr;
        cuda_check(cudaMalloc(&d, std::max<int64_t>(1, 3 * n) * sizeof(double)), "cudaMalloc");
        try {
            cuda_check(cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
            math_check(d, n, d + n, nullptr);
            cuda_check(cudaMemcpy(out, d + n, 2 * n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        } catch (...) {
            cudaFree(d);
            throw;
        }
        cudaFree(d);
    });
}

int expmc_bench_gather(int device, uint64_t bytes, int32_t loads_per_thread, int32_t reps, double* gbps) {
    return guarded([&] {
        need(gbps != nullptr && bytes >= 64 && loads_per_thread > 0 && reps > 0, EXPMC_EINVAL, "bad gather arguments");
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        int sms = 0;
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
        uint64_t loads = 0;
        const float ms = bench_gather(bytes, loads_per_thread, reps, sms, &loads);
        *gbps = static_cast<double>(loads) * 32.0 / (static_cast<double>(ms) * 1e-3) / 1e9;
    });
}

int expmc_ctx_reset_counters(expmc_ctx* c) {
    return guarded([&] {
        need(c != nullptr, EXPMC_EINVAL, "null context");
        c->ctr = expmc_counters{};
    });
}

int expmc_run_level(expmc_ctx* c, int64_t entry, double beta, int32_t level, int32_t base_level, uint64_t first_index,
                    uint64_t additional, uint64_t seed, expmc_level_stats* out) {
    return guarded([&] {
        need(c && out, EXPMC_EINVAL, "null argument");
        expmc_level_req r{entry, seed, first_index, additional, level, base_level};
        run_level_batch(c, beta, EXPMC_LANE_ENTRY, &r, 1, out);
    });
}

int expmc_run_level_forward(expmc_ctx* c, double beta, int32_t level, int32_t base_level, uint64_t first_index,
                            uint64_t additional, uint64_t seed, expmc_level_stats* out) {
    return guarded([&] {
        need(c && out, EXPMC_EINVAL, "null argument");
        expmc_level_req r{0, seed, first_index, additional, level, base_level};
        run_level_batch(c, beta, EXPMC_LANE_FORWARD, &r, 1, out);
    });
}

int expmc_run_level_fem(expmc_ctx* c, int64_t entry, double beta, int32_t level, int32_t base_level,
                        uint64_t first_index, uint64_t additional, uint64_t seed, expmc_level_stats* out) {
    return guarded([&] {
        need(c && out, EXPMC_EINVAL, "null argument");
        expmc_level_req r{entry, seed, first_index, additional, level, base_level};
        run_level_batch(c, beta, EXPMC_LANE_FEM, &r, 1, out);
    });
}

int expmc_run_level_batch(expmc_ctx* c, double beta, uint32_t lane, int64_t nreq, const expmc_level_req* req,
                          expmc_level_stats* out) {
    return guarded([&] {
        need(c && (nreq == 0 || (req && out)), EXPMC_EINVAL, "null argument");
        need(lane <= EXPMC_LANE_FEM, EXPMC_ENOTIMPL, "unknown sampling lane (0 entry, 1 forward, 2 fem)");
        run_level_batch(c, beta, lane, req, nreq, out);
    });
}

int expmc_sample_debug(expmc_ctx* c, double beta, uint32_t lane, int64_t nreq, const expmc_level_req* req,
                       double* eta_fine, double* eta_coarse, uint64_t* cost, uint64_t* jumps, int64_t* end_state) {
    return guarded([&] {
        need(c && (nreq == 0 || req), EXPMC_EINVAL, "null argument");
        const std::vector<SampleOut> o = sample_debug(c, beta, lane, nreq, req);
        for (int64_t i = 0; i < nreq; ++i) {
            if (eta_fine) eta_fine[i] = o[i].fine;
            if (eta_coarse) eta_coarse[i] = o[i].coarse;
            if (cost) cost[i] = o[i].cost;
            if (jumps) jumps[i] = o[i].jumps;
            if (end_state) end_state[i] = o[i].end_state;
        }
    });
}

int expmc_sample_debug_ex(expmc_ctx* c, double beta, uint32_t lane, int64_t nreq, const expmc_level_req* req,
                          expmc_sample_record* out) {
    return guarded([&] {
        need(c && (nreq == 0 || (req && out)), EXPMC_EINVAL, "null argument");
        const std::vector<SampleOut> o = sample_debug(c, beta, lane, nreq, req);
        for (int64_t i = 0; i < nreq; ++i)
            out[i] = expmc_sample_record{o[i].fine, o[i].coarse, o[i].value, o[i].integ_f, o[i].integ_c,
                                         o[i].cost, o[i].jumps, o[i].end_state};
    });
}

int expmc_ctx_set_load(expmc_ctx* c, const double* load) {
    return guarded([&] {
        need(c && (load || c->n == 0), EXPMC_EINVAL, "null argument");
        if (c->n == 0) return;
        bind(c);
        if (!c->d_load) dev_alloc(&c->d_load, c->n, c->stream);
        cuda_check(cudaMemcpyAsync(c->d_load, load, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
        c->ctr.h2d_bytes += c->n * sizeof(double);
        cuda_check(cudaStreamSynchronize(c->stream), "set load");
    });
}

int expmc_ctx_create_scaled(const expmc_csr* A, const double* row_scale, const double* u, int device,
                            expmc_ctx** out) {
    int rc = EXPMC_OK;
    std::vector<double> val;
    expmc_csr scaled{};
    rc = guarded([&] {
        need(A != nullptr && out != nullptr, EXPMC_EINVAL, "null argument");
        need(A->n >= 0, EXPMC_EINVAL, "matrix dimension must be nonnegative");
        need(A->n == 0 || (A->row_ptr && row_scale), EXPMC_EINVAL, "null CSR or row scale");
        need(A->n == 0 || A->nnz == 0 || A->val, EXPMC_EINVAL, "null CSR arrays");
        // decompose_impl's row loop (chain.cpp:29-38): scale checked first, then each v = s a_ij
        val.resize(static_cast<size_t>(A->nnz > 0 ? A->nnz : 0));
        for (int64_t i = 0; i < A->n; ++i) {
            const double sc = row_scale[i];
            need(std::isfinite(sc), EXPMC_EINVAL, "row scale is NaN or Inf");
            for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1] && k < A->nnz; ++k) {
                val[static_cast<size_t>(k)] = sc * A->val[k];
                need(std::isfinite(val[static_cast<size_t>(k)]), EXPMC_EINVAL, "matrix entry is NaN or Inf");
            }
        }
        scaled = *A;
        scaled.val = val.data();
    });
    if (rc != EXPMC_OK) return rc;
    return expmc_ctx_create(&scaled, u, device, out);
}

}  // extern "C"
