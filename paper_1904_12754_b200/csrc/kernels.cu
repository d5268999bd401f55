// sm_100a kernels of the MLMC random-walk estimator.
//
//  k_sample   -- path sampler + level coupling + per-chunk reduction (the hot kernel).
//                Replaces parallel_samples<SumAcc> (parallel.hpp:31-54) around
//                LevelSampler::single/coupled (paths.cpp:99-141) in run_level_ex
//                (mlmc.cpp:76-148).  One warp owns one 512-sample chunk (parallel.hpp:20);
//                lanes pull the chunk's samples dynamically (a lane that finishes a path
//                starts the next unclaimed sample at once), so warp time tracks the mean
//                path length, not the longest path.  The chunk's (sum, sum_sq, cost, jumps)
//                is reduced with a fixed xor-shuffle tree -> deterministic, independent of
//                grid size, GPU count and scheduling.
//  k_sample_grouped -- the event sampler's entry-mode variant: closed-form samples screened
//                out over groups of 4 chunks, one walker pass over the rest (ed_walker.cuh).
//  k_combine  -- per-item ordered combine of the chunk partials (SumAcc::combine in
//                ascending chunk order, parallel.hpp:52); a tree for event-sampler batches.
//  k_debug    -- one thread per requested sample (golden per-sample parity).
//  k_count_edges / k_fill_tables (+ _heavy: hub rows, a warp each) -- the transition-table
//                builder (decompose_impl, chain.cpp:15-71) straight from CSR on the device.
#include <cub/device/device_scan.cuh>

#include "internal.hpp"
#include "ed_walker.cuh"
#include "fem_walker.cuh"
#include "walker.cuh"

namespace expmc_b200 {

namespace {

#ifndef EXPMC_SAMPLER_MINB
#define EXPMC_SAMPLER_MINB 4  // resident 256-thread blocks per SM the sampler is register-budgeted for
#endif

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t find_item(const uint64_t* __restrict__ chunk0, uint32_t nitems,
                                              uint64_t g, uint32_t hint) {
    // chunk0 is non-decreasing; find the last i with chunk0[i] <= g (items with zero chunks
    // never occur: count == 0 requests are dropped on the host).  Warps draw chunk ids in
    // increasing order, so gallop forward from the previous item first.
    uint32_t lo = hint;
    if (lo >= nitems || chunk0[lo] > g) lo = 0;
    uint32_t step = 1, hi = lo + 1;
    while (hi < nitems && chunk0[hi] <= g) {
        lo = hi;
        hi = lo + step;
        step <<= 1;
    }
    if (hi > nitems) hi = nitems;
    // invariant: chunk0[lo] <= g, and (hi == nitems or chunk0[hi] > g)
    while (hi - lo > 1) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (chunk0[mid] <= g) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Chan's pairwise merge of Welford accumulators (WelfordAcc::combine, parallel.hpp:92-104),
// in the reference's evaluation order.
__device__ __forceinline__ void welford_merge(double& mean, double& m2, uint64_t& n, double omean, double om2,
                                              uint64_t on) {
    if (on == 0) return;
    if (n == 0) {
        mean = omean;
        m2 = om2;
        n = on;
        return;
    }
    const double delta = __dsub_rn(omean, mean);
    const double total = static_cast<double>(n + on);
    mean = __dadd_rn(mean, __dmul_rn(delta, __ddiv_rn(static_cast<double>(on), total)));
    m2 = __dadd_rn(m2, __dadd_rn(om2, __dmul_rn(__dmul_rn(delta, delta),
                                                 __ddiv_rn(__dmul_rn(static_cast<double>(n), static_cast<double>(on)),
                                                           total))));
    n += on;
}

// The path sampler.  Sums (W = false): per-chunk (sum x, sum x^2, cost, jumps) for run_level
// (SumAcc).  Welford (W = true): the classical-MC accumulator (WelfordAcc, parallel.hpp:80-104):
// every sample's value is parked in its chunk slot in shared memory and lane 0 folds the chunk
// in sample order -- the reference's sequential Welford, so mc_* results match it.
// %lanemask_lt read where it is used (one S2R) instead of a value kept live across the loop.
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

#ifndef EXPMC_DEFER
#define EXPMC_DEFER 0
#endif
constexpr uint32_t kQueue = 64;  // deferred-finish ring per warp (pending < 32 + 32)

template <class P, bool W>
__global__ void __launch_bounds__(kThreads, P::kMinBlocks) k_sample(SamplerArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned full = 0xFFFFFFFFu;
    // Deferred finish (reference-order sums): a finishing lane queues its end record in shared
    // memory and restarts at once; the values are computed 32 at a time by the whole warp
    // instead of by the ~1/3 of the lanes that finish in a given trip.
    constexpr bool kDefer = P::kDefer && !W && EXPMC_DEFER;
    __shared__ double s_qa[kDefer ? kWarps * kQueue : 1], s_qb[kDefer ? kWarps * kQueue : 1];
    __shared__ uint32_t s_qs[kDefer ? kWarps * kQueue : 1];
    double* const qa = s_qa + (kDefer ? (threadIdx.x >> 5) * kQueue : 0);
    double* const qb = s_qb + (kDefer ? (threadIdx.x >> 5) * kQueue : 0);
    uint32_t* const qs = s_qs + (kDefer ? (threadIdx.x >> 5) * kQueue : 0);
    __shared__ double s_x[W ? kWarps * kChunk : 1];
    double* const wx = s_x + (W ? (threadIdx.x >> 5) * kChunk : 0);
    // screened policies: the chunk's slots that need the full walker, ascending
    __shared__ uint16_t s_list[P::kScreen ? kWarps * kChunk : 1];
    uint16_t* const wl = s_list + (P::kScreen ? (threadIdx.x >> 5) * kChunk : 0);
    __shared__ LogEntry s_log[128];
    load_log_table(s_log);
    __syncthreads();
    __shared__ ItemConst s_ic[kWarps];  // per-warp item constants: read at use, not held in registers
    ItemConst& ic = s_ic[threadIdx.x >> 5];
    uint32_t hint = 0;
    uint32_t prepared = 0xFFFFFFFFu;  // the item whose constants ic holds (chunks of an item come in runs)
    // sample sharding: this GPU owns the chunks g = own0 + k * world of the window
    const uint64_t rem = a.g_begin % a.shard_world;
    const uint64_t own0 = a.g_begin + (a.shard_rank + a.shard_world - rem) % a.shard_world;
    for (;;) {
        uint32_t gi = 0;
        if (lane == 0) gi = atomicAdd(a.counter, 1u);
        gi = __shfl_sync(full, gi, 0);
        const uint64_t g = own0 + static_cast<uint64_t>(gi) * a.shard_world;
        if (g >= a.g_end) return;

        const uint32_t item = find_item(a.chunk0, a.nitems, g, hint);
        hint = item;
        if (item != prepared) {  // warp-uniform
            if (lane == 0) {
                ItemConst c = load_item(a.items, item);
                P::prepare(c, a.rows, a.init, a.flags);
                ic = c;
            }
            __syncwarp();
            prepared = item;
        }
        const DevItem& it = a.items[item];
        const uint64_t first = it.first, end = it.first + it.count;
        const uint64_t chunk = first / kChunk + (g - a.chunk0[item]);
        const uint64_t lo = first > chunk * kChunk ? first : chunk * kChunk;
        const uint64_t hi = end < (chunk + 1) * kChunk ? end : (chunk + 1) * kChunk;
        // parallel.hpp:46-49 in uint64: for the chunk ending at 2^64 the reference's bound
        // (chunk + 1) * kChunk wraps to 0 and its sample loop runs zero times -- so does this one
        const uint32_t cnt = hi > lo ? static_cast<uint32_t>(hi - lo) : 0u;

        double sum = 0.0, sum_sq = 0.0, extra = 0.0;
        unsigned long long cost = 0, jumps = 0;
        // Work list of the walker loop: slots 0..cnt-1 of the chunk or -- when the item has a
        // closed-form first hold (ed_walker.cuh) -- only the slots that a converged screening
        // pass found to need the full walker.  The screen costs one Philox block per sample with
        // every lane busy; closed-form samples never enter the divergent walker loop.
        uint32_t nwork = cnt;
        bool listed = false;
        if constexpr (P::kScreen) {
            if (ic.m_safe != 0) {
                listed = true;
                nwork = 0;
                uint32_t nheld = 0;  // this lane's closed-form samples, all of value hold_x
                for (uint32_t j0 = 0; j0 < cnt; j0 += 32u) {
                    const uint32_t j = j0 + lane;
                    const bool valid = j < cnt;
                    const bool held = valid && P::screen(ic, lo + j);
                    if constexpr (W) {
                        if (held) wx[j] = ic.hold_x;
                    }
                    nheld += held;
                    const unsigned need = __ballot_sync(full, valid && !held);
                    if (valid && !held) wl[nwork + __popc(need & lanemask_lt())] = static_cast<uint16_t>(j);
                    nwork += __popc(need);
                }
                if constexpr (!W) {  // n equal terms: n x and n x^2 (the statistical sampler's sums)
                    const double hx = ic.hold_x, k = static_cast<double>(nheld);
                    sum = __dmul_rn(k, hx);
                    sum_sq = __dmul_rn(k, __dmul_rn(hx, hx));
                }
                cost += static_cast<unsigned long long>(nheld) * ic.nsteps;  // N rejected draws each (ed_segment(0, N))
                __syncwarp();
            }
        }
        typename P::W w;
        // The running sample's slot in the chunk; kIdle: the lane has no sample (no separate flag:
        // a bool kept across the loop costs byte-permute instructions on every trip).
        constexpr uint32_t kIdle = 0xFFFFFFFFu;
        uint32_t my = kIdle;
        // A chunk's samples share their upper 32 index bits (chunks are 512-aligned), so sample
        // lo + my is (lo's upper word, lo's lower word + my) without a carry: the stream's second
        // counter word is chunk-invariant.
        const uint64_t lo_hi = lo & 0xFFFFFFFF00000000ull;
        const uint32_t lo_lo = static_cast<uint32_t>(lo);
        // Lanes start work entries 0..31; a lane whose sample ends takes the next unstarted
        // entry in the same divergent section as its finish (one ballot per trip).
        if (lane < nwork) {
            my = listed ? wl[lane] : lane;
            P::start(w, ic, a.init, a.rows, lo_hi | (lo_lo + my));
        }
        // next: work entries started so far, uncapped (min(nwork, 32) at first, + 1 per finished
        // sample): the loop ends when every entry has finished, next == nwork + min(nwork, 32) -- a
        // warp-uniform compare instead of a vote over the lanes' idle flags
        uint32_t next = nwork < 32u ? nwork : 32u;
        const uint32_t next_end = nwork + next;
        uint32_t qh = 0, qn = 0;  // deferred finish: ring head and pending records (warp-uniform)
        while (next != next_end) {
            const bool done = my != kIdle && P::event(w, ic, a.init, a.rows, a.edges, s_log, cost, jumps);
            const unsigned fin = __ballot_sync(full, done);
            if (done) {
                if constexpr (kDefer) {
                    double ra, rb;
                    uint32_t se;
                    P::end_record(w, ic, ra, rb, se);
                    const uint32_t slot = (qh + qn + __popc(fin & lanemask_lt())) & (kQueue - 1u);
                    qa[slot] = ra;
                    qb[slot] = rb;
                    qs[slot] = se;
                } else {
                    double ex;
                    const double x = P::sample(w, ic, a.init, a.rows, ex);
                    if constexpr (W) {
                        wx[my] = x;
                    } else {
                        sum = __dadd_rn(sum, x);
                        sum_sq = __dadd_rn(sum_sq, __dmul_rn(x, x));
                        if constexpr (P::kExtra) extra = __dadd_rn(extra, ex);
                    }
                }
                const uint32_t mine = next + __popc(fin & lanemask_lt());
                if (mine < nwork) {
                    my = listed ? wl[mine] : mine;
                    P::start(w, ic, a.init, a.rows, lo_hi | (lo_lo + my));
                } else {
                    my = kIdle;
                }
            }
            next += __popc(fin);
            if constexpr (kDefer) {
                qn += __popc(fin);
                if (qn >= 32u) {  // a converged pass over 32 records
                    __syncwarp();
                    const uint32_t slot = (qh + lane) & (kQueue - 1u);
                    const double x = P::value(qa[slot], qb[slot], qs[slot], ic, a.init, a.rows);
                    sum = __dadd_rn(sum, x);
                    sum_sq = __dadd_rn(sum_sq, __dmul_rn(x, x));
                    qh = (qh + 32u) & (kQueue - 1u);
                    qn -= 32u;
                    __syncwarp();  // the slots are rewritten by later finishes
                }
            }
        }
        if constexpr (kDefer) {  // drain the ring
            __syncwarp();
            if (lane < qn) {
                const uint32_t slot = (qh + lane) & (kQueue - 1u);
                const double x = P::value(qa[slot], qb[slot], qs[slot], ic, a.init, a.rows);
                sum = __dadd_rn(sum, x);
                sum_sq = __dadd_rn(sum_sq, __dmul_rn(x, x));
            }
            __syncwarp();
        }
        if constexpr (W) {  // WelfordAcc::add over the chunk in sample order (parallel.hpp:86-92)
            __syncwarp();
            if (lane == 0) {
                double mean = 0.0, m2 = 0.0;
                for (uint32_t k = 0; k < cnt; ++k) {
                    const double x = wx[k];
                    const double delta = __dsub_rn(x, mean);
                    mean = __dadd_rn(mean, __ddiv_rn(delta, static_cast<double>(k + 1)));
                    m2 = __dadd_rn(m2, __dmul_rn(delta, __dsub_rn(x, mean)));
                }
                sum = mean;
                sum_sq = m2;
            }
            __syncwarp();
        }
        // the fine steps of every sample (cost = draws + steps, paths.hpp:22-23): cnt N, once
        if (lane == 0) cost += static_cast<unsigned long long>(cnt) * ic.nsteps;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            if constexpr (!W) sum = __dadd_rn(sum, __shfl_xor_sync(full, sum, o));
            if constexpr (!W) sum_sq = __dadd_rn(sum_sq, __shfl_xor_sync(full, sum_sq, o));
            if constexpr (P::kExtra) extra = __dadd_rn(extra, __shfl_xor_sync(full, extra, o));
            cost += __shfl_xor_sync(full, cost, o);
            jumps += __shfl_xor_sync(full, jumps, o);
        }
        if (lane == 0) {
            const uint64_t k = g - a.part_base;
            a.partials.sum[k] = sum;
            a.partials.sum_sq[k] = sum_sq;
            if constexpr (P::kExtra) a.partials.extra[k] = extra;
            a.partials.cost[k] = cost;
            a.partials.jumps[k] = jumps;
        }
    }
}

// Geometric screen of one chunk (ed_walker.cuh): append the chunk's jumpers to the warp's work
// list wl[nwork..] as (slot << 9) | offset and return the new list length.  Gaps come 32 at a
// time from the chunk's own Philox stream (lane kSkipLane, counter = absolute chunk index) and
// are placed by a warp prefix sum.  One accurate log per 32 gaps (libdevice: off the hot path).
__device__ __forceinline__ uint32_t geometric_screen(const ItemConst& ic, uint64_t chunk, uint32_t off, uint32_t cnt,
                                                     uint32_t slot, uint16_t* wl, uint32_t nwork) {
    const unsigned full = 0xFFFFFFFFu;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t k3 = (ic.key3 & 0x00FFFFFFu) | (kSkipLane << 24);
    const uint32_t k0 = static_cast<uint32_t>(ic.seed), k1 = static_cast<uint32_t>(ic.seed >> 32);
    const double scale = ic.skip_scale;
    // Positions are offsets in the WHOLE chunk (sample chunk*512 + p): a chunk that run_level
    // extensions split (samples [lo, hi) of it now, the rest in a later call) must see the same
    // jumper set in both calls, so the gaps are always laid from the chunk's first sample and
    // this call keeps the jumpers in [off, off + cnt).  Listed entries are offsets from lo.
    const uint32_t end = off + cnt;
    uint32_t pos = 0;
    for (uint32_t it = 0; pos < end; ++it) {  // warp-uniform
        uint32_t c0 = it * 32u + lane, c1 = static_cast<uint32_t>(chunk), c2 = static_cast<uint32_t>(chunk >> 32), c3 = k3;
        philox10(c0, c1, c2, c3, k0, k1);
        const uint64_t k53 = ((static_cast<uint64_t>(c2) << 32) | c3) >> 11;  // rng.hpp:32-35
        // U = M 2^-53 in (0, 1]; G = floor(log U / log p) >= 0, capped (only G < cnt matters)
        const double lu = log(__dmul_rn(static_cast<double>((uint64_t{1} << 53) - k53), 0x1.0p-53));
        const double gf = __dmul_rn(lu, scale);
        uint32_t incl = (gf < 1048576.0 ? static_cast<uint32_t>(gf) : 1048576u) + 1u;  // gap + 1
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // inclusive warp prefix sum
            const uint32_t y = __shfl_up_sync(full, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t p = pos + incl - 1u;  // this lane's jumper
        const bool jump = p >= off && p < end;
        const unsigned need = __ballot_sync(full, jump);
        if (jump) wl[nwork + __popc(need & lanemask_lt())] = static_cast<uint16_t>((slot << 9) | (p - off));
        nwork += __popc(need);
        pos += __shfl_sync(full, incl, 31);
    }
    return nwork;
}

// Screened event sampler, chunk groups (EdPolicy<false>, sums): a warp claims an aligned group
// of kGroup consecutive chunks of its window and screens all of an item's chunks in the group before it runs the
// walker loop, so the few samples that jump (5-10 % on C3/C4) fill the lanes of one walker pass
// instead of a fraction of 32 per chunk.  The portion's totals go to its first chunk's partial
// and the other chunks of the portion get zeros; the event sampler's combine is an unordered
// sum, so the item totals are the same terms (determinism: the group boundaries are fixed and
// the lane assignment is the ballot's, as in k_sample).
#ifndef EXPMC_GROUP
#define EXPMC_GROUP 4
#endif
constexpr uint32_t kGroup = EXPMC_GROUP;

// The grouped kernel runs at 3 blocks per SM (85 registers): its walker loop spills at 64 once
// the geometric screen shares the kernel (C4 65,536-component step 142 -> 136 ms, C3 1486 ->
// 1375 ms against 4 blocks per SM; profiles/r02/SUMMARY.md).
#ifndef EXPMC_GROUPED_MINB
#define EXPMC_GROUPED_MINB 3
#endif

template <class P>
__global__ void __launch_bounds__(kThreads, EXPMC_GROUPED_MINB) k_sample_grouped(SamplerArgs a) {
    static_assert(P::kScreen && !P::kExtra, "grouped chunks: screened policies only");
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wid = threadIdx.x >> 5;
    const unsigned full = 0xFFFFFFFFu;
    __shared__ uint16_t s_list[kWarps * kGroup * kChunk];  // (group slot << 9) | offset in chunk
    uint16_t* const wl = s_list + wid * kGroup * kChunk;
    __shared__ uint64_t s_lo[kWarps][kGroup];              // first sample of each group slot
    __shared__ LogEntry s_log[128];
    load_log_table(s_log);
    __syncthreads();
    __shared__ ItemConst s_ic[kWarps];
    ItemConst& ic = s_ic[wid];
    // The portion cursor lives in shared memory, not registers: it is dead during the walker
    // loop, which needs every register it can get (64 at 4 blocks per SM).
    struct Cursor {
        uint64_t gq, ghi;            // the claimed group's first chunk id, end of its window part
        unsigned long long nsamp;    // samples of the current portion
        uint32_t j, j0, hint;        // next slot, the portion's first slot, find_item hint
    };
    __shared__ Cursor s_cur[kWarps];
    Cursor& cur = s_cur[wid];
    if (lane == 0) cur.hint = 0;
    // Groups are aligned blocks of kGroup absolute chunk ids, dealt to the ranks of a sample-
    // sharded run whole (group q on rank q % world): the portions -- and so every chunk
    // partial -- are the same for any GPU count, and the all-reduced window is the one-GPU one.
    const uint64_t q_begin = a.g_begin / kGroup;
    const uint64_t qrem = q_begin % a.shard_world;
    const uint64_t qown = q_begin + (a.shard_rank + a.shard_world - qrem) % a.shard_world;
    for (;;) {
        uint32_t gi = 0;
        if (lane == 0) gi = atomicAdd(a.counter, 1u);
        gi = __shfl_sync(full, gi, 0);
        {
            const uint64_t gq = (qown + static_cast<uint64_t>(gi) * a.shard_world) * kGroup;  // first chunk id
            if (gq >= a.g_end) return;
            const uint64_t glo = gq > a.g_begin ? gq : a.g_begin;
            if (lane == 0) {
                cur.gq = gq;
                cur.ghi = gq + kGroup < a.g_end ? gq + kGroup : a.g_end;
                cur.j = static_cast<uint32_t>(glo - gq);
            }
            __syncwarp();
        }
        for (;;) {
            uint32_t nwork = 0, nheld = 0;
            {
                const uint64_t gq = cur.gq, ghi = cur.ghi;
                uint32_t j = cur.j;
                if (gq + j >= ghi) break;
                const uint32_t item = find_item(a.chunk0, a.nitems, gq + j, cur.hint);
                __syncwarp();
                if (lane == 0) {
                    cur.hint = item;
                    ItemConst c = load_item(a.items, item);
                    P::prepare(c, a.rows, a.init, a.flags | kFlagGrouped);
                    ic = c;
                }
                __syncwarp();
                const DevItem& it = a.items[item];
                const uint64_t first = it.first, end = it.first + it.count;
                const uint64_t item_g1 = a.chunk0[item + 1];
                // ---- screen the portion: the group's chunks of this item
                const uint32_t j0 = j;
                unsigned long long nsamp = 0;
                for (; gq + j < ghi; ++j) {
                    const uint64_t g = gq + j;
                    if (g >= item_g1) break;
                    const uint64_t chunk = first / kChunk + (g - a.chunk0[item]);
                    const uint64_t lo = first > chunk * kChunk ? first : chunk * kChunk;
                    const uint64_t hi = end < (chunk + 1) * kChunk ? end : (chunk + 1) * kChunk;
                    const uint32_t cnt = hi > lo ? static_cast<uint32_t>(hi - lo) : 0u;  // parallel.hpp:46-49
                    if (lane == 0) s_lo[wid][j] = lo;
                    nsamp += cnt;
                    if (ic.skip_scale != 0.0) {
                        const uint32_t n1 = geometric_screen(ic, chunk, static_cast<uint32_t>(lo - chunk * kChunk), cnt, j,
                                                             wl, nwork);
                        if (lane == 0) nheld += cnt - (n1 - nwork);
                        nwork = n1;
                        continue;
                    }
                    for (uint32_t q0 = 0; q0 < cnt; q0 += 32u) {
                        const uint32_t qq = q0 + lane;
                        const bool valid = qq < cnt;
                        const bool held = valid && ic.m_safe != 0 && P::screen(ic, lo + qq);
                        nheld += held;
                        const unsigned need = __ballot_sync(full, valid && !held);
                        if (valid && !held) wl[nwork + __popc(need & lanemask_lt())] = static_cast<uint16_t>((j << 9) | qq);
                        nwork += __popc(need);
                    }
                }
                if (lane == 0) {
                    cur.j0 = j0;
                    cur.j = j;
                    cur.nsamp = nsamp;
                }
            }
            __syncwarp();
            // ---- the walker loop over the listed samples (k_sample's, entries decoded)
            const double hx = ic.hold_x, kh = static_cast<double>(nheld);
            double sum = __dmul_rn(kh, hx), sum_sq = __dmul_rn(kh, __dmul_rn(hx, hx));
            unsigned long long cost = static_cast<unsigned long long>(nheld) * ic.nsteps, jumps = 0;
            typename P::W w;
            bool active = false;
            if (lane < nwork) {
                const uint32_t e = wl[lane];
                P::start(w, ic, a.init, a.rows, s_lo[wid][e >> 9] + (e & 511u));
                active = true;
            }
            uint32_t next = nwork < 32u ? nwork : 32u;
            while (__any_sync(full, active)) {
                const bool done = active && P::event(w, ic, a.init, a.rows, a.edges, s_log, cost, jumps);
                const unsigned fin = __ballot_sync(full, done);
                if (done) {
                    double ex;
                    const double x = P::sample(w, ic, a.init, a.rows, ex);
                    sum = __dadd_rn(sum, x);
                    sum_sq = __dadd_rn(sum_sq, __dmul_rn(x, x));
                    const uint32_t mine = next + __popc(fin & lanemask_lt());
                    if (mine < nwork) {
                        const uint32_t e = wl[mine];
                        P::start(w, ic, a.init, a.rows, s_lo[wid][e >> 9] + (e & 511u));
                    } else {
                        active = false;
                    }
                }
                next += __popc(fin);
            }
            __syncwarp();  // the cursor is re-read from shared memory, not held across the loop
            if (lane == 0) cost += cur.nsamp * ic.nsteps;  // the fine steps of every sample
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sum = __dadd_rn(sum, __shfl_xor_sync(full, sum, o));
                sum_sq = __dadd_rn(sum_sq, __shfl_xor_sync(full, sum_sq, o));
                cost += __shfl_xor_sync(full, cost, o);
                jumps += __shfl_xor_sync(full, jumps, o);
            }
            // portion totals on its first chunk, zeros on the rest
            const uint32_t j0 = cur.j0, j1 = cur.j;
            const uint64_t k0 = cur.gq - a.part_base;
            for (uint32_t t = j0 + lane; t < j1; t += 32u) {
                const uint64_t k = k0 + t;
                const bool head = t == j0;
                a.partials.sum[k] = head ? sum : 0.0;
                a.partials.sum_sq[k] = head ? sum_sq : 0.0;
                a.partials.cost[k] = head ? cost : 0ull;
                a.partials.jumps[k] = head ? jumps : 0ull;
            }
            __syncwarp();  // ic, the cursor and the list are rewritten by the next portion
        }
    }
}

// Ordered combines: one warp per item.  The fp64 sums must be taken in ascending chunk order
// (one dependent add per chunk), so the warp stages tiles of the item's chunk partials in
// shared memory with coalesced loads (32 in flight per lane group) and lane 0 runs the
// sequential chain out of shared memory; the integer counts are associative and are reduced
// across the lanes.  (A thread per item waited one global-load latency per chunk: 280 ms of a
// 16k-component C4 step went to the hub items' 10^4-10^5 chunks.)
constexpr int kCombWarps = 4;
constexpr int kCombTile = 256;

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    return x;
}

// ordered == false (event-driven sampler: statistical parity, no sequential order to keep):
// each lane sums a strided share of the chunks and a fixed xor tree joins the lanes -- still
// deterministic and GPU-count independent, without the sequential chain.
__global__ void __launch_bounds__(kCombWarps * 32) k_combine(const uint64_t* __restrict__ chunk0, uint32_t nitems,
                                                             uint64_t g_begin, uint64_t g_end, ChunkPartials p,
                                                             bool with_extra, bool ordered,
                                                             Partial* __restrict__ totals) {
    __shared__ double s_v[kCombWarps][3][kCombTile];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t i = blockIdx.x * kCombWarps + w;
    if (i >= nitems) return;  // warp-uniform
    const uint64_t c0 = chunk0[i] > g_begin ? chunk0[i] : g_begin;
    const uint64_t c1 = chunk0[i + 1] < g_end ? chunk0[i + 1] : g_end;
    if (c0 >= c1) return;
    double sum = 0.0, sum_sq = 0.0, extra = 0.0;
    if (lane == 0) {
        sum = totals[i].sum;
        sum_sq = totals[i].sum_sq;
        extra = totals[i].extra;
    }
    unsigned long long cost = 0, jumps = 0;
    if (!ordered) {
        double ls = 0.0, lq = 0.0, le = 0.0;
        for (uint64_t g = c0 + lane; g < c1; g += 32) {
            const uint64_t k = g - g_begin;
            ls = __dadd_rn(ls, p.sum[k]);
            lq = __dadd_rn(lq, p.sum_sq[k]);
            if (with_extra) le = __dadd_rn(le, p.extra[k]);
            cost += p.cost[k];
            jumps += p.jumps[k];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ls = __dadd_rn(ls, __shfl_xor_sync(0xFFFFFFFFu, ls, o));
            lq = __dadd_rn(lq, __shfl_xor_sync(0xFFFFFFFFu, lq, o));
            if (with_extra) le = __dadd_rn(le, __shfl_xor_sync(0xFFFFFFFFu, le, o));
        }
        sum = __dadd_rn(sum, ls);
        sum_sq = __dadd_rn(sum_sq, lq);
        extra = __dadd_rn(extra, le);
    }
    for (uint64_t base = c0; ordered && base < c1; base += kCombTile) {
        const uint32_t n = static_cast<uint32_t>(c1 - base < kCombTile ? c1 - base : kCombTile);
        for (uint32_t j = lane; j < n; j += 32) {
            const uint64_t k = base + j - g_begin;
            s_v[w][0][j] = p.sum[k];
            s_v[w][1][j] = p.sum_sq[k];
            if (with_extra) s_v[w][2][j] = p.extra[k];
            cost += p.cost[k];
            jumps += p.jumps[k];
        }
        __syncwarp();
        if (lane == 0) {  // ascending chunk order (parallel.hpp:52)
#pragma unroll 8
            for (uint32_t j = 0; j < n; ++j) {
                sum = __dadd_rn(sum, s_v[w][0][j]);
                sum_sq = __dadd_rn(sum_sq, s_v[w][1][j]);
                if (with_extra) extra = __dadd_rn(extra, s_v[w][2][j]);
            }
        }
        __syncwarp();
    }
    cost = warp_sum_u64(cost);
    jumps = warp_sum_u64(jumps);
    if (lane == 0) {
        Partial t = totals[i];
        t.sum = sum;
        t.sum_sq = sum_sq;
        if (with_extra) t.extra = extra;
        t.cost += cost;
        t.jumps += jumps;
        totals[i] = t;
    }
}

// Welford combine: per item, Chan-merge its chunks' (mean, m2, n) in ascending chunk order
// (parallel_samples' ordered combine, parallel.hpp:52).  n of a chunk is its sample count.
// Same warp-per-item staging as k_combine.
__global__ void __launch_bounds__(kCombWarps * 32) k_combine_welford(const uint64_t* __restrict__ chunk0,
                                                                     const DevItem* __restrict__ items,
                                                                     uint32_t nitems, uint64_t g_begin, uint64_t g_end,
                                                                     ChunkPartials p, Partial* __restrict__ totals) {
    __shared__ double s_v[kCombWarps][2][kCombTile];
    __shared__ uint32_t s_n[kCombWarps][kCombTile];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t i = blockIdx.x * kCombWarps + w;
    if (i >= nitems) return;
    const uint64_t c0 = chunk0[i] > g_begin ? chunk0[i] : g_begin;
    const uint64_t c1 = chunk0[i + 1] < g_end ? chunk0[i + 1] : g_end;
    if (c0 >= c1) return;
    Partial t = totals[i];  // sum = mean, sum_sq = m2, extra = n (exact below 2^53)
    uint64_t n = static_cast<uint64_t>(t.extra);
    const uint64_t first = items[i].first, end = first + items[i].count;
    unsigned long long cost = 0, jumps = 0;
    for (uint64_t base = c0; base < c1; base += kCombTile) {
        const uint32_t m = static_cast<uint32_t>(c1 - base < kCombTile ? c1 - base : kCombTile);
        for (uint32_t j = lane; j < m; j += 32) {
            const uint64_t g = base + j;
            const uint64_t k = g - g_begin;
            const uint64_t chunk = first / kChunk + (g - chunk0[i]);
            const uint64_t lo = first > chunk * kChunk ? first : chunk * kChunk;
            const uint64_t hi = end < (chunk + 1) * kChunk ? end : (chunk + 1) * kChunk;
            s_v[w][0][j] = p.sum[k];
            s_v[w][1][j] = p.sum_sq[k];
            s_n[w][j] = static_cast<uint32_t>(hi > lo ? hi - lo : 0);
            cost += p.cost[k];
            jumps += p.jumps[k];
        }
        __syncwarp();
        if (lane == 0)
            for (uint32_t j = 0; j < m; ++j) welford_merge(t.sum, t.sum_sq, n, s_v[w][0][j], s_v[w][1][j], s_n[w][j]);
        __syncwarp();
    }
    cost = warp_sum_u64(cost);
    jumps = warp_sum_u64(jumps);
    if (lane == 0) {
        t.cost += cost;
        t.jumps += jumps;
        t.extra = static_cast<double>(n);
        totals[i] = t;
    }
}

template <class P>
__global__ void k_debug(const RowRec* __restrict__ rows, EdgeTables edges,
                        const DevItem* __restrict__ items, uint32_t n, LaneData init, uint32_t flags,
                        SampleOut* __restrict__ out) {
    __shared__ LogEntry s_log[128];
    load_log_table(s_log);
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    ItemConst ic = load_item(items, i);
    P::prepare(ic, rows, init, flags);
    typename P::W w;
    P::start(w, ic, init, rows, items[i].first);
    unsigned long long draws = 0, jumps = 0;
    while (!P::event(w, ic, init, rows, edges, s_log, draws, jumps)) {
    }
    SampleOut o;
    P::record(w, ic, init, rows, o);
    o.cost = draws + ic.nsteps;
    o.jumps = jumps;
    out[i] = o;
}

// ---------------------------------------------------------------- transition-table builder
enum : unsigned { kErrNonFinite = 1u, kErrRange = 2u, kErrCanon = 4u };

// Rows with more than kHeavyNnz stored entries (graph hubs: up to ~10^5-10^6 at C3/C4) are
// handled by a warp each (k_count_heavy / k_fill_heavy); the thread-per-row kernels skip them
// and queue them.  One thread walking a hub row serialised ~200 ms of the C4 build.
constexpr int64_t kHeavyNnz = 128;

__global__ void k_count_edges(int64_t n, const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                              const double* __restrict__ val, uint64_t* __restrict__ deg, unsigned* err,
                              uint32_t* __restrict__ heavy, unsigned* nheavy) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    unsigned bad = 0;
    if (e < b) bad |= kErrCanon;
    if (e - b > kHeavyNnz) {
        heavy[atomicAdd(nheavy, 1u)] = static_cast<uint32_t>(i);
        return;
    }
    uint64_t cnt = 0;
    int64_t prev = -1;
    for (int64_t k = b; k < e; ++k) {
        const int64_t c = col[k];
        const double v = val[k];
        if (c < 0 || c >= n) bad |= kErrRange;
        if (!isfinite(v)) bad |= kErrNonFinite;
        if (c <= prev) bad |= kErrCanon;
        prev = c;
        if (c != i && v != 0.0) ++cnt;
    }
    deg[i] = cnt;
    if (bad) atomicOr(err, bad);
}

// Warp per queued heavy row: the same checks and count, lanes striding over the row.
__global__ void k_count_heavy(int64_t n, const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                              const double* __restrict__ val, uint64_t* __restrict__ deg, unsigned* err,
                              const uint32_t* __restrict__ heavy, const unsigned* nheavy) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); h < *nheavy; h += nw) {
        const int64_t i = heavy[h];
        const int64_t b = row_ptr[i], e = row_ptr[i + 1];
        unsigned bad = 0;
        unsigned long long cnt = 0;
        for (int64_t k = b + lane; k < e; k += 32) {
            const int64_t c = col[k];
            const double v = val[k];
            if (c < 0 || c >= n) bad |= kErrRange;
            if (!isfinite(v)) bad |= kErrNonFinite;
            if (k > b && c <= col[k - 1]) bad |= kErrCanon;
            if (c != i && v != 0.0) ++cnt;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
            bad |= __shfl_xor_sync(0xFFFFFFFFu, bad, o);
        }
        if (lane == 0) {
            deg[i] = cnt;
            if (bad) atomicOr(err, bad);
        }
    }
}

// decompose_impl per row (chain.cpp:29-64), same operation order: running |a_ij| sum, CDF =
// running sum / rate, last entry exactly 1, sign = (a_ij < 0), d = a_ii + rate.
__global__ void k_fill_tables(int64_t n, const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                              const double* __restrict__ val, const double* __restrict__ u,
                              const uint64_t* __restrict__ begin, RowRec* __restrict__ rows,
                              double* __restrict__ cdf, uint32_t* __restrict__ tgt) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (row_ptr[i + 1] - row_ptr[i] > kHeavyNnz) return;  // k_fill_heavy
    const uint64_t e0 = begin[i];
    uint64_t e = e0;
    double diag = 0.0, rate = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        const int64_t c = col[k];
        const double v = val[k];
        if (c == i) {
            diag = v;
            continue;
        }
        if (v == 0.0) continue;
        rate = __dadd_rn(rate, fabs(v));
        cdf[e] = rate;
        tgt[e] = static_cast<uint32_t>(c) | (v < 0.0 ? kSignBit : 0u);
        ++e;
    }
    const uint32_t deg = static_cast<uint32_t>(e - e0);
    bool uniform = true;  // cdf_j == fl((j+1)/deg) for all j: kUniformRow
    if (rate > 0.0) {
        for (uint64_t k = e0; k + 1 < e; ++k) {
            const double c = __ddiv_rn(cdf[k], rate);
            cdf[k] = c;
            uniform = uniform && c == __ddiv_rn(static_cast<double>(k - e0 + 1), static_cast<double>(deg));
        }
        cdf[e - 1] = 1.0;
    }
    RowRec r;
    r.d = __dadd_rn(diag, rate);
    r.rate = rate;
    r.u = u[i];
    r.begin = static_cast<uint32_t>(e0);
    r.deg = deg | (uniform && deg > 0 ? kUniformRow : 0u);
    rows[i] = r;
}

// The same per heavy row with one warp: tiles of 32 entries are compacted with a ballot (chain
// edges keep column order), the running |a_ij| sum stays ONE sequential fp64 chain (lane 0,
// out of shared memory) so every CDF entry is bit-identical to the thread-per-row result, and
// the normalisation / uniformity pass runs across the lanes.
constexpr int kFillWarps = 4;

__global__ void __launch_bounds__(kFillWarps * 32) k_fill_heavy(const int64_t* __restrict__ row_ptr,
                                                                const int64_t* __restrict__ col,
                                                                const double* __restrict__ val,
                                                                const double* __restrict__ u,
                                                                const uint64_t* __restrict__ begin,
                                                                RowRec* __restrict__ rows, double* __restrict__ cdf,
                                                                uint32_t* __restrict__ tgt,
                                                                const uint32_t* __restrict__ heavy,
                                                                const unsigned* nheavy) {
    __shared__ double s_a[kFillWarps][32];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const unsigned full = 0xFFFFFFFFu;
    const uint32_t nw = gridDim.x * kFillWarps;
    for (uint32_t h = blockIdx.x * kFillWarps + w; h < *nheavy; h += nw) {
        const int64_t i = heavy[h];
        const int64_t b = row_ptr[i], e = row_ptr[i + 1];
        const uint64_t e0 = begin[i];
        uint64_t pos = e0;
        double diag = 0.0, rate = 0.0;  // rate: lane 0's chain, broadcast after the row
        for (int64_t k0 = b; k0 < e; k0 += 32) {
            const int64_t k = k0 + lane;
            int64_t c = -1;
            double v = 0.0;
            if (k < e) {
                c = col[k];
                v = val[k];
                if (c == i) diag = v;  // at most one lane of one tile (canonical CSR)
            }
            const bool edge = k < e && c != i && v != 0.0;
            const unsigned m = __ballot_sync(full, edge);
            const uint32_t r = __popc(m & lanemask_lt());
            if (edge) {
                s_a[w][r] = fabs(v);
                tgt[pos + r] = static_cast<uint32_t>(c) | (v < 0.0 ? kSignBit : 0u);
            }
            __syncwarp();
            const uint32_t cntt = __popc(m);
            if (lane == 0) {
                for (uint32_t j = 0; j < cntt; ++j) {
                    rate = __dadd_rn(rate, s_a[w][j]);  // chain.cpp:39-46, column order
                    s_a[w][j] = rate;
                }
            }
            __syncwarp();
            if (lane < cntt) cdf[pos + lane] = s_a[w][lane];
            __syncwarp();
            pos += cntt;
        }
        rate = __shfl_sync(full, rate, 0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {  // diag: the one lane that saw it (others hold 0.0)
            const double od = __shfl_xor_sync(full, diag, o);
            if (od != 0.0) diag = od;
        }
        const uint32_t deg = static_cast<uint32_t>(pos - e0);
        bool uniform = true;
        if (rate > 0.0) {
            __syncwarp();  // the row's cdf stores are visible to the warp
            for (uint64_t k = e0 + lane; k + 1 < pos; k += 32) {
                const double c = __ddiv_rn(cdf[k], rate);
                cdf[k] = c;
                uniform = uniform && c == __ddiv_rn(static_cast<double>(k - e0 + 1), static_cast<double>(deg));
            }
            if (lane == 0) cdf[pos - 1] = 1.0;
        }
        uniform = __all_sync(full, uniform);
        if (lane == 0) {
            RowRec rr;
            rr.d = __dadd_rn(diag, rate);
            rr.rate = rate;
            rr.u = u[i];
            rr.begin = static_cast<uint32_t>(e0);
            rr.deg = deg | (uniform && deg > 0 ? kUniformRow : 0u);
            rows[i] = rr;
        }
    }
}

__global__ void k_set_vector(int64_t n, const double* __restrict__ u, RowRec* __restrict__ rows) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) rows[i].u = u[i];
}

__global__ void k_export_rows(int64_t n, const RowRec* __restrict__ rows, double* d, double* rate, int64_t* row_ptr) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const RowRec r = rows[i];
    if (d) d[i] = r.d;
    if (rate) rate[i] = r.rate;
    if (row_ptr) row_ptr[i] = r.begin;
}

__global__ void k_export_edges(uint64_t m, EdgeTables edges, double* cdf, int64_t* target, uint8_t* sign) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t t = edges.tgt[i];
    if (cdf) cdf[i] = edges.cdf[i];
    if (target) target[i] = t & kTargetMask;
    if (sign) sign[i] = (t & kSignBit) ? 1 : 0;
}

// ---- alias tables (event-driven sampler, non-uniform rows; AliasRec in internal.hpp)
__device__ __forceinline__ bool needs_alias(uint32_t degf) {
    return !(degf & kUniformRow) && (degf & kDegMask) > 1u;
}

__global__ void k_count_nonuniform(int64_t n, const RowRec* __restrict__ rows, unsigned long long* count) {
    unsigned long long c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c += needs_alias(rows[i].deg);
    c = warp_sum_u64(c);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(count, c);
}

// Vose's alias method, one thread per row, in place over the row's slots: q_j = p_j deg with
// p_j = cdf_j - cdf_{j-1} (the row's transition probabilities as the reference's CDF stores
// them, chain.cpp:49-58); slots with q < 1 ("small") and q >= 1 ("large") are kept as two
// stacks at the two ends of the row's scratch range; each small slot is topped up by the
// large slot on top of its stack, which gives away 1 - q_s and moves to the small stack when
// it falls below 1.  Leftovers (rounding) keep their own target with probability 1.  The row's
// implied law (prob_j + sum_{i: alias(i) = j} (1 - prob_i)) / deg equals p_j to rounding
// (tests/test_alias.py).  O(deg) per row; hub rows take one thread longer, once per context.
__global__ void k_build_alias(int64_t n, const RowRec* __restrict__ rows, EdgeTables e, AliasRec* __restrict__ al,
                              uint32_t* __restrict__ scratch) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t degf = rows[i].deg;
    if (!needs_alias(degf)) return;
    const uint32_t b = rows[i].begin, deg = degf & kDegMask;
    const double fdeg = static_cast<double>(deg);
    uint32_t ns = 0, nl = 0;
    double prev = 0.0;
    for (uint32_t j = 0; j < deg; ++j) {
        const double c = e.cdf[b + j];
        const double q = __dmul_rn(__dsub_rn(c, prev), fdeg);
        prev = c;
        al[b + j].prob = q;
        al[b + j].alias = j;
        if (q < 1.0) scratch[b + ns++] = j;
        else scratch[b + deg - 1u - nl++] = j;
    }
    while (ns > 0u && nl > 0u) {
        const uint32_t sm = scratch[b + --ns];
        const uint32_t lg = scratch[b + deg - nl];  // top of the large stack
        al[b + sm].alias = lg;                       // prob[sm] stays q_sm
        const double ql = __dsub_rn(__dadd_rn(al[b + lg].prob, al[b + sm].prob), 1.0);
        al[b + lg].prob = ql;
        if (ql < 1.0) {
            --nl;
            scratch[b + ns++] = lg;
        }
    }
    while (nl > 0u) al[b + scratch[b + deg - nl--]].prob = 1.0;
    while (ns > 0u) al[b + scratch[b + --ns]].prob = 1.0;
    for (uint32_t j = 0; j < deg; ++j) {  // slot indices -> target words
        AliasRec r = al[b + j];
        r.self = e.tgt[b + j];
        r.alias = r.prob < 1.0 ? e.tgt[b + r.alias] : r.self;
        al[b + j] = r;
    }
}

__global__ void k_build_erec(uint64_t m, const RowRec* __restrict__ rows, const uint32_t* __restrict__ tgt,
                             EdgeRec* __restrict__ erec) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t t = tgt[i];
    const RowRec r = rows[t & kTargetMask];
    EdgeRec e;
    e.tgt = t;
    e.begin = r.begin;
    e.deg = r.deg;
    e.pad = 0u;
    e.rate = r.rate;
    e.d = r.d;
    erec[i] = e;
}

__global__ void k_export_alias(uint64_t m, const AliasRec* __restrict__ al, double* prob, int64_t* self,
                               int64_t* alias_target) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const AliasRec r = al[i];
    prob[i] = r.prob;
    // target | sign as a signed word: -(target + 1) for a negative entry
    self[i] = (r.self & kSignBit) ? -static_cast<int64_t>(r.self & kTargetMask) - 1 : static_cast<int64_t>(r.self);
    alias_target[i] =
        (r.alias & kSignBit) ? -static_cast<int64_t>(r.alias & kTargetMask) - 1 : static_cast<int64_t>(r.alias);
}

// d_max / d_sum: fixed two-level tree (block partials, then one block) -> deterministic.
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 1024;

__global__ void k_dstats_partial(const RowRec* __restrict__ rows, int64_t n, double* part) {
    __shared__ double smax[kRedThreads], ssum[kRedThreads];
    double m = -INFINITY, s = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kRedThreads) {
        const double d = rows[i].d;
        m = fmax(m, d);
        s = __dadd_rn(s, d);
    }
    smax[threadIdx.x] = m;
    ssum[threadIdx.x] = s;
    __syncthreads();
    for (int o = kRedThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
            ssum[threadIdx.x] = __dadd_rn(ssum[threadIdx.x], ssum[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = smax[0];
        part[2 * blockIdx.x + 1] = ssum[0];
    }
}

__global__ void k_dstats_final(const double* part, int nb, double* out2) {
    __shared__ double smax[kRedThreads], ssum[kRedThreads];
    double m = -INFINITY, s = 0.0;
    for (int i = threadIdx.x; i < nb; i += kRedThreads) {
        m = fmax(m, part[2 * i]);
        s = __dadd_rn(s, part[2 * i + 1]);
    }
    smax[threadIdx.x] = m;
    ssum[threadIdx.x] = s;
    __syncthreads();
    for (int o = kRedThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
            ssum[threadIdx.x] = __dadd_rn(ssum[threadIdx.x], ssum[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out2[0] = smax[0];
        out2[1] = ssum[0];
    }
}

// Random 32-B sector gather: the roofline denominator for the sampler's table reads.  Every
// load is independent (hash-generated sector index), so the kernel measures the memory
// system's random-sector throughput, not latency.
__global__ void __launch_bounds__(256) k_gather(const uint4* __restrict__ buf, uint64_t nsectors, int loads,
                                                uint64_t salt, unsigned* __restrict__ sink) {
    uint64_t x = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull ^ salt;
    unsigned acc = 0;
#pragma unroll 8
    for (int i = 0; i < loads; ++i) {
        x ^= x >> 33;
        x *= 0xFF51AFD7ED558CCDull;
        x ^= x >> 29;
        const uint64_t s = __umul64hi(x, nsectors);
        const uint4 a = __ldcg(buf + 2 * s);
        const uint4 b = __ldcg(buf + 2 * s + 1);
        acc += a.x ^ a.w ^ b.y ^ b.z;
    }
    if (acc == 0x12345678u) sink[0] = acc;  // keep the loads alive
}

// Self-test of the device math against the toolkit: dexp vs exp (bitwise), fast_log vs log.
__global__ void k_math_check(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[2 * i] = dexp(x[i]);
    out[2 * i + 1] = exp(x[i]);
}

inline unsigned grid_for(int64_t n, int threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

}  // namespace

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Status(EXPMC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int sampler_threads() { return kThreads; }

int sampler_blocks_per_sm(int mode) {
    int b = 0;
    if (mode == kSamplerFem)
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample<FemPolicy, false>, kThreads, 0), "occupancy");
    else if (mode == EXPMC_SAMPLER_EVENT)
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample_grouped<EdPolicyG>, kThreads, 0),
                   "occupancy");
    else
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample<RefPolicy<false>, false>, kThreads, 0),
                   "occupancy");
    return b > 0 ? b : 1;
}

// Entry and forward mode are separate instantiations: a batch is one lane, and the entry-mode
// kernel (the hot path) carries no trace of the forward start draw.
template <bool W>
void launch_sampler_t(const SamplerArgs& a, int grid, int mode, uint32_t lane, cudaStream_t s, bool level0) {
    if constexpr (!W) {
        if (lane == EXPMC_LANE_FEM) {
            k_sample<FemPolicy, false><<<grid, kThreads, 0, s>>>(a);
            cuda_check(cudaGetLastError(), "k_sample launch");
            return;
        }
    }
    if (mode == EXPMC_SAMPLER_EVENT) {
        if (lane == EXPMC_LANE_FORWARD) k_sample<EdPolicy<true>, W><<<grid, kThreads, 0, s>>>(a);
        else if constexpr (W) k_sample<EdPolicy<false>, W><<<grid, kThreads, 0, s>>>(a);
        else k_sample_grouped<EdPolicyG><<<grid, kThreads, 0, s>>>(a);
    } else {
        if (lane == EXPMC_LANE_FORWARD) k_sample<RefPolicy<true>, W><<<grid, kThreads, 0, s>>>(a);
        else if (!W && level0) k_sample<RefPolicy0, false><<<grid, kThreads, 0, s>>>(a);
        else k_sample<RefPolicy<false>, W><<<grid, kThreads, 0, s>>>(a);
    }
    cuda_check(cudaGetLastError(), "k_sample launch");
}

void launch_sampler(const SamplerArgs& a, int grid, int mode, uint32_t lane, cudaStream_t s, bool level0) {
    launch_sampler_t<false>(a, grid, mode, lane, s, level0);
}

void launch_sampler_welford(const SamplerArgs& a, int grid, int mode, uint32_t lane, cudaStream_t s) {
    if (lane == EXPMC_LANE_FEM) throw Status(EXPMC_ENOTIMPL, "classical MC has no fem lane");
    launch_sampler_t<true>(a, grid, mode, lane, s, false);
}

void launch_combine_welford(const uint64_t* chunk0, const DevItem* items, uint32_t nitems, uint64_t g_begin,
                            uint64_t g_end, const ChunkPartials& partials, Partial* totals, cudaStream_t s) {
    k_combine_welford<<<grid_for(nitems, kCombWarps), kCombWarps * 32, 0, s>>>(chunk0, items, nitems, g_begin, g_end,
                                                                               partials, totals);
    cuda_check(cudaGetLastError(), "k_combine_welford launch");
}

void launch_combine(const uint64_t* chunk0, uint32_t nitems, uint64_t g_begin, uint64_t g_end,
                    const ChunkPartials& partials, bool with_extra, bool ordered, Partial* totals, cudaStream_t s) {
    k_combine<<<grid_for(nitems, kCombWarps), kCombWarps * 32, 0, s>>>(chunk0, nitems, g_begin, g_end, partials,
                                                                       with_extra, ordered, totals);
    cuda_check(cudaGetLastError(), "k_combine launch");
}

void launch_debug(const RowRec* rows, EdgeTables edges, const DevItem* items, uint32_t n, const LaneData& init,
                  SampleOut* out, int mode, uint32_t lane, uint32_t flags, cudaStream_t s) {
    const int g = grid_for(n, 128);
    if (lane == EXPMC_LANE_FEM) {
        k_debug<FemPolicy><<<g, 128, 0, s>>>(rows, edges, items, n, init, flags, out);
    } else if (mode == EXPMC_SAMPLER_EVENT) {
        if (lane == EXPMC_LANE_FORWARD) k_debug<EdPolicy<true>><<<g, 128, 0, s>>>(rows, edges, items, n, init, flags, out);
        else k_debug<EdPolicy<false>><<<g, 128, 0, s>>>(rows, edges, items, n, init, flags, out);
    } else {
        if (lane == EXPMC_LANE_FORWARD) k_debug<RefPolicy<true>><<<g, 128, 0, s>>>(rows, edges, items, n, init, flags, out);
        else k_debug<RefPolicy<false>><<<g, 128, 0, s>>>(rows, edges, items, n, init, flags, out);
    }
    cuda_check(cudaGetLastError(), "k_debug launch");
}

void launch_count_edges(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val, uint64_t* deg,
                        unsigned int* err, uint32_t* heavy, unsigned int* nheavy, int num_sms, cudaStream_t s) {
    if (n == 0) return;
    k_count_edges<<<grid_for(n, 256), 256, 0, s>>>(n, row_ptr, col, val, deg, err, heavy, nheavy);
    cuda_check(cudaGetLastError(), "k_count_edges launch");
    k_count_heavy<<<num_sms * 4, 256, 0, s>>>(n, row_ptr, col, val, deg, err, heavy, nheavy);
    cuda_check(cudaGetLastError(), "k_count_heavy launch");
}

void launch_fill_tables(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val, const double* u,
                        const uint64_t* begin, RowRec* rows, double* cdf, uint32_t* tgt, const uint32_t* heavy,
                        const unsigned int* nheavy, int num_sms, cudaStream_t s) {
    if (n == 0) return;
    k_fill_tables<<<grid_for(n, 128), 128, 0, s>>>(n, row_ptr, col, val, u, begin, rows, cdf, tgt);
    cuda_check(cudaGetLastError(), "k_fill_tables launch");
    k_fill_heavy<<<num_sms * 8, kFillWarps * 32, 0, s>>>(row_ptr, col, val, u, begin, rows, cdf, tgt, heavy, nheavy);
    cuda_check(cudaGetLastError(), "k_fill_heavy launch");
}

void launch_set_vector(int64_t n, const double* u, RowRec* rows, cudaStream_t s) {
    if (n == 0) return;
    k_set_vector<<<grid_for(n, 256), 256, 0, s>>>(n, u, rows);
    cuda_check(cudaGetLastError(), "k_set_vector launch");
}

void launch_export(int64_t n, const RowRec* rows, double* d, double* rate, int64_t* row_ptr, cudaStream_t s) {
    if (n == 0) return;
    k_export_rows<<<grid_for(n, 256), 256, 0, s>>>(n, rows, d, rate, row_ptr);
    cuda_check(cudaGetLastError(), "k_export_rows launch");
}

void launch_export_edges(uint64_t m, EdgeTables edges, double* cdf, int64_t* target, uint8_t* sign,
                         cudaStream_t s) {
    if (m == 0) return;
    k_export_edges<<<grid_for(static_cast<int64_t>(m), 256), 256, 0, s>>>(m, edges, cdf, target, sign);
    cuda_check(cudaGetLastError(), "k_export_edges launch");
}

void launch_count_nonuniform(int64_t n, const RowRec* rows, unsigned long long* count, cudaStream_t s) {
    cuda_check(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s), "memset count");
    if (n == 0) return;
    k_count_nonuniform<<<std::min<int64_t>(grid_for(n, 256), 4096), 256, 0, s>>>(n, rows, count);
    cuda_check(cudaGetLastError(), "k_count_nonuniform launch");
}

void launch_build_alias(int64_t n, const RowRec* rows, EdgeTables edges, AliasRec* alias, uint32_t* scratch,
                        cudaStream_t s) {
    if (n == 0) return;
    k_build_alias<<<grid_for(n, 128), 128, 0, s>>>(n, rows, edges, alias, scratch);
    cuda_check(cudaGetLastError(), "k_build_alias launch");
}

void launch_build_erec(uint64_t m, const RowRec* rows, const uint32_t* tgt, EdgeRec* erec, cudaStream_t s) {
    if (m == 0) return;
    k_build_erec<<<grid_for(static_cast<int64_t>(m), 256), 256, 0, s>>>(m, rows, tgt, erec);
    cuda_check(cudaGetLastError(), "k_build_erec launch");
}

void launch_export_alias(uint64_t m, const AliasRec* alias, double* prob, int64_t* self, int64_t* alias_target,
                         cudaStream_t s) {
    if (m == 0) return;
    k_export_alias<<<grid_for(static_cast<int64_t>(m), 256), 256, 0, s>>>(m, alias, prob, self, alias_target);
    cuda_check(cudaGetLastError(), "k_export_alias launch");
}

float bench_gather(uint64_t bytes, int loads_per_thread, int reps, int num_sms, uint64_t* total_loads) {
    const uint64_t nsectors = bytes / 32;
    uint4* buf = nullptr;
    unsigned* sink = nullptr;
    cuda_check(cudaMalloc(&buf, nsectors * 32), "cudaMalloc gather");
    cuda_check(cudaMalloc(&sink, sizeof(unsigned)), "cudaMalloc sink");
    cuda_check(cudaMemset(buf, 1, nsectors * 32), "memset gather");
    const int grid = num_sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {  // first launch is warm-up
        cudaEventRecord(e0);
        k_gather<<<grid, 256>>>(buf, nsectors, loads_per_thread, 0x1234567ull + r, sink);
        cudaEventRecord(e1);
        cuda_check(cudaEventSynchronize(e1), "gather");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(sink);
    *total_loads = static_cast<uint64_t>(grid) * 256 * static_cast<uint64_t>(loads_per_thread);
    return best;
}

void math_check(const double* x, int64_t n, double* out, cudaStream_t s) {
    if (n == 0) return;
    k_math_check<<<grid_for(n, 256), 256, 0, s>>>(x, n, out);
    cuda_check(cudaGetLastError(), "k_math_check launch");
}

size_t scan_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cuda_check(cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const uint64_t*>(nullptr),
                                             static_cast<uint64_t*>(nullptr), static_cast<int>(n)),
               "scan sizing");
    return bytes;
}

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, void* tmp, size_t tmp_bytes, cudaStream_t s) {
    cuda_check(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, static_cast<int>(n), s), "scan");
}

size_t dstat_temp_bytes(int64_t) { return sizeof(double) * 2 * kRedBlocks; }

void d_stats(const RowRec* rows, int64_t n, double* out2, void* tmp, size_t, cudaStream_t s) {
    double* part = static_cast<double*>(tmp);
    k_dstats_partial<<<kRedBlocks, kRedThreads, 0, s>>>(rows, n, part);
    cuda_check(cudaGetLastError(), "k_dstats_partial launch");
    k_dstats_final<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, out2);
    cuda_check(cudaGetLastError(), "k_dstats_final launch");
}

}  // namespace expmc_b200
