// Event-driven walker: the statistically equivalent fast sampler.
//
// The reference redraws a fresh holding time at every fine-step boundary (paths.cpp:95-96):
// one uniform per step even when nothing happens, 2^l of them per path.  The CTMC is
// memoryless, so the same law follows from one exponential clock per jump: hold in state s
// for E/rate(s), jump, repeat until the clock passes beta.  The fine-step boundaries
// k*dt (k = 0..N, N = 2^l) that fall inside a holding interval all see state s, so their
// Strang weights are added in closed form:
//   single  (paths.cpp:110):      expo  = dt * sum_k w_k d(s_k),  w = 1/2 at k = 0, N, else 1
//   coupled (paths.cpp:134-136):  coarse = dt * sum_k c_k d(s_k), c = 2 at interior even k,
//                                                                 1 at k = 0, N, 0 at odd k
//                                 delta  = dt * sum_k e_k d(s_k), e = +1 odd, -1 interior even,
//                                                                 -1/2 at k = 0, N
// (doubled integer weights below keep the per-segment sums exact).  A path now costs
// O(jumps) instead of O(2^l) events; the random numbers differ from the reference's, so
// parity is statistical (tests/test_gpu_ed.py).  The cost counter is the reference's model
// for the path this walker drew -- draws = jumps + #{k in 1..N : rate(s_k) > 0} (each
// non-absorbing step ends with one rejected draw, paths.cpp:50-53), cost = draws + N -- so the
// driver's allocation (mlmc.cpp:216) sees the same unit costs in expectation.
//
// Closed-form first hold (entry mode): every sample of an item starts in the same row with
// the same clock, so whether its first holding interval outlasts [0, beta] is decided by the
// first draw alone: E = -log(1 - u) >= rate * beta, i.e. M = 2^53 - K <= 2^53 e^{-rate beta}.
// EdPolicy::prepare computes, once per chunk, a threshold m_safe a relative 2^-30 inside that
// boundary (far outside the ~4 ulp error of the log / divide the full event evaluates) and the
// values of the stay-at-entry path with the same ed_segment / ed_finish code.  A draw with
// M < m_safe then ends the sample at once with those values -- the same outcome the full
// event computes, without its log, divide, segment sums and exp.  On C3/C4 (t = 1/lambda)
// over 95 % of samples never jump.  Draws near the boundary and every later event take the
// full path.  EXPMC_SAMPLER_FLAG_FULL_HOLD switches the shortcut off (A/B tests).
//
// Geometric screening (entry mode, chunk kernel k_sample_grouped): testing every sample's
// first draw costs a Philox block per sample, and on C3/C4 95 % of them only learn that the
// sample stays at the entry.  Whether a sample is held is a Bernoulli(p) event with
// p = P(M < m_safe) = (m_safe - 1) 2^-53, independent across samples, so the chunk's jumpers
// are located directly: the gaps between consecutive jumpers are Geometric(1 - p),
// G = floor(log(U) / log(p)), drawn 32 at a time from a per-chunk Philox stream (lane
// kSkipLane of the item's key, counter = chunk index) and placed by a warp prefix sum.  A
// listed jumper's first draw must then follow the law of M given M >= m_safe: its own stream's
// first word is mapped onto [m_safe, 2^53] (kCond, ed_event).  Same path law, one Philox block
// per 32 gaps instead of per sample.  Used when p > kSkipMinHeld; EXPMC_SAMPLER_FLAG_SCREEN_EACH
// restores the per-sample screen (A/B tests).
#pragma once

#ifndef EXPMC_SAMPLER_MINB
#define EXPMC_SAMPLER_MINB 4  // resident 256-thread blocks per SM the sampler is register-budgeted for
#endif

#include "walker.cuh"

namespace expmc_b200 {

constexpr uint32_t kFresh = 2u;
constexpr uint32_t kCond = 4u;        // first draw conditioned on leaving the entry (geometric screen)
constexpr uint32_t kSkipLane = 5u;    // Philox lane of the per-chunk gap stream (0-3, 6, 7 are taken)
constexpr double kSkipMinHeld = 0.75; // geometric screening when P(held) exceeds this
constexpr uint32_t kFlagGrouped = 1u << 31;  // prepare() called by k_sample_grouped (internal flag bit)

template <class ST>
struct EdWalkerT {
    ST st;
    Row cur;
    uint32_t state;
    int32_t sign;
    uint32_t dconst;   // bit 0: every visited state has the entry's d (=> coupled difference is 0)
                       // bit 1 (kFresh): no event yet (the closed-form first hold applies)
    uint64_t kcur;     // first fine-step boundary not yet assigned a state
    double t;          // start time of the current holding interval
    double acc_a;      // doubled-weight sum of d: expo (single) or coarse (coupled)
    double acc_b;      // doubled-weight sum of d: delta (coupled)
    double dfirst;
};
using EdWalker = EdWalkerT<Stream>;
// k_sample_grouped's walker: the Philox key schedule comes from the warp's round-key table
// (ItemConst::rk, one item per warp at a time), so the stream holds no key registers.  An
// entry-mode event consumes the stream as E_1 v_1 E_2 v_2 ... E_k (a jump draws the holding time
// and the neighbour; the last holding time ends the path), so block b holds exactly event b + 1's
// two words: one Philox block per event and no word queue (StreamEv) -- the same words in the
// same order as the queued stream (EXPMC_EDEV=0), results bitwise equal.
// EXPMC_ED_PREFETCH: a jump prefetches the landing row's u (A/B builds).
#ifndef EXPMC_ED_PREFETCH
#define EXPMC_ED_PREFETCH 0
#endif
#ifndef EXPMC_EDEV
#define EXPMC_EDEV 1
#endif
#if EXPMC_EDEV
using EdWalkerRK = EdWalkerT<StreamEv>;
#else
using EdWalkerRK = EdWalkerT<StreamRK>;
#endif

__device__ __forceinline__ void ed_stream_init(Stream& st, const ItemConst& ic, uint64_t sample) {
    stream_init(st, ic.seed, sample, ic.key3);
}
__device__ __forceinline__ void ed_stream_init(StreamRK& st, const ItemConst& ic, uint64_t sample) {
    stream_init(st, sample, ic.key3);
}
__device__ __forceinline__ void ed_stream_init(StreamEv& st, const ItemConst& ic, uint64_t sample) {
    stream_init(st, sample, ic.key3);
}

template <bool F, class WK>
__device__ __forceinline__ void ed_start(WK& w, const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows,
                                         uint64_t sample) {
    ed_stream_init(w.st, ic, sample);
    const uint32_t s0 = draw_start<F>(w.st, ic, fi);
    w.cur = F ? load_row(rows, s0) : ic.r0;  // entry mode: the item's row (EdPolicy::prepare)
    w.state = s0;
    w.sign = 1;
    // a sample listed by the geometric screen (k_sample_grouped) draws its first hold
    // conditioned on leaving the entry; otherwise the closed-form first-hold test applies
    w.dconst = 1u | (ic.skip_scale != 0.0 ? kCond : kFresh);
    w.kcur = 0;
    w.t = 0.0;
    w.acc_a = 0.0;
    w.acc_b = 0.0;
    w.dfirst = w.cur.d;
}

// Boundaries [ka, kb] (ka <= kb <= N) all see the current state.
template <class WK>
__device__ __forceinline__ void ed_segment(WK& w, const ItemConst& ic, uint64_t ka, uint64_t kb,
                                           unsigned long long& draws) {
    const uint64_t n = kb - ka + 1;
    const int64_t ends = static_cast<int64_t>(ka == 0) + static_cast<int64_t>(kb == ic.nsteps);
    if (w.cur.rate != 0.0) draws += n - (ka == 0 ? 1u : 0u);  // one rejected draw per non-absorbing step end
    const double d = w.cur.d;
    if (ic.base) {
        const int64_t w2 = 2 * static_cast<int64_t>(n) - ends;
        w.acc_a = __dadd_rn(w.acc_a, __dmul_rn(d, static_cast<double>(w2)));
    } else {
        const int64_t ev = static_cast<int64_t>(kb >> 1) - static_cast<int64_t>((ka + 1) >> 1) + 1;
        const int64_t od = static_cast<int64_t>(n) - ev;
        const int64_t c2 = 4 * ev - 2 * ends;
        const int64_t e2 = 2 * od - 2 * ev + ends;
        w.acc_a = __dadd_rn(w.acc_a, __dmul_rn(d, static_cast<double>(c2)));
        w.acc_b = __dadd_rn(w.acc_b, __dmul_rn(d, static_cast<double>(e2)));
    }
}

// One holding interval: draw its length, assign the boundaries it covers, jump (or finish).
template <class WK>
__device__ __forceinline__ bool ed_event(WK& w, const ItemConst& ic, const RowRec* __restrict__ rows,
                                         const EdgeTables& edges, const LogEntry* s_log, unsigned long long& draws,
                                         unsigned long long& jumps) {
    stream_reserve2(w.st, ic.rk);
    if (w.dconst & (kFresh | kCond)) {
        if (w.dconst & kCond) {
            // listed by the geometric screen: M uniform on [m_safe, 2^53] from the first word
            const uint64_t range = (uint64_t{1} << 53) - ic.m_safe + 1u;
            const uint64_t m = ic.m_safe + __umul64hi(w.st.w0, range);
            w.st.w0 = ((uint64_t{1} << 53) - m) << 11;  // K = 2^53 - M
        } else if ((uint64_t{1} << 53) - (w.st.w0 >> 11) < ic.m_safe) {  // holds past beta at the entry
            w.dconst &= ~kFresh;
            draws += ic.nsteps;  // ed_segment(0, N) on a non-absorbing row
            w.sign = 0;          // marks the closed-form path for ed_sample / record
            return true;
        }
        w.dconst &= ~(kFresh | kCond);
    }
    double tjump = INFINITY;
    if (w.cur.rate != 0.0) {
        const double e = -fast_log(__ull2double_rn((uint64_t{1} << 53) - stream_pop_bits(w.st)), -53, s_log, c_log_poly);
        tjump = __dadd_rn(w.t, fast_div(e, w.cur.rate));
    }
    if (!(tjump < ic.tend)) {  // holds to the end of the interval [0, beta]
        if (w.kcur <= ic.nsteps) ed_segment(w, ic, w.kcur, ic.nsteps, draws);
        return true;
    }
    // boundaries k with k*dt < tjump: k <= ceil(tjump/dt) - 1
    const double q = __dmul_rn(tjump, ic.inv_dt);
    const uint64_t kq = static_cast<uint64_t>(ceil(q));
    const uint64_t kend = kq == 0 ? 0 : kq - 1;  // kq >= 1 unless tjump == 0
    if (kq >= 1 && kend >= w.kcur) {
        ed_segment(w, ic, w.kcur, kend, draws);
        w.kcur = kend + 1;
    }
    w.t = tjump;
    ++jumps;
    ++draws;  // the accepted holding-time draw of the jump (paths.cpp:51-54)
    const uint64_t kv = stream_pop_bits(w.st);
    uint32_t ts;
    if (edges.erec != nullptr && !alias_row(edges, w.cur.deg)) {
        // one 32-B sector: the edge's target word and the target row's payload (EdgeRec)
        const EdgeRec* p = edges.erec + static_cast<uint32_t>(w.cur.begin + pick_slot(edges, w.cur.begin, w.cur.deg, kv));
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
        const double2 rd = __ldg(reinterpret_cast<const double2*>(p) + 1);
        ts = q.x;
        w.cur.d = rd.y;
        w.cur.rate = rd.x;
        w.cur.begin = q.y;
        w.cur.deg = q.z;
    } else {
        ts = pick_edge<true>(edges, w.cur.begin, w.cur.deg, kv);
        w.cur = load_row(rows, ts & kTargetMask);
    }
    if (ts & kSignBit) w.sign = -w.sign;
    w.state = ts & kTargetMask;
#if EXPMC_ED_PREFETCH
    // most jumping paths end within a jump or two: start u[state]'s sector on its way now, the
    // path's end reads it (ed_finish) one event later at the earliest
    asm volatile("prefetch.global.L2 [%0];" ::"l"(&rows[w.state].u));
#endif
    if (w.cur.d != w.dfirst) w.dconst = 0u;
    return false;
}

template <bool F, class WK>
__device__ __forceinline__ void ed_finish(const WK& w, const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows,
                                          double& fine, double& coarse) {
    const double sg = static_cast<double>(w.sign);
    const double u_end = terminal_factor<F>(ic, fi, rows, w.state);
    const double h = __dmul_rn(0.5, ic.dt);
    if (ic.base) {
        const double expo = __dmul_rn(h, w.acc_a);
        fine = __dmul_rn(__dmul_rn(sg, expo == 0.0 ? 1.0 : dexp(expo)), u_end);
        coarse = 0.0;
    } else {
        const double uf = __dmul_rn(sg, u_end);
        const double c = __dmul_rn(h, w.acc_a);
        const double ec = c == 0.0 ? 1.0 : dexp(c);
        coarse = __dmul_rn(uf, ec);
        fine = w.dconst ? coarse : __dmul_rn(uf, dexp(__dadd_rn(c, __dmul_rn(h, w.acc_b))));
    }
}

template <bool F, class WK>
__device__ __forceinline__ double ed_sample(const WK& w, const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows) {
    if (w.sign == 0) return ic.hold_x;
    if (!ic.base && w.dconst) return 0.0;
    double fine, coarse;
    ed_finish<F>(w, ic, fi, rows, fine, coarse);
    return ic.base ? fine : __dsub_rn(fine, coarse);
}

// ---- policies the chunk kernel is templated on (F: forward mode, lane 1)
// sample() returns the run_level sample x; kExtra policies also produce the SumAcc side
// channel (fem).  record() fills the per-sample debug output.
template <bool F>
struct RefPolicy {
    using W = Walker;
    static constexpr bool kExtra = false;
    static constexpr bool kScreen = false;
    static __device__ __forceinline__ bool screen(const ItemConst&, uint64_t) { return false; }
    static constexpr int kMinBlocks = EXPMC_SAMPLER_MINB;
    static __device__ __forceinline__ void prepare(ItemConst& ic, const RowRec* rows, const LaneData&, uint32_t flags) {
        prepare_hold(ic, rows, flags);
    }
    static __device__ __forceinline__ void start(W& w, const ItemConst& ic, const LaneData& ld, const RowRec* rows,
                                                 uint64_t s) {
        walker_start<F>(w, ic, ld, rows, s);
    }
    static __device__ __forceinline__ bool event(W& w, const ItemConst& ic, const LaneData&, const RowRec* rows,
                                                 const EdgeTables& e, const LogEntry* lg, unsigned long long& dr,
                                                 unsigned long long& j) {
        return walker_event(w, ic, rows, e, lg, dr, j);
    }
    static __device__ __forceinline__ double sample(const W& w, const ItemConst& ic, const LaneData& ld,
                                                    const RowRec* rows, double&) {
        return walker_sample<F>(w, ic, ld, rows);
    }
    static constexpr bool kDefer = true;  // sample() split into end_record() + value()
    static __device__ __forceinline__ void end_record(const W& w, const ItemConst& ic, double& a, double& b,
                                                      uint32_t& se) {
        walker_end_record(w, ic, a, b, se);
    }
    static __device__ __forceinline__ double value(double a, double b, uint32_t se, const ItemConst& ic,
                                                   const LaneData& ld, const RowRec* rows) {
        return walker_value<F>(a, b, se, ic, ld, rows);
    }
    static __device__ __forceinline__ void record(const W& w, const ItemConst& ic, const LaneData& ld,
                                                  const RowRec* rows, SampleOut& o) {
        walker_finish<F>(w, ic, ld, rows, o.fine, o.coarse);
        o.value = ic.base ? o.fine : __dsub_rn(o.fine, o.coarse);
        o.integ_f = o.integ_c = 0.0;
        o.end_state = w.state;
    }
};

// Level-0 items of the entry lane (base level, nsteps == 1): the reference-order walker
// without step bookkeeping (Walker0).  A batch's level-0 items are launched with this policy,
// the rest with RefPolicy (context.cu: sample_launch).
#ifndef EXPMC_B0_MINB
#define EXPMC_B0_MINB EXPMC_SAMPLER_MINB
#endif
struct RefPolicy0 {
    using W = Walker0;
    static constexpr bool kDefer = false;
    static constexpr bool kExtra = false;
    static constexpr bool kScreen = false;
    static __device__ __forceinline__ bool screen(const ItemConst&, uint64_t) { return false; }
    static constexpr int kMinBlocks = EXPMC_B0_MINB;
    static __device__ __forceinline__ void prepare(ItemConst& ic, const RowRec* rows, const LaneData&, uint32_t flags) {
        prepare_hold(ic, rows, flags);
#if EXPMC_RKEYS
        set_round_keys(ic.rk, ic.seed);  // lane 0; k_sample's __syncwarp publishes it with the item constants
#endif
    }
    static __device__ __forceinline__ void start(W& w, const ItemConst& ic, const LaneData&, const RowRec*, uint64_t s) {
        walker0_start(w, ic, s);
    }
    static __device__ __forceinline__ bool event(W& w, const ItemConst& ic, const LaneData&, const RowRec* rows,
                                                 const EdgeTables& e, const LogEntry* lg, unsigned long long& dr,
                                                 unsigned long long& j) {
#if EXPMC_L0TUNE
        return walker0_event(w, ic, rows, e, lg, dr, j);  // the step's end is the sample's end
#else
        return walker_hold(w, rows, e, lg, dr, j, ic.rk);
#endif
    }
    static __device__ __forceinline__ double sample(const W& w, const ItemConst& ic, const LaneData&,
                                                    const RowRec* rows, double&) {
        return walker0_sample(w, ic, rows);
    }
};

template <bool F>
struct EdPolicy {
    using W = EdWalker;
    static constexpr bool kDefer = false;
    static constexpr bool kExtra = false;
    static constexpr bool kScreen = !F;  // entry mode: all samples start in ic.entry
    // The first event's closed-form test alone: block 0 of the sample's stream, first word.
    static __device__ __forceinline__ bool screen(const ItemConst& ic, uint64_t sample) {
        uint32_t c0 = 0, c1 = static_cast<uint32_t>(sample), c2 = static_cast<uint32_t>(sample >> 32), c3 = ic.key3;
        philox10(c0, c1, c2, c3, static_cast<uint32_t>(ic.seed), static_cast<uint32_t>(ic.seed >> 32));
        const uint64_t k53 = ((static_cast<uint64_t>(c2) << 32) | c3) >> 11;  // rng.hpp:32-35
        return (uint64_t{1} << 53) - k53 < ic.m_safe;
    }
    static constexpr int kMinBlocks = EXPMC_SAMPLER_MINB;
    // The closed-form first hold (header): threshold and stay-at-entry values, once per chunk.
    static __device__ __forceinline__ void prepare(ItemConst& ic, const RowRec* rows, const LaneData& ld,
                                                   uint32_t flags) {
        ic.skip_scale = 0.0;
        if (F) return;
        const Row r = load_row(rows, ic.entry);
        ic.r0 = r;
        if (flags & EXPMC_SAMPLER_FLAG_FULL_HOLD) return;
        if (!(r.rate > 0.0)) return;  // absorbing entry: the full event draws nothing anyway
        // P(no jump before beta) = e^{-rate beta}; M below 2^53 of that, less 2^-30 relative
        const double m = __dmul_rn(__dmul_rn(dexp(-__dmul_rn(r.rate, ic.tend)), 0x1.0p53), 1.0 - 0x1.0p-30);
        if (!(m >= 2.0)) return;
        EdWalker w;
        w.cur = r;
        w.state = ic.entry;
        w.sign = 1;
        w.dconst = 1u;
        w.t = 0.0;
        w.acc_a = 0.0;
        w.acc_b = 0.0;
        w.dfirst = r.d;
        unsigned long long draws = 0;
        ed_segment(w, ic, 0, ic.nsteps, draws);  // the holding interval covers every boundary
        ed_finish<false>(w, ic, ld, rows, ic.hold_fine, ic.hold_coarse);
        ic.hold_x = ic.base ? ic.hold_fine : 0.0;  // ed_sample's coupled constant-d case
        ic.m_safe = static_cast<uint64_t>(m);
        // P(held) = #{M in 1..2^53 : M < m_safe} / 2^53, exact in fp64 (m_safe < 2^53)
        const double p_held = __dmul_rn(static_cast<double>(ic.m_safe - 1u), 0x1.0p-53);
        if ((flags & kFlagGrouped) && !(flags & EXPMC_SAMPLER_FLAG_SCREEN_EACH) && p_held > kSkipMinHeld)
            ic.skip_scale = 1.0 / log(p_held);
    }
    static __device__ __forceinline__ void start(W& w, const ItemConst& ic, const LaneData& ld, const RowRec* rows,
                                                 uint64_t s) {
        ed_start<F>(w, ic, ld, rows, s);
    }
    static __device__ __forceinline__ bool event(W& w, const ItemConst& ic, const LaneData&, const RowRec* rows,
                                                 const EdgeTables& e, const LogEntry* lg, unsigned long long& dr,
                                                 unsigned long long& j) {
        return ed_event(w, ic, rows, e, lg, dr, j);
    }
    static __device__ __forceinline__ double sample(const W& w, const ItemConst& ic, const LaneData& ld,
                                                    const RowRec* rows, double&) {
        return ed_sample<F>(w, ic, ld, rows);
    }
    static __device__ __forceinline__ void record(const W& w, const ItemConst& ic, const LaneData& ld,
                                                  const RowRec* rows, SampleOut& o) {
        if (w.sign == 0) {
            o.fine = ic.hold_fine;
            o.coarse = ic.hold_coarse;
            o.value = ic.hold_x;
        } else {
            ed_finish<F>(w, ic, ld, rows, o.fine, o.coarse);
            o.value = ic.base ? o.fine : __dsub_rn(o.fine, o.coarse);
        }
        o.integ_f = o.integ_c = 0.0;
        o.end_state = w.state;
    }
};

// The grouped kernel's entry-mode policy: EdPolicy<false> with the keyless stream (the round-key
// table is written by prepare(), lane 0, and published by the kernel's __syncwarp).
struct EdPolicyG : EdPolicy<false> {
    using W = EdWalkerRK;
    static __device__ __forceinline__ void prepare(ItemConst& ic, const RowRec* rows, const LaneData& ld, uint32_t flags) {
        EdPolicy<false>::prepare(ic, rows, ld, flags);
        set_round_keys(ic.rk, ic.seed);
    }
    static __device__ __forceinline__ void start(W& w, const ItemConst& ic, const LaneData& ld, const RowRec* rows,
                                                 uint64_t s) {
        ed_start<false>(w, ic, ld, rows, s);
    }
    static __device__ __forceinline__ bool event(W& w, const ItemConst& ic, const LaneData&, const RowRec* rows,
                                                 const EdgeTables& e, const LogEntry* lg, unsigned long long& dr,
                                                 unsigned long long& j) {
        return ed_event(w, ic, rows, e, lg, dr, j);
    }
    static __device__ __forceinline__ double sample(const W& w, const ItemConst& ic, const LaneData& ld,
                                                    const RowRec* rows, double&) {
        return ed_sample<false>(w, ic, ld, rows);
    }
};

}  // namespace expmc_b200
