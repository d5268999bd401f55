// Device-side path machinery: Philox4x32-10 streams and the reference-order CTMC walker.
//
// Reference-order means draw-for-draw identical to the reference's CPU sampler:
//   RngStream (rng.hpp:21-73), evolve_common (paths.cpp:44-71), LevelSampler::single /
//   ::coupled (paths.cpp:99-141), LevelSampler ctor thresholds (paths.cpp:84-91).
// Every floating-point expression that can round differently under FMA contraction is
// written with explicit __d*_rn intrinsics in the reference's evaluation order; the only
// remaining sources of difference are CUDA's exp vs glibc (< 1 ulp) and holding tests whose
// draw lies within a few ulps of the threshold (the probability-space test below).
//
// SIMT shape: a warp advances 32 independent paths one EVENT per loop trip (one pass of
// evolve_common's for(;;) body).  Each event has exactly one call site for every expensive
// operation -- one Philox block (the stream keeps a 3-word queue so one refill per event is
// always enough for the u and v draws) and no divide (the holding test runs in probability
// space, see below) -- so a diverged warp pays each of them at most once per trip.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "internal.hpp"

// Product-form probability-space holding test (see walker_hold): 1 = on (default since round 2,
// C2 kernel -1.9 %), 0 = the round-1 divide form (A/B builds).
#ifndef EXPMC_PROD
#define EXPMC_PROD 1
#endif

namespace expmc_b200 {

// log1p polynomial of fast_log in constant memory: DFMA reads it as a c[] operand directly.
__constant__ double c_log_poly[9] = EXPMC_LOG_POLY;
__constant__ double c_exp_poly[14] = EXPMC_EXP_POLY;

// exp(x), bitwise the toolkit's (fastmath.cuh), coefficients read from constant memory.
__device__ __forceinline__ double dexp(double x) { return exp_fast(x, c_exp_poly); }
__device__ const LogEntry g_log_table[128] = {
#include "log_table.inc"
};

// Copy the log table to shared memory (call from every thread, then __syncthreads()).
__device__ __forceinline__ void load_log_table(LogEntry* s_log) {
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s_log[i] = g_log_table[i];
}

// ----------------------------------------------------------------------------- Philox
struct Stream {
    uint32_t k0, k1;       // key = (seed_lo, seed_hi)                       rng.hpp:25
    uint32_t c1, c2, c3;   // counter words 1..3 = (sample_lo, sample_hi, level|lane<<24)
    uint32_t block;        // counter word 0, one per 128-bit block           rng.hpp:56
    uint64_t w0, w1, w2;   // queue of unconsumed 64-bit words, w0 next
    uint32_t n;            // queued words
};

__device__ __forceinline__ void stream_init(Stream& s, uint64_t seed, uint64_t sample, uint32_t key3) {
    s.k0 = static_cast<uint32_t>(seed);
    s.k1 = static_cast<uint32_t>(seed >> 32);
    s.c1 = static_cast<uint32_t>(sample);
    s.c2 = static_cast<uint32_t>(sample >> 32);
    s.c3 = key3;
    s.block = 0;
    s.n = 0;  // w0..w2 are written before they are read
}

// Philox4x32 with 10 rounds and the Weyl key schedule (rng.hpp:44-62).
__device__ __forceinline__ void philox10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                         uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
        const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
        c1 = static_cast<uint32_t>(p1);
        c3 = static_cast<uint32_t>(p0);
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// Make sure two words are queued (an event draws at most u and v).  A refill appends the
// block's words in the reference's consumption order: (c2,c3) first, then (c0,c1)
// (rng.hpp:32-36, 63-65).
__device__ __forceinline__ void stream_reserve2(Stream& s) {
    if (s.n < 2u) {
        uint32_t c0 = s.block++, c1 = s.c1, c2 = s.c2, c3 = s.c3;
        philox10(c0, c1, c2, c3, s.k0, s.k1);
        const uint64_t first = (static_cast<uint64_t>(c2) << 32) | c3;
        const uint64_t second = (static_cast<uint64_t>(c0) << 32) | c1;
        if (s.n == 0u) {
            s.w0 = first;
            s.w1 = second;
        } else {
            s.w1 = first;
            s.w2 = second;
        }
        s.n += 2u;
    }
}

__device__ __forceinline__ void stream_reserve2(Stream& s, const uint4*) { stream_reserve2(s); }  // keyed stream: no table

// The 53-bit integer K of the next uniform v = K 2^-53 (rng.hpp:34-35).
template <class ST>
__device__ __forceinline__ uint64_t stream_pop_bits(ST& s) {
    const uint64_t bits = s.w0;
    s.w0 = s.w1;
    s.w1 = s.w2;
    --s.n;
    return bits >> 11;
}

__device__ __forceinline__ double to_uniform(uint64_t k53) { return __dmul_rn(__ull2double_rn(k53), 0x1.0p-53); }

// next_uniform: 53 random bits -> [0,1) exactly as rng.hpp:35.
__device__ __forceinline__ double stream_pop(Stream& s) { return to_uniform(stream_pop_bits(s)); }

// Keyless stream (EXPMC_RKEYS): the Weyl key schedule of the warp's item seed is precomputed once
// per item into the warp's item constants in shared memory (ItemConst::rk, 80 B), and a refill
// reads the ten (k0, k1) round-key pairs with five 128-bit shared loads instead of adding the key
// increments (18 integer adds per block) -- and the stream holds no key registers.  The table
// sits in ItemConst so that its address is the item-constant pointer the loop already holds
// (a table of its own cost six address instructions per Philox block).
#ifndef EXPMC_RKEYS
#define EXPMC_RKEYS 1
#endif
// EXPMC_QEND: the reference-order walker reads u and v in place and advances its word queue once
// at the event's end instead of shifting it on every pop (A/B builds).
#ifndef EXPMC_QEND
#define EXPMC_QEND 1
#endif
__device__ __forceinline__ void set_round_keys(uint4* t, uint64_t seed) {  // t = ItemConst::rk (prepare, lane 0)
    uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        t[r] = make_uint4(k0, k1, k0 + 0x9E3779B9u, k1 + 0xBB67AE85u);
        k0 += 2u * 0x9E3779B9u;
        k1 += 2u * 0xBB67AE85u;
    }
}

struct StreamRK {
    uint32_t c1, c2, c3;   // counter words 1..3 (the key comes from ItemConst::rk)
    uint32_t block;
    uint64_t w0, w1, w2;
    uint32_t n;
};

__device__ __forceinline__ void stream_init(StreamRK& s, uint64_t sample, uint32_t key3) {
    s.c1 = static_cast<uint32_t>(sample);
    s.c2 = static_cast<uint32_t>(sample >> 32);
    s.c3 = key3;
    s.block = 0;
    s.n = 0;
}

// Philox4x32-10 with the warp's precomputed round keys (rng.hpp:44-62).
__device__ __forceinline__ void philox10_rk(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, const uint4* t) {
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        const uint4 k = t[r];
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // round keys (k.x, k.y) then (k.z, k.w)
            const uint32_t ka = h ? k.z : k.x, kb = h ? k.w : k.y;
            const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
            const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
            const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ ka;
            const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ kb;
            c1 = static_cast<uint32_t>(p1);
            c3 = static_cast<uint32_t>(p0);
            c0 = n0;
            c2 = n2;
        }
    }
}

__device__ __forceinline__ void stream_reserve2(StreamRK& s, const uint4* rk) {
    if (s.n < 2u) {
        uint32_t c0 = s.block++, c1 = s.c1, c2 = s.c2, c3 = s.c3;
        philox10_rk(c0, c1, c2, c3, rk);
        const uint64_t first = (static_cast<uint64_t>(c2) << 32) | c3;
        const uint64_t second = (static_cast<uint64_t>(c0) << 32) | c1;
        if (s.n == 0u) {
            s.w0 = first;
            s.w1 = second;
        } else {
            s.w1 = first;
            s.w2 = second;
        }
        s.n += 2u;
    }
}

// One-step stream (level-0 walker, EXPMC_EV0).  A level-0 sample is one fine step, and a step
// ends at its first non-jump draw: the sample consumes u_1 v_1 u_2 v_2 ... u_k (a jump draws u
// and v, paths.cpp:52-57; the final u, or an absorbing row, ends it).  Block b of the stream
// holds (first, second) = (u_{b+1}, v_{b+1}) in consumption order (rng.hpp:32-36, 63-65), so
// every event starts on a fresh block: one unconditional Philox call per event, no word queue
// (the queue's bookkeeping and its divergent refill branch are gone).  Same words, same order.
#ifndef EXPMC_EV0
#define EXPMC_EV0 1
#endif
#if EXPMC_EV0 && !EXPMC_QEND
#error "EXPMC_EV0 reads u and v in place (EXPMC_QEND)"
#endif
// EXPMC_L0TUNE: the level-0 walker's own event function (walker0_event) instead of walker_hold.
#ifndef EXPMC_L0TUNE
#define EXPMC_L0TUNE 1
#endif
#if EXPMC_L0TUNE && !(EXPMC_RKEYS && EXPMC_EV0 && EXPMC_PROD)
#error "EXPMC_L0TUNE is written for the one-block-per-event keyless stream and the product form"
#endif
struct StreamEv {
    uint32_t c1, c2, c3;
    uint32_t block;
    uint64_t w0, w1;  // this event's u and v words
};

__device__ __forceinline__ void stream_init(StreamEv& s, uint64_t sample, uint32_t key3) {
    s.c1 = static_cast<uint32_t>(sample);
    s.c2 = static_cast<uint32_t>(sample >> 32);
    s.c3 = key3;
    s.block = 0;
}

__device__ __forceinline__ void stream_reserve2(StreamEv& s, const uint4* rk) {
    uint32_t c0 = s.block++, c1 = s.c1, c2 = s.c2, c3 = s.c3;
    philox10_rk(c0, c1, c2, c3, rk);
    s.w0 = (static_cast<uint64_t>(c2) << 32) | c3;
    s.w1 = (static_cast<uint64_t>(c0) << 32) | c1;
}

// One-block stream read in order: the first pop returns the event's first word, the second its second.
__device__ __forceinline__ uint64_t stream_pop_bits(StreamEv& s) {
    const uint64_t bits = s.w0;
    s.w0 = s.w1;
    return bits >> 11;
}

// The event's words are consumed: advance the queue by u, or by u and v after a jump.
template <class ST>
__device__ __forceinline__ void stream_advance(ST& s, bool jump) {
    s.w0 = jump ? s.w2 : s.w1;
    s.w1 = s.w2;
    s.n -= jump ? 2u : 1u;
}
__device__ __forceinline__ void stream_advance(StreamEv&, bool) {}  // the next event refills

// ----------------------------------------------------------------------------- tables
struct Row {  // u_i is not kept in registers: walker_finish reloads it for the end state
    double d, rate;
    uint32_t begin, deg;
};

// &rows[i] by one 32 x 32 -> 64-bit multiply-add (for an index that comes out of a mask the
// compiler otherwise splits the shift over six instructions).
__device__ __forceinline__ const RowRec* row_at(const RowRec* __restrict__ rows, uint32_t i) {
    uint64_t p;
    asm("mad.wide.u32 %0, %1, 32, %2;" : "=l"(p) : "r"(i), "l"(reinterpret_cast<uint64_t>(rows)));
    return reinterpret_cast<const RowRec*>(p);
}

__device__ __forceinline__ Row load_row(const RowRec* __restrict__ rows, uint32_t i) {
    const RowRec* p = row_at(rows, i);
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));  // rate, begin, deg
    Row r;
    r.d = __ldg(&p->d);
    r.rate = __hiloint2double(static_cast<int>(a.y), static_cast<int>(a.x));
    r.begin = a.z;
    r.deg = a.w;
    return r;
}

// The jump half of a row record (rate, begin, deg); the level-0 walker reads d only when the
// path ends (walker0_sample).
__device__ __forceinline__ void load_row_jump(const RowRec* __restrict__ rows, uint32_t i, Row& r) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(row_at(rows, i)));
    r.rate = __hiloint2double(static_cast<int>(a.y), static_cast<int>(a.x));
    r.begin = a.z;
    r.deg = a.w;
}

// Neighbour choice (paths.cpp:57-65): k = upper_bound(cdf[begin:begin+deg], v) clamped to
// deg-1, then (target, sign) = tgt[begin + k].  Returns the packed target|sign word.
//
// Uniform rows (kUniformRow: cdf_j == fl((j+1)/deg) for all j) never read the CDF.  With
// v = K 2^-53 and |v - (j+1)/deg| >= 2^-53 for every j, fl((j+1)/deg) <= v iff
// (j+1)/deg <= v (the rounding error of fl is <= 2^-54), so upper_bound = floor(K deg / 2^53),
// an exact 128-bit integer product.  Draws within 2^-53 of a boundary (probability 2 deg 2^-53)
// take the generic path, which compares against the stored CDF exactly as std::upper_bound
// does: the choice is the reference's in every case.  Generic rows of degree <= 4 read their
// CDF with independent loads and count (#{j : cdf_j <= v} == upper_bound on a non-decreasing
// array); wider rows binary-search.
//
// kAlias (event-driven sampler only: its parity is statistical): a non-uniform row with an
// alias table draws slot j = floor(v deg) = hi64(K 2^11 deg) and keeps its own target iff the
// fraction lo64(K 2^11 deg) 2^-64 is below prob_j -- one 16-B load, any degree.
__device__ __forceinline__ bool alias_row(const EdgeTables& e, uint32_t degf) {
    return !(degf & kUniformRow) && e.alias != nullptr && (degf & kDegMask) > 1u;
}

// The chosen slot (offset in the row) for the exact paths: uniform rows and the CDF search.
// pick_slot_np2 is pick_slot for a row that is not (uniform with a power-of-two degree).
__device__ __forceinline__ uint32_t pick_slot(const EdgeTables& e, uint32_t begin, uint32_t degf, uint64_t k53);
__device__ __forceinline__ uint32_t pick_slot_np2(const EdgeTables& e, uint32_t begin, uint32_t degf, uint64_t k53);

template <bool kAlias = false>
__device__ __forceinline__ uint32_t pick_edge(const EdgeTables& e, uint32_t begin, uint32_t degf, uint64_t k53) {
    if (kAlias && alias_row(e, degf)) {
        const uint32_t deg = degf & kDegMask;
        const uint64_t x = k53 << 11;
        const uint32_t j = static_cast<uint32_t>(__umul64hi(x, deg));
        const double f = __dmul_rn(__ull2double_rn((x * deg) >> 11), 0x1.0p-53);
        const uint4 r = __ldg(reinterpret_cast<const uint4*>(e.alias + begin + j));
        return f < __hiloint2double(static_cast<int>(r.y), static_cast<int>(r.x)) ? r.z : r.w;
    }
    return __ldg(e.tgt + static_cast<uint32_t>(begin + pick_slot(e, begin, degf, k53)));  // edges < 2^32: a 32-bit index
}

__device__ __forceinline__ uint32_t pick_slot(const EdgeTables& e, uint32_t begin, uint32_t degf, uint64_t k53) {
    const uint32_t deg = degf & kDegMask;
    if ((degf & kUniformRow) && (deg & (deg - 1u)) == 0u) {
        // power-of-two degree 2^p (every interior row of a 2-D Laplacian: 4): cdf_j = (j+1) 2^-p
        // and v 2^p = K 2^(p-53) are exact, so upper_bound = K >> (53 - p) <= deg - 1, no boundary case
        return static_cast<uint32_t>(k53 >> (53 - (31 - __clz(deg))));
    }
    return pick_slot_np2(e, begin, degf, k53);
}

__device__ __forceinline__ uint32_t pick_slot_np2(const EdgeTables& e, uint32_t begin, uint32_t degf, uint64_t k53) {
    const uint32_t deg = degf & kDegMask;
    uint32_t k = 0;
    bool done = false;
    if (degf & kUniformRow) {
        // t = fl(v deg) is within deg 2^-53 of v deg; a fractional part at least 2 deg 2^-53 away
        // from 0 and 1 puts v deg at least deg 2^-53 from every integer: floor(t) is then the
        // exact upper_bound and the boundary condition above holds.
        const double dg = static_cast<double>(deg);
        const double t = __dmul_rn(to_uniform(k53), dg);
        const double fl = floor(t);
        const double f = __dsub_rn(t, fl);
        const double margin = __dmul_rn(dg, 0x1.0p-52);
        k = static_cast<uint32_t>(fl);
        done = f >= margin && f <= __dsub_rn(1.0, margin);
    }
    if (!done) {
        const double v = to_uniform(k53);
        const double* c = e.cdf + begin;
        if (deg <= 4u) {
            k = (__ldg(c) <= v) + (deg > 1u && __ldg(c + 1) <= v) + (deg > 2u && __ldg(c + 2) <= v) +
                (deg > 3u && __ldg(c + 3) <= v);
        } else {
            uint32_t lo = 0, count = deg;
            while (count > 0u) {
                const uint32_t step = count >> 1;
                const uint32_t it = lo + step;
                if (!(v < __ldg(c + it))) {
                    lo = it + 1u;
                    count -= step + 1u;
                } else {
                    count = step;
                }
            }
            k = lo;
        }
    }
    return k < deg - 1u ? k : deg - 1u;
}

// ----------------------------------------------------------------------------- walker
// Holding-interval test.  The reference decides "no jump in the rest of the interval" by
// u >= q with q = -expm1(-rate*remaining) (paths.cpp:53, 68, 90) and, on a jump, spends
// E = -log1p(-u) of the interval (paths.cpp:54).  With 1 - u = M 2^-53 exactly (M = 2^53 - K),
// u < q is 1 - u > S, S = e^{-rate*remaining}: the walker works in probability space ("S-mode")
// with no logarithm and no exponential.  After jumps with draws u_1..u_k in the current step,
// S = S0 / prod_j (1 - u_j) (e^{-rate (remaining - E/rate)} = S / (1 - u)), so the test is
// prod_j (1 - u_j) (1 - u) 2^53 > S0 2^53: the walker keeps the product (hold, starts at 1) and
// the step's S0 2^53 (thr) -- one multiply per event and none of round 1's divides per jump
// ("product form", EXPMC_PROD; EXPMC_PROD=0 keeps hold = S 2^53 and divides by 1 - u per jump).
// A fresh step starts from S0 = e^{-rate dt}, cached per item for
// the entry row's rate (every interior row of C1/C2/C5 shares it).  When a jump changes the
// rate, the rest of the step continues in time space ("T-mode", hold = -remaining with
// remaining = -log(S)/rate, then the reference's log-space test E < rate*remaining per event);
// so does a step whose S0 would underflow (rate dt >= 690).  Draws, jump chain and every
// sample value are the reference's; only a u within a few ulps of its threshold may round the
// other way (probability ~1e-16 per event, the same order as the CUDA-vs-glibc expm1/log1p
// differences that reference-order sampling accepts anyway).
constexpr double kSModeMaxX = 690.0;  // e^{-690} ~ 2^-995: S0 2^53 stays a normal number

// Per-item constants (uniform across the warp while it works on one chunk).
struct ItemConst {
    uint64_t seed;
    uint64_t nsteps;
    double dt;
    double half_dt;  // dt_ * 0.5, the left factor of paths.cpp:110
    double tend;     // N * dt (= beta), event-driven walker
    double inv_dt;   // 1 / dt, event-driven walker
    double h_fine;   // fem: dt / 3, the fine Simpson scale (mlmc.cpp:68, 90)
    double h_coarse; // fem: (2 dt) / 3, the coarse Simpson scale (mlmc.cpp:68, 91)
    uint32_t entry;
    uint32_t key3;
    uint32_t base;
    // reference-order walker: S-mode start value S0 2^53 for steps in rows of rate s0_rate
    double s0_rate;     // -1: no cached rate
    double s0_hold;
    union {
        double smode_max_x; // reference-order walker: rate dt below which a fresh step runs in S-mode (-1: T-mode only)
        double skip_scale;  // event walker: 1 / log P(M < m_safe) < 0, jumpers located by geometric gaps
    };                      //   (0: off; EdPolicy::prepare always writes it)
    Row r0;             // entry mode: the entry's row record and its fresh-step hold (the
    double h0;          //   restart of every sample reads them from here, not from the tables)
    double hold0;       // level-0 walker: the restart's hold (product form: 1 in S-mode, else h0)
    double h0s;         // level-0 walker: the restart's threshold, h0 2^11 = S0 2^64 in S-mode (else h0, unused)
    double ea_key;      // base level: e^{ea_key} = ea_val, the exponent of a path that keeps the
    double ea_val;      //   entry's d (every interior path of C5) -- one exp per chunk, not per sample
    // event-driven entry mode: closed-form first holding interval (EdPolicy::prepare)
    uint64_t m_safe;    // M = 2^53 - K < m_safe => the path never leaves the entry (0: off)
    double hold_fine;   // that path's (fine, coarse) and run_level sample x
    double hold_coarse;
    double hold_x;
    uint4 rk[5];        // keyless streams: the item seed's Philox round keys (set_round_keys)
};

// sample_initial (paths.cpp:32-36): the path's first draw picks the start state by
// upper_bound over the CDF of u -- an exact binary search over the same fp64 CDF.
template <bool F, class ST>
__device__ __forceinline__ uint32_t draw_start(ST& st, const ItemConst& ic, const LaneData& fi) {
    if (!F) return ic.entry;
    stream_reserve2(st, ic.rk);
    const uint64_t k53 = stream_pop_bits(st);
    const double v = to_uniform(k53);
    // the draw's guide bucket bounds the search (context.cu: ensure_forward_init)
    const uint32_t b = static_cast<uint32_t>(k53 >> (53u - fi.gbits));
    uint32_t lo = __ldg(fi.guide + b);
    uint32_t count = __ldg(fi.guide + b + 1) - lo;
    while (count > 0u) {
        const uint32_t step = count >> 1;
        const uint32_t it = lo + step;
        if (!(v < __ldg(fi.cdf + it))) {
            lo = it + 1u;
            count -= step + 1u;
        } else {
            count = step;
        }
    }
    return lo;
}

// The terminal factor: u[end] (entry mode, paths.cpp:112,138) or sum(u) (forward, 156,178).
template <bool F>
__device__ __forceinline__ double terminal_factor(const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows,
                                                  uint32_t state) {
    return F ? fi.total : __ldg(&rows[state].u);
}

struct Walker {
    Stream st;
    Row cur;               // row record of the current state
    uint32_t state;
    int32_t sign;
    uint32_t half;         // coupled: 0 before the pair's middle node, 1 after
    double hold;           // S-mode (> 0): prod (1 - u_j) (EXPMC_PROD) or e^{-rate*remaining} 2^53;
                           //   T-mode (<= 0): -remaining
#if EXPMC_PROD
    double thr;            // product form: S-mode hold = prod (1 - u_j) over the step's jumps and
                           //   thr = S0 2^53 of the step; jump iff hold m > thr (no divide)
#endif
    double acc_a, acc_b;   // single: expo; coupled: coarse, delta
    double d0, d1;         // d[s0], d[s1]
    uint64_t left;         // fine steps not yet completed, the current one included (counts down:
                           //   the step-end test needs no item constant)
};


// Start value of a fresh fine step in a row of the given rate (paths.cpp:95-96).
__device__ __forceinline__ double fresh_hold(const ItemConst& ic, double rate) {
    if (rate == ic.s0_rate) return ic.s0_hold;
    const double x = __dmul_rn(rate, ic.dt);
    return x < ic.smode_max_x ? __dmul_rn(dexp(-x), 0x1.0p53) : -ic.dt;
}

// Per chunk (lane 0): the entry row and its fresh-step hold (every sample restarts from them)
// and the S0 cache for the entry row's rate; flags may force T-mode.
__device__ __forceinline__ void prepare_hold(ItemConst& ic, const RowRec* __restrict__ rows, uint32_t flags) {
    ic.r0 = load_row(rows, ic.entry);
    if (flags & EXPMC_SAMPLER_FLAG_LOG_HOLD) {
        ic.smode_max_x = -1.0;
    } else {
        const double x = __dmul_rn(ic.r0.rate, ic.dt);
        if (x < ic.smode_max_x) {
            ic.s0_rate = ic.r0.rate;
            ic.s0_hold = __dmul_rn(dexp(-x), 0x1.0p53);
        }
    }
    ic.h0 = fresh_hold(ic, ic.r0.rate);
#if EXPMC_PROD
    ic.hold0 = ic.h0 > 0.0 ? 1.0 : ic.h0;  // set_hold(w, h0)
    ic.h0s = ic.h0 > 0.0 ? __dmul_rn(ic.h0, 0x1.0p11) : ic.h0;
#else
    ic.hold0 = ic.h0;
#endif
    if (ic.base && ic.nsteps <= 64u) {  // walker_event / last_step_sums on a constant-d path
        double a = 0.0;
        for (uint64_t k = 0; k < ic.nsteps; ++k) a = __dadd_rn(a, __dmul_rn(ic.half_dt, __dadd_rn(ic.r0.d, ic.r0.d)));
        ic.ea_key = a;
        ic.ea_val = a == 0.0 ? 1.0 : dexp(a);
    }
}

// A fresh step's hold (fresh_hold's value): the product form keeps S0 2^53 as the threshold and
// starts the product at 1.
template <class WK>
__device__ __forceinline__ void set_hold(WK& w, double h) {
#if EXPMC_PROD
    w.thr = h;
    w.hold = h > 0.0 ? 1.0 : h;
#else
    w.hold = h;
#endif
}

template <bool F>
__device__ __forceinline__ void walker_start(Walker& w, const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows,
                                             uint64_t sample) {
    stream_init(w.st, ic.seed, sample, ic.key3);
    const uint32_t s0 = draw_start<F>(w.st, ic, fi);
    if (!F) {  // entry mode: the item's cached start (prepare_hold; +3 % on C2)
        w.cur = ic.r0;
        set_hold(w, ic.h0);
    } else {
        w.cur = load_row(rows, s0);
        set_hold(w, fresh_hold(ic, w.cur.rate));
    }
    w.state = s0;
    w.sign = 1;
    w.half = 0;
    w.acc_a = 0.0;
    w.acc_b = 0.0;
    w.d0 = w.cur.d;  // d1 is written at the pair's middle node before it is read
    w.left = ic.nsteps;
}

// One pass of evolve_common's for(;;) body (paths.cpp:48-69): the holding-interval test and,
// on a jump, the neighbour draw.  Returns true when the holding interval ends the fine step.
// Exponential draws and jumps are counted straight into the caller's accumulators (cost =
// draws + fine steps, paths.hpp:22-23; the fine steps are added when the sample ends).
template <class WK>
__device__ __forceinline__ bool walker_hold(WK& w, const RowRec* __restrict__ rows, const EdgeTables& edges,
                                            const LogEntry* s_log, unsigned long long& draws,
                                            unsigned long long& jumps, const uint4* rk = nullptr) {
    stream_reserve2(w.st, rk);  // the event's only Philox call site (rk: keyless streams)
    bool step_done = true;
    if (w.cur.rate != 0.0) {  // rate == 0: absorbing row, holding time +inf (paths.cpp:50)
#if EXPMC_QEND
        const uint64_t k53 = w.st.w0 >> 11;  // u; consumed with v (on a jump) at the event's end
#else
        const uint64_t k53 = stream_pop_bits(w.st);
#endif
        ++draws;
        const double m = __ull2double_rn((uint64_t{1} << 53) - k53);  // (1 - u) 2^53, exact
        const bool smode = w.hold > 0.0;
        double e = 0.0;
        bool jump;
#if EXPMC_PROD
        double t = 0.0;
        if (smode) {
            t = __dmul_rn(w.hold, m);  // prod (1 - u_j) (1 - u) 2^53
            jump = t > w.thr;          // (1 - u) > S0 / prod (1 - u_j) = S  <=>  u < q
        } else {
#else
        if (smode) {
            jump = m > w.hold;  // 1 - u > S  <=>  u < q
        } else {
#endif
            // T-mode: E = -log1p(-u) = -log(m 2^-53) (fastmath.cuh: <= 1 ulp), jump iff E < rate * remaining
            e = -fast_log(m, -53, s_log, c_log_poly);
            jump = e < __dmul_rn(w.cur.rate, -w.hold);
        }
        if (jump) {
#if EXPMC_PROD
            // S-mode: the product times (1 - u), exact rescale; T-mode: -(remaining - E / rate) (paths.cpp:54)
            double h1 = smode ? __dmul_rn(t, 0x1.0p-53) : -__dsub_rn(-w.hold, fast_div(e, w.cur.rate));
#else
            // S-mode: S / (1 - u) (scaled); T-mode: -(remaining - E / rate) (paths.cpp:54)
            const double q = fast_div(smode ? __dmul_rn(w.hold, 0x1.0p53) : e, smode ? m : w.cur.rate);
            double h1 = smode ? q : -__dsub_rn(-w.hold, q);
#endif
            ++jumps;
            const double rate0 = w.cur.rate;
#if EXPMC_QEND
            const uint32_t ts = pick_edge(edges, w.cur.begin, w.cur.deg, w.st.w1 >> 11);
#else
            const uint32_t ts = pick_edge(edges, w.cur.begin, w.cur.deg, stream_pop_bits(w.st));
#endif
            if (ts & kSignBit) w.sign = -w.sign;
            w.state = ts & kTargetMask;
            w.cur = load_row(rows, w.state);
#if EXPMC_PROD
            if (smode && w.cur.rate != rate0)  // to T-mode: S 2^53 = S0 2^53 / prod, -remaining = log(S) / rate
                h1 = fast_div(fast_log(fast_div(w.thr, h1), -53, s_log, c_log_poly), rate0);
#else
            if (smode && w.cur.rate != rate0)  // S-mode needs one rate per step: to T-mode
                h1 = fast_div(fast_log(h1, -53, s_log, c_log_poly), rate0);  // -remaining = log(S) / rate
#endif
            w.hold = h1;
            // remaining <= 0: rounding pushed past the boundary, the step ends (paths.cpp:67)
            step_done = !(smode ? h1 != 0.0 : h1 < 0.0);
        }
#if EXPMC_QEND
        // the queue advances once per event: by u, or by u and v after a jump
        stream_advance(w.st, jump);
#endif
    }
    return step_done;
}

// One event of the path: walker_hold plus the step bookkeeping of single / coupled
// (paths.cpp:108-110, 130-136) when the holding interval ends the fine step.  Returns true
// when the sample's last fine step has completed.
__device__ __forceinline__ bool walker_event(Walker& w, const ItemConst& ic, const RowRec* __restrict__ rows,
                                             const EdgeTables& edges, const LogEntry* s_log,
                                             unsigned long long& draws, unsigned long long& jumps) {
    if (!walker_hold(w, rows, edges, s_log, draws, jumps)) return false;
    // The sample's last step ends it; its sums are taken by walker_finish / walker_sample, in
    // the finishing lanes' own divergent section (level-0 chunks: no step-end section at all).
    if (w.left == 1u) return true;
    // ---- a non-final fine step ended in w.state
    const double dn = w.cur.d;
    if (ic.base) {
        // expo += dt_ * 0.5 * (d[s0] + d[state])                             paths.cpp:110
        w.acc_a = __dadd_rn(w.acc_a, __dmul_rn(ic.half_dt, __dadd_rn(w.d0, dn)));
        w.d0 = dn;
    } else if (w.half == 0u) {
        w.d1 = dn;  // s1 = state after the first fine step of the pair       paths.cpp:132
        w.half = 1u;
    } else {
        // half_ends = 0.5 (d0 + d2); coarse += dt (d0 + d2); delta += dt (d1 - half_ends)
        const double s02 = __dadd_rn(w.d0, dn);  //                            paths.cpp:134-136
        const double half_ends = __dmul_rn(0.5, s02);
        w.acc_a = __dadd_rn(w.acc_a, __dmul_rn(ic.dt, s02));
        w.acc_b = __dadd_rn(w.acc_b, __dmul_rn(ic.dt, __dsub_rn(w.d1, half_ends)));
        w.d0 = dn;
        w.half = 0u;
    }
    --w.left;
    set_hold(w, fresh_hold(ic, w.cur.rate));  // next fine step: fresh holding interval of length dt (paths.cpp:95-96)
    return false;
}

// The last step's sums, the same operations walker_event applies to every other step:
// single: expo + dt_ 0.5 (d[s0] + d[end]) (paths.cpp:110); coupled (the last step closes a pair):
// coarse + dt (d0 + d2), delta + dt (d1 - 0.5 (d0 + d2)) (paths.cpp:134-136).
__device__ __forceinline__ void last_step_sums(const Walker& w, const ItemConst& ic, double& a, double& b) {
    const double dn = w.cur.d;
    if (ic.base) {
        a = __dadd_rn(w.acc_a, __dmul_rn(ic.half_dt, __dadd_rn(w.d0, dn)));
        b = w.acc_b;
    } else {
        const double s02 = __dadd_rn(w.d0, dn);
        const double half_ends = __dmul_rn(0.5, s02);
        a = __dadd_rn(w.acc_a, __dmul_rn(ic.dt, s02));
        b = __dadd_rn(w.acc_b, __dmul_rn(ic.dt, __dsub_rn(w.d1, half_ends)));
    }
}

// exp(x) with the exact shortcut exp(0) = 1 (both libms return exactly 1): rows whose d is
// constant along the path (every interior row of a Laplacian) never pay for the exp.
__device__ __forceinline__ double exp_or_one(double x) { return x == 0.0 ? 1.0 : dexp(x); }

// Terminal values: single -> (sign * e^expo) * u[end] (paths.cpp:112);
// coupled -> uf = sign * u[end]; (uf e^{coarse+delta}, uf e^{coarse}) (paths.cpp:138-140).
template <bool F>
__device__ __forceinline__ void walker_finish(const Walker& w, const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows,
                                              double& fine, double& coarse) {
    double acc_a, acc_b;
    last_step_sums(w, ic, acc_a, acc_b);
    const double sg = static_cast<double>(w.sign);
    const double u_end = terminal_factor<F>(ic, fi, rows, w.state);  // same sector as the last row record read
    if (ic.base) {
        fine = __dmul_rn(__dmul_rn(sg, acc_a == ic.ea_key ? ic.ea_val : exp_or_one(acc_a)), u_end);
        coarse = 0.0;
    } else {
        const double uf = __dmul_rn(sg, u_end);
        fine = __dmul_rn(uf, exp_or_one(__dadd_rn(acc_a, acc_b)));
        coarse = __dmul_rn(uf, exp_or_one(acc_a));
    }
}

// The level-statistics sample x = P_l (base) or P_l - P_{l-1} (coupled), as run_level_ex adds
// it (mlmc.cpp:103-108).  delta == 0 makes fine and coarse bitwise equal, so x = 0 exactly.
template <bool F>
__device__ __forceinline__ double walker_sample(const Walker& w, const ItemConst& ic, const LaneData& fi, const RowRec* __restrict__ rows) {
    double acc_a, acc_b;
    last_step_sums(w, ic, acc_a, acc_b);
    if (!ic.base && acc_b == 0.0) return 0.0;
    // same values as walker_finish, with one exp call site shared by both modes
    const double sg = static_cast<double>(w.sign);
    const double u_end = terminal_factor<F>(ic, fi, rows, w.state);
    // single: e^expo (the item's cached value when the path kept the entry's d); coupled: e^coarse
    const double ea = ic.base && acc_a == ic.ea_key ? ic.ea_val : exp_or_one(acc_a);
    if (ic.base) return __dmul_rn(__dmul_rn(sg, ea), u_end);
    const double uf = __dmul_rn(sg, u_end);
    return __dsub_rn(__dmul_rn(uf, dexp(__dadd_rn(acc_a, acc_b))), __dmul_rn(uf, ea));
}

// Deferred finish (k_sample, EXPMC_DEFER): the finishing lane records only its last step's sums
// and its packed end (state | sign bit); the value -- walker_sample's arithmetic, same operation
// order -- is computed later from that record by a converged pass of the warp.
__device__ __forceinline__ void walker_end_record(const Walker& w, const ItemConst& ic, double& a, double& b,
                                                  uint32_t& se) {
    last_step_sums(w, ic, a, b);
    se = w.state | (w.sign < 0 ? kSignBit : 0u);
}

template <bool F>
__device__ __forceinline__ double walker_value(double acc_a, double acc_b, uint32_t se, const ItemConst& ic,
                                               const LaneData& fi, const RowRec* __restrict__ rows) {
    if (!ic.base && acc_b == 0.0) return 0.0;
    const double sg = (se & kSignBit) ? -1.0 : 1.0;
    const double u_end = terminal_factor<F>(ic, fi, rows, se & kTargetMask);
    const double ea = ic.base && acc_a == ic.ea_key ? ic.ea_val : exp_or_one(acc_a);
    if (ic.base) return __dmul_rn(__dmul_rn(sg, ea), u_end);
    const double uf = __dmul_rn(sg, u_end);
    return __dsub_rn(__dmul_rn(uf, dexp(__dadd_rn(acc_a, acc_b))), __dmul_rn(uf, ea));
}

// ----------------------------------------------------------------------------- level 0
// Base level with one fine step (l = l0 = 0: every C1/C2 component's first and largest level;
// ~80 % of C2's loop trips).  The sample ends with the step, so the walker needs none of the
// step bookkeeping -- no accumulators, d0/d1, pair half or step count (11 registers of
// Walker): expo = dt 0.5 (d[entry] + d[end]) (paths.cpp:108-110), value = sign e^expo u[end]
// (paths.cpp:112), the same operations in the same order as walker_event + walker_sample.
struct Walker0 {
#if EXPMC_RKEYS && EXPMC_EV0
    StreamEv st;
#elif EXPMC_RKEYS
    StreamRK st;
#else
    Stream st;
#endif
    Row cur;
    uint32_t state;
#if EXPMC_L0TUNE
    uint32_t sign;  // kSignBit when the path's sign is -1, else 0
#else
    int32_t sign;
#endif
    double hold;
#if EXPMC_PROD
    double thr;
#endif
};

__device__ __forceinline__ void walker0_start(Walker0& w, const ItemConst& ic, uint64_t sample) {
#if EXPMC_RKEYS
    stream_init(w.st, sample, ic.key3);
#else
    stream_init(w.st, ic.seed, sample, ic.key3);
#endif
    w.cur = ic.r0;
    w.state = ic.entry;
#if EXPMC_L0TUNE
    w.thr = ic.h0s;  // set_hold(w, ic.h0) with the threshold as S0 2^64 (walker0_event)
    w.hold = ic.hold0;
    w.sign = 0u;
#else
    set_hold(w, ic.h0);
    w.sign = 1;
#endif
}

#if EXPMC_L0TUNE
// walker_hold for the level-0 walker, the same tests and values with the instruction count of
// the common case cut (C2: uniform rows of degree 4, one rate, S-mode):
//   * one Philox block per event, u = (c2, c3), v = (c0, c1) (StreamEv), round keys read through
//     the item-constant pointer;
//   * uniform row of degree 2^p: upper_bound = K >> (53 - p) = v word >> (64 - p), one funnel
//     shift of the v word's high half; the (uniform, power of two) test is one and-not on
//     deg ^ kUniformRow; table addresses from 32-bit indices;
//   * the sign is kept as a sign bit and xor-ed with the target word's;
//   * the step-end tests leave the common path: an S-mode jump that keeps the rate leaves
//     hold = prod (1 - u_j) 2^0 > 0 (t > thr >= 2^-942), never the boundary case h1 == 0.
__device__ __forceinline__ bool walker0_event(Walker0& w, const ItemConst& ic, const RowRec* __restrict__ rows,
                                              const EdgeTables& edges, const LogEntry* s_log,
                                              unsigned long long& draws, unsigned long long& jumps) {
    uint32_t c0 = w.st.block++, c1 = w.st.c1, c2 = w.st.c2, c3 = w.st.c3;
    philox10_rk(c0, c1, c2, c3, ic.rk);
    bool done = true;
    if (w.cur.rate != 0.0) {  // rate == 0: absorbing row, holding time +inf (paths.cpp:50)
        ++draws;
        // m = (1 - u) 2^64 = 2^64 - (K << 11), K = (c2, c3) >> 11 (rng.hpp:32-35): the word with its
        // low 11 bits cleared converts exactly (53 significant bits) and the subtraction is exact --
        // no 64-bit shift and integer subtract.  The walker's threshold carries the same 2^11
        // (Walker0::thr = S0 2^64): every product below is the 2^53 form's times a power of two.
        const uint64_t uw = (static_cast<uint64_t>(c2) << 32) | (c3 & 0xFFFFF800u);
        const double m = __dsub_rn(0x1.0p64, __ull2double_rn(uw));
        const bool smode = w.hold > 0.0;
        double t = 0.0, e = 0.0;
        bool jump;
        if (smode) {
            t = __dmul_rn(w.hold, m);  // prod (1 - u_j) (1 - u) 2^64
            jump = t > w.thr;          // u < q
        } else {
            e = -fast_log(m, -64, s_log, c_log_poly);
            jump = e < __dmul_rn(w.cur.rate, -w.hold);
        }
        if (jump) {
            ++jumps;
            // S-mode: the product times (1 - u), exact rescale, > 0; T-mode: -(remaining - E / rate) (paths.cpp:54)
            double h1 = smode ? __dmul_rn(t, 0x1.0p-64) : -__dsub_rn(-w.hold, fast_div(e, w.cur.rate));
            const uint32_t degf = w.cur.deg;
            const uint32_t x = degf ^ kUniformRow;  // uniform row: its degree; other rows: bit 31 set
            uint32_t k;
            if ((x & (x - 1u)) == 0u)  // uniform, degree 2^p (deg >= 1 in a row with rate > 0)
                k = __funnelshift_rc(c0, 0u, 1u + static_cast<uint32_t>(__clz(x)));  // c0 >> (32 - p); 0 for p = 0
            else
                k = pick_slot_np2(edges, w.cur.begin, degf, ((static_cast<uint64_t>(c0) << 32) | c1) >> 11);
            const uint32_t ts = __ldg(edges.tgt + static_cast<uint32_t>(w.cur.begin + k));
            w.sign ^= ts & kSignBit;
            w.state = ts & kTargetMask;
            load_row_jump(rows, w.state, w.cur);  // the old row is dead here: the half record loads in place
            done = false;
            if (smode) {
                // S-mode lasts while the rate is the entry's (the sample's only fresh hold is the
                // entry's, walker0_start): a jump to another rate continues in T-mode,
                // S 2^53 = S0 2^53 / prod, -remaining = log(S) / rate
                const double rate0 = ic.r0.rate;
                if (w.cur.rate != rate0) {
                    h1 = fast_div(fast_log(fast_div(__dmul_rn(w.thr, 0x1.0p-11), h1), -53, s_log, c_log_poly), rate0);
                    done = h1 == 0.0;
                }
            } else {
                done = !(h1 < 0.0);  // remaining <= 0: rounding pushed past the boundary (paths.cpp:67)
            }
            w.hold = h1;
        }
    }
    return done;
}
#endif

__device__ __forceinline__ double walker0_sample(const Walker0& w, const ItemConst& ic, const RowRec* __restrict__ rows) {
#if EXPMC_L0TUNE
    // the end half of the last row's record: (d, u), one 128-bit load
    const double2 du = __ldg(reinterpret_cast<const double2*>(&rows[w.state].d));
    // a path that ends in a row with the entry's d has a == ea_key (the same sum of the same terms)
    double ea = ic.ea_val;
    if (du.x != ic.r0.d) {
        const double a = __dmul_rn(ic.half_dt, __dadd_rn(ic.r0.d, du.x));  // last_step_sums; 0 + a == a for every test below
        ea = a == ic.ea_key ? ic.ea_val : exp_or_one(a);
    }
    // (sign e^a) u[end]: the sign bit xor-ed into e^a is the product by +-1
    const double sea = __hiloint2double(__double2hiint(ea) ^ static_cast<int>(w.sign), __double2loint(ea));
    return __dmul_rn(sea, du.y);
#else
    const double a = __dadd_rn(0.0, __dmul_rn(ic.half_dt, __dadd_rn(ic.r0.d, w.cur.d)));  // last_step_sums
    const double sg = static_cast<double>(w.sign);
    const double ea = a == ic.ea_key ? ic.ea_val : exp_or_one(a);
    return __dmul_rn(__dmul_rn(sg, ea), __ldg(&rows[w.state].u));
#endif
}

__device__ __forceinline__ ItemConst load_item(const DevItem* __restrict__ items, uint32_t i) {
    const DevItem it = items[i];
    ItemConst ic;
    ic.seed = it.seed;
    ic.nsteps = it.nsteps;
    ic.dt = it.dt;
    ic.half_dt = __dmul_rn(it.dt, 0.5);
    ic.tend = __dmul_rn(it.dt, static_cast<double>(it.nsteps));
    ic.inv_dt = __ddiv_rn(1.0, it.dt);
    ic.h_fine = 0.0;  // fem only: FemPolicy::prepare
    ic.h_coarse = 0.0;
    ic.entry = it.entry;
    ic.key3 = it.key3;
    ic.base = it.base;
    ic.m_safe = 0;
    ic.hold_fine = ic.hold_coarse = ic.hold_x = 0.0;
    ic.s0_rate = -1.0;
    ic.s0_hold = 0.0;
    ic.smode_max_x = kSModeMaxX;
    ic.r0 = Row{0.0, 0.0, 0u, 0u};
    ic.h0 = 0.0;
    ic.hold0 = 0.0;
    ic.h0s = 0.0;
    ic.ea_key = 0.0;  // exp_or_one(0) = 1
    ic.ea_val = 1.0;
    return ic;
}

}  // namespace expmc_b200
