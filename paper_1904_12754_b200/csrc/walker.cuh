// Device-side path machinery: Philox4x32-10 streams and the reference-order CTMC walker.
//
// Reference-order means draw-for-draw identical to the reference's CPU sampler:
//   RngStream (rng.hpp:21-73), evolve_common (paths.cpp:44-71), LevelSampler::single /
//   ::coupled (paths.cpp:99-141), LevelSampler ctor thresholds (paths.cpp:84-91).
// Every floating-point expression that can round differently under FMA contraction is
// written with explicit __d*_rn intrinsics in the reference's evaluation order; the only
// remaining source of difference is CUDA's log1p/expm1/exp vs glibc (both < 1 ulp).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace expmc_b200 {

// ----------------------------------------------------------------------------- Philox
struct Stream {
    uint32_t k0, k1;      // key = (seed_lo, seed_hi)                  rng.hpp:25
    uint32_t c1, c2, c3;  // counter words 1..3 = (sample_lo, sample_hi, level|lane<<24)
    uint32_t block;       // counter word 0, one per 128-bit block      rng.hpp:56
    uint64_t buf;         // the second word of the last block (buffer_[0])
    uint32_t has;         // 1 if buf is still unconsumed
};

__device__ __forceinline__ void stream_init(Stream& s, uint64_t seed, uint64_t sample, uint32_t key3) {
    s.k0 = static_cast<uint32_t>(seed);
    s.k1 = static_cast<uint32_t>(seed >> 32);
    s.c1 = static_cast<uint32_t>(sample);
    s.c2 = static_cast<uint32_t>(sample >> 32);
    s.c3 = key3;
    s.block = 0;
    s.buf = 0;
    s.has = 0;
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

// next_uniform (rng.hpp:32-36): a refill yields words (c0c1, c2c3); c2c3 is consumed first.
__device__ __forceinline__ double next_uniform(Stream& s) {
    uint64_t bits;
    if (!s.has) {
        uint32_t c0 = s.block++, c1 = s.c1, c2 = s.c2, c3 = s.c3;
        philox10(c0, c1, c2, c3, s.k0, s.k1);
        s.buf = (static_cast<uint64_t>(c0) << 32) | c1;
        bits = (static_cast<uint64_t>(c2) << 32) | c3;
        s.has = 1;
    } else {
        bits = s.buf;
        s.has = 0;
    }
    return __dmul_rn(__ull2double_rn(bits >> 11), 0x1.0p-53);
}

// ----------------------------------------------------------------------------- tables
struct Row {
    double d, rate, u;
    uint32_t begin, deg;
};

__device__ __forceinline__ Row load_row(const RowRec* __restrict__ rows, uint32_t i) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(rows + i));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(rows + i) + 1);
    Row r;
    r.d = a.x;
    r.rate = a.y;
    r.u = __hiloint2double(static_cast<int>(b.y), static_cast<int>(b.x));
    r.begin = b.z;
    r.deg = b.w;
    return r;
}

__device__ __forceinline__ double edge_cdf(const uint4& e) {
    return __hiloint2double(static_cast<int>(e.y), static_cast<int>(e.x));
}

// Neighbour choice k = upper_bound(cdf[begin:begin+deg], v), clamped to deg-1
// (paths.cpp:57-63).  The row's CDF is non-decreasing, so upper_bound == #{j : cdf_j <= v};
// rows of degree <= 4 load all their edge records at once (independent loads, one round
// trip) and count; wider rows binary-search exactly like std::upper_bound.
__device__ __forceinline__ void pick_edge(const EdgeRec* __restrict__ edges, uint32_t begin, uint32_t deg,
                                          double v, uint32_t& target, uint32_t& sign) {
    const uint4* e = reinterpret_cast<const uint4*>(edges + begin);
    if (deg <= 4u) {
        const uint4 z = make_uint4(0u, 0x7FF00000u, 0u, 0u);  // cdf = +inf, never <= v
        const uint4 r0 = __ldg(e);
        const uint4 r1 = deg > 1u ? __ldg(e + 1) : z;
        const uint4 r2 = deg > 2u ? __ldg(e + 2) : z;
        const uint4 r3 = deg > 3u ? __ldg(e + 3) : z;
        uint32_t c = (edge_cdf(r0) <= v) + (edge_cdf(r1) <= v) + (edge_cdf(r2) <= v) + (edge_cdf(r3) <= v);
        c = c < deg - 1u ? c : deg - 1u;
        const uint4 r = c == 0u ? r0 : c == 1u ? r1 : c == 2u ? r2 : r3;
        target = r.z;
        sign = r.w;
        return;
    }
    uint32_t lo = 0, count = deg;
    while (count > 0u) {
        const uint32_t step = count >> 1;
        const uint32_t it = lo + step;
        const double c = __ldg(reinterpret_cast<const double*>(edges + begin + it));
        if (!(v < c)) {
            lo = it + 1u;
            count -= step + 1u;
        } else {
            count = step;
        }
    }
    const uint32_t k = lo < deg - 1u ? lo : deg - 1u;
    const uint4 r = __ldg(e + k);
    target = r.z;
    sign = r.w;
}

// ----------------------------------------------------------------------------- walker
// Per-item constants (uniform across the warp while it works on one chunk).
struct ItemConst {
    uint64_t seed;
    uint64_t nsteps;
    double dt;
    double half_dt;  // dt_ * 0.5, the left factor of paths.cpp:110
    double qdt_entry;
    Row entry_row;
    uint32_t entry;
    uint32_t key3;
    uint32_t base;
};

struct Walker {
    Stream st;
    Row cur;               // row record of the current state
    uint32_t state;
    uint32_t qstate;       // state whose step-start threshold is cached in qdt
    int32_t sign;
    uint32_t half;         // coupled: 0 before the pair's middle node, 1 after
    double remaining;      // time left in the current fine step
    double q;              // no-jump threshold for the current holding interval
    double qdt;            // -expm1(-rate[qstate] * dt), the LevelSampler nojump_ entry
    double acc_a, acc_b;   // single: expo; coupled: coarse, delta
    double d0, d1;         // d[s0], d[s1]
    uint64_t step;         // completed fine steps
    uint64_t draws, jumps;
};

__device__ __forceinline__ void walker_start(Walker& w, const ItemConst& ic, uint64_t sample) {
    stream_init(w.st, ic.seed, sample, ic.key3);
    w.cur = ic.entry_row;
    w.state = ic.entry;
    w.qstate = ic.entry;
    w.sign = 1;
    w.half = 0;
    w.remaining = ic.dt;
    w.q = ic.qdt_entry;
    w.qdt = ic.qdt_entry;
    w.acc_a = 0.0;
    w.acc_b = 0.0;
    w.d0 = ic.entry_row.d;
    w.d1 = 0.0;
    w.step = 0;
    w.draws = 0;
    w.jumps = 0;
}

// One event of the path: one pass of evolve_common's for(;;) body, plus the step
// bookkeeping of single/coupled when the holding interval ends the fine step.
// Returns true when the sample's last fine step has completed.
__device__ __forceinline__ bool walker_event(Walker& w, const ItemConst& ic, const RowRec* __restrict__ rows,
                                             const EdgeRec* __restrict__ edges) {
    bool step_done = true;
    if (w.cur.rate != 0.0) {  // rate == 0: absorbing row, holding time +inf (paths.cpp:50)
        const double u = next_uniform(w.st);
        ++w.draws;
        if (u < w.q) {  // u >= q: holding time exceeds the rest of the interval (paths.cpp:53)
            // remaining -= -log1p(-u) / rate                                  paths.cpp:54
            w.remaining = __dsub_rn(w.remaining, __ddiv_rn(-log1p(-u), w.cur.rate));
            ++w.jumps;
            const double v = next_uniform(w.st);
            uint32_t target, sgn;
            pick_edge(edges, w.cur.begin, w.cur.deg, v, target, sgn);
            if (sgn) w.sign = -w.sign;
            w.state = target;
            w.cur = load_row(rows, target);
            if (w.remaining > 0.0) {  // else: rounding pushed past the boundary (paths.cpp:67)
                w.q = -expm1(__dmul_rn(-w.cur.rate, w.remaining));  // paths.cpp:68
                step_done = false;
            }
        }
    }
    if (!step_done) return false;

    // ---- the fine step ended in w.state
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
    if (++w.step == ic.nsteps) return true;
    // next fine step: fresh holding interval of length dt with q = nojump_[state] (paths.cpp:95-96)
    w.remaining = ic.dt;
    if (w.state != w.qstate) {
        w.qdt = -expm1(__dmul_rn(-w.cur.rate, ic.dt));  // paths.cpp:90
        w.qstate = w.state;
    }
    w.q = w.qdt;
    return false;
}

// Terminal values: single -> (sign * e^expo) * u[end] (paths.cpp:112);
// coupled -> uf = sign * u[end]; (uf e^{coarse+delta}, uf e^{coarse}) (paths.cpp:138-140).
__device__ __forceinline__ void walker_finish(const Walker& w, const ItemConst& ic, double& fine,
                                              double& coarse) {
    const double sg = static_cast<double>(w.sign);
    if (ic.base) {
        fine = __dmul_rn(__dmul_rn(sg, exp(w.acc_a)), w.cur.u);
        coarse = 0.0;
    } else {
        const double uf = __dmul_rn(sg, w.cur.u);
        fine = __dmul_rn(uf, exp(__dadd_rn(w.acc_a, w.acc_b)));
        coarse = __dmul_rn(uf, exp(w.acc_a));
    }
}

__device__ __forceinline__ ItemConst load_item(const DevItem* __restrict__ items, uint32_t i,
                                               const RowRec* __restrict__ rows) {
    const DevItem it = items[i];
    ItemConst ic;
    ic.seed = it.seed;
    ic.nsteps = it.nsteps;
    ic.dt = it.dt;
    ic.half_dt = __dmul_rn(it.dt, 0.5);
    ic.entry = it.entry;
    ic.key3 = it.key3;
    ic.base = it.base;
    ic.entry_row = load_row(rows, it.entry);
    ic.qdt_entry = -expm1(__dmul_rn(-ic.entry_row.rate, it.dt));
    return ic;
}

}  // namespace expmc_b200
