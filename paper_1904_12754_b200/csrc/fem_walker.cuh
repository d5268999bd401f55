// fem mode (lane 2): the inhomogeneous sampler of the lumped-mass FEM system
// M u' = -K u + F, run on the chain of -M^{-1}K with load g = M^{-1}F (solve_convdiff_point,
// fem.cpp:51-73).  Each path carries, besides the homogeneous functional, the Duhamel integral
// of the load along its fine nodes with composite-Simpson weights:
//
//   fem_single   (paths.cpp:183-203):  integ += w_j sign e^{expo_j} g[state_j] at every fine
//                                      node; value = sign e^{expo} u[end] + integ
//   fem_coupled  (paths.cpp:205-245):  fine nodes 2m+1 (pair middle) and 2m+2 (pair end) on
//                                      the fine rule, nodes m+1 on the coarse rule; the run_level
//                                      sample is u[end] (eta_f - eta_c) + (integ_f - integ_c) and
//                                      integ_f - integ_c also feeds the SumAcc side channel
//                                      `extra` (mlmc.cpp:126-133, parallel.hpp:60)
//
// The draws, jumps and exponents are the reference-order walker's (walker_hold is shared with
// entry mode, so quadrature consumes no draws -- test_paths.cpp:325-358); the node weights are
// run_level_ex's scaled_simpson (mlmc.cpp:66-75): h * {1, 4, 2, ..., 4, 1}, h = step / 3.
// Every expression keeps the reference's evaluation order under explicit __d*_rn.
#pragma once

#include "ed_walker.cuh"
#include "walker.cuh"

#ifndef EXPMC_FEM_MINB
#define EXPMC_FEM_MINB 3  // three 256-thread blocks per SM: 80 registers for the quadrature state
#endif

namespace expmc_b200 {

struct FemWalker {
    Walker w;
    double integ_f, integ_c;
    double e0, e1;  // the last node's exponentials: base e^{expo}; coupled e^{coarse+delta}, e^{coarse}
};

// scaled_simpson weight of node j on a rule of `panels` panels with scale h (mlmc.cpp:66-75).
__device__ __forceinline__ double simpson_weight(uint64_t j, uint64_t panels, double h) {
    const double c = (j == 0 || j == panels) ? 1.0 : ((j & 1u) ? 4.0 : 2.0);
    return __dmul_rn(h, c);
}

__device__ __forceinline__ void fem_start(FemWalker& f, const ItemConst& ic, const double* __restrict__ load,
                                          const RowRec* __restrict__ rows, uint64_t sample) {
    walker_start<false>(f.w, ic, LaneData{nullptr, 0.0, 0u, nullptr, nullptr, 0u}, rows, sample);
    const double g0 = __ldg(load + ic.entry);
    f.integ_f = __dmul_rn(ic.h_fine, g0);    // fine_w[0] * load[entry]            paths.cpp:195, 223
    f.integ_c = __dmul_rn(ic.h_coarse, g0);  // coarse_w[0] * load[entry]          paths.cpp:224
    f.e0 = f.e1 = 1.0;
}

// One event; at a fine node the quadrature terms.  The node's one or two exponentials go
// through a single exp call site (a two-trip loop), and the terminal values reuse the last
// node's: no exp at the end of a sample.
__device__ __forceinline__ bool fem_event(FemWalker& f, const ItemConst& ic, const double* __restrict__ load,
                                          const RowRec* __restrict__ rows, const EdgeTables& edges,
                                          const LogEntry* s_log, unsigned long long& draws,
                                          unsigned long long& jumps) {
    Walker& w = f.w;
    if (!walker_hold(w, rows, edges, s_log, draws, jumps)) return false;
    const double dn = w.cur.d;
    const uint64_t j = ic.nsteps - w.left + 1;  // fine node index of the step that just ended
    // exponents of this node
    //   base:      expo += dt_ * 0.5 * (d[s0] + d[state])                       paths.cpp:198
    //   pair mid:  mid = coarse + delta + dt_ * 0.5 * (d[s0] + d[s1])          paths.cpp:230
    //   pair end:  coarse += dt (d0 + d2); delta += dt (d1 - 0.5 (d0 + d2))    paths.cpp:234-236
    double x0, x1 = 0.0;
    int nexp = 1;
    const bool mid = !ic.base && w.half == 0u;
    if (ic.base) {
        w.acc_a = __dadd_rn(w.acc_a, __dmul_rn(ic.half_dt, __dadd_rn(w.d0, dn)));
        x0 = w.acc_a;
        w.d0 = dn;
    } else if (mid) {
        w.d1 = dn;
        w.half = 1u;
        x0 = __dadd_rn(__dadd_rn(w.acc_a, w.acc_b), __dmul_rn(ic.half_dt, __dadd_rn(w.d0, dn)));
    } else {
        const double s02 = __dadd_rn(w.d0, dn);
        const double half_ends = __dmul_rn(0.5, s02);
        w.acc_a = __dadd_rn(w.acc_a, __dmul_rn(ic.dt, s02));
        w.acc_b = __dadd_rn(w.acc_b, __dmul_rn(ic.dt, __dsub_rn(w.d1, half_ends)));
        w.d0 = dn;
        w.half = 0u;
        x0 = __dadd_rn(w.acc_a, w.acc_b);
        x1 = w.acc_a;
        nexp = 2;
    }
    double e[2];
#pragma unroll 1
    for (int k = 0; k < nexp; ++k) e[k] = dexp(k == 0 ? x0 : x1);
    const double sg = static_cast<double>(w.sign);
    const double g = __ldg(load + w.state);
    if (nexp == 1) {
        // integ += fine_w[j] * sign * exp(x) * load[state]                  paths.cpp:199-200, 231-232
        f.integ_f = __dadd_rn(f.integ_f, __dmul_rn(__dmul_rn(__dmul_rn(simpson_weight(j, ic.nsteps, ic.h_fine), sg),
                                                             e[0]), g));
        if (ic.base) f.e0 = e[0];
    } else {
        // eta_f = sign e^{coarse+delta}, eta_c = sign e^{coarse};
        // integ_f += fine_w[2m+2] eta_f g; integ_c += coarse_w[m+1] eta_c g     paths.cpp:237-242
        const double eta_f = __dmul_rn(sg, e[0]);
        const double eta_c = __dmul_rn(sg, e[1]);
        f.integ_f = __dadd_rn(f.integ_f, __dmul_rn(__dmul_rn(simpson_weight(j, ic.nsteps, ic.h_fine), eta_f), g));
        f.integ_c = __dadd_rn(f.integ_c,
                              __dmul_rn(__dmul_rn(simpson_weight(j >> 1, ic.nsteps >> 1, ic.h_coarse), eta_c), g));
        f.e0 = e[0];
        f.e1 = e[1];
    }
    if (--w.left == 0) return true;
    set_hold(w, fresh_hold(ic, w.cur.rate));
    return false;
}

// Terminal values.  base: value = sign e^{expo} u[end] + integ (paths.cpp:202); coupled:
// eta_f / eta_c of the last pair (the sign has not changed since), x = u[end] (eta_f - eta_c) +
// (integ_f - integ_c), extra = integ_f - integ_c (mlmc.cpp:126-133).
__device__ __forceinline__ double fem_finish(const FemWalker& f, const ItemConst& ic, const RowRec* __restrict__ rows,
                                             double& eta_f, double& eta_c, double& extra) {
    const Walker& w = f.w;
    const double sg = static_cast<double>(w.sign);
    const double u_end = __ldg(&rows[w.state].u);
    if (ic.base) {
        eta_f = eta_c = 0.0;
        extra = 0.0;
        return __dadd_rn(__dmul_rn(__dmul_rn(sg, f.e0), u_end), f.integ_f);
    }
    eta_f = __dmul_rn(sg, f.e0);
    eta_c = __dmul_rn(sg, f.e1);
    const double du = __dmul_rn(u_end, __dsub_rn(eta_f, eta_c));
    extra = __dsub_rn(f.integ_f, f.integ_c);
    return __dadd_rn(du, extra);
}

// Chunk-kernel policy of fem batches (always reference-order: every fine node costs an exp, so
// the event-driven sampler has nothing to skip).
struct FemPolicy {
    using W = FemWalker;
    static constexpr bool kDefer = false;
    static constexpr bool kExtra = true;
    static constexpr bool kScreen = false;
    static __device__ __forceinline__ bool screen(const ItemConst&, uint64_t) { return false; }
    static constexpr int kMinBlocks = EXPMC_FEM_MINB;
    static __device__ __forceinline__ void prepare(ItemConst& ic, const RowRec* rows, const LaneData&, uint32_t flags) {
        prepare_hold(ic, rows, flags);
        ic.h_fine = __ddiv_rn(ic.dt, 3.0);  // scaled_simpson's h = step / 3 (mlmc.cpp:68)
        ic.h_coarse = __ddiv_rn(__dmul_rn(2.0, ic.dt), 3.0);
    }
    static __device__ __forceinline__ void start(W& f, const ItemConst& ic, const LaneData& ld, const RowRec* rows,
                                                 uint64_t s) {
        fem_start(f, ic, ld.load, rows, s);
    }
    static __device__ __forceinline__ bool event(W& f, const ItemConst& ic, const LaneData& ld, const RowRec* rows,
                                                 const EdgeTables& e, const LogEntry* lg, unsigned long long& dr,
                                                 unsigned long long& j) {
        return fem_event(f, ic, ld.load, rows, e, lg, dr, j);
    }
    static __device__ __forceinline__ double sample(const W& f, const ItemConst& ic, const LaneData&,
                                                    const RowRec* rows, double& extra) {
        double ef, ec;
        return fem_finish(f, ic, rows, ef, ec, extra);
    }
    static __device__ __forceinline__ void record(const W& f, const ItemConst& ic, const LaneData&,
                                                  const RowRec* rows, SampleOut& o) {
        double extra;
        o.value = fem_finish(f, ic, rows, o.fine, o.coarse, extra);
        if (ic.base) o.fine = o.value;
        o.integ_f = f.integ_f;
        o.integ_c = f.integ_c;
        o.end_state = f.w.state;
    }
};

}  // namespace expmc_b200
