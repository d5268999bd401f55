// Host check of the two holding-test rewrites (same fp64 sequences as the device code, division
// and exp from the host libm, which the device matches to <= 1 ulp):
//  (1) walker.cuh S-mode: the reference decides each event by u < q, q = -expm1(-rate*remaining),
//      and spends E = -log1p(-u) on a jump (paths.cpp:44-71).  S-mode tracks S = e^{-rate*rem}
//      2^53 and decides 1 - u > S, S <- S / (1 - u).  Simulates many steps of random rows both
//      ways from the same draws and counts decision mismatches (expected: none; a mismatch
//      needs u within a few ulps of the threshold, probability ~1e-16 per event).
//  (2) ed_walker.cuh closed-form first hold: for M = 2^53 - K < m_safe the full event
//      (E = -fast_log(M 2^-53), tjump = E / rate) must say "no jump before tend".
// Prints "mismatches events hold_violations hold_checks".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>

#include "fastmath.cuh"

using namespace expmc_b200;

static const LogEntry kTable[128] = {
#include "log_table.inc"
};
static const double kPoly[9] = EXPMC_LOG_POLY;

int main(int argc, char** argv) {
    const long steps = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 g(2024);
    std::uniform_real_distribution<double> rr(0.05, 8.0), dd(1e-3, 1.0);
    long mism = 0, events = 0;
    for (long s = 0; s < steps; ++s) {
        const double rate = rr(g), dt = dd(g);
        // reference: remaining in time space, expm1 / log1p as paths.cpp
        double rem = dt;
        double S = std::exp(-rate * dt) * 0x1.0p53;  // S-mode, scaled
        for (;;) {
            const uint64_t k = g() >> 11;
            const double u = static_cast<double>(k) * 0x1.0p-53;
            const double m = static_cast<double>((uint64_t{1} << 53) - k);
            const double q = -std::expm1(-rate * rem);
            const bool jr = u < q;
            const bool js = m > S;
            ++events;
            if (jr != js) { ++mism; break; }
            if (!jr) break;
            rem -= -std::log1p(-u) / rate;
            S = S * 0x1.0p53 / m;
            if (!(rem > 0.0)) break;
        }
    }
    long viol = 0, checks = 0;
    std::uniform_real_distribution<double> lr(-12.0, 4.0);
    for (long i = 0; i < steps; ++i) {
        const double rate = std::pow(10.0, lr(g)), tend = std::pow(10.0, lr(g) / 2);
        const double m = std::exp(-(rate * tend)) * 0x1.0p53 * (1.0 - 0x1.0p-30);
        if (!(m >= 2.0)) continue;
        const uint64_t ms = static_cast<uint64_t>(m);
        for (uint64_t M : {ms - 1, ms - 2, ms / 2 + 1, uint64_t{1}}) {
            if (M == 0 || M >= ms) continue;
            const double e = -fast_log(static_cast<double>(M), -53, kTable, kPoly);
            const double tj = e / rate;
            ++checks;
            if (tj < tend) ++viol;
        }
    }
    std::printf("%ld %ld %ld %ld\n", mism, events, viol, checks);
    return 0;
}
