// Host check of fastmath.cuh's fast_log (bit-identical to the device path: same fma sequence)
// against a long-double reference.  Prints "max_ulp n_checked"; tests/test_fastmath.py
// compiles and runs it.
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

static double ulp_err(double got, long double exact) {
    const double e = static_cast<double>(exact);
    const double ulp = std::nextafter(std::fabs(e), INFINITY) - std::fabs(e);
    return static_cast<double>(std::fabs(static_cast<long double>(got) - exact) / ulp);
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 2000000;
    std::mt19937_64 g(12345);
    double worst = 0.0, worst_x = 0.0;
    long checked = 0;
    auto check = [&](double x) {
        const double got = fast_log(x, 0, kTable, kPoly);
        const long double ex = logl(static_cast<long double>(x));
        if (x == 1.0) {
            if (got != 0.0) { std::printf("log(1) != 0\n"); std::exit(1); }
            return;
        }
        const double e = ulp_err(got, ex);
        if (e > worst) { worst = e; worst_x = x; }
        ++checked;
    };
    // the sampler's arguments: x = 1 - u, u = k 2^-53 uniform, plus the extremes
    for (long i = 0; i < n; ++i) check(1.0 - static_cast<double>(g() >> 11) * 0x1.0p-53);
    for (long i = 0; i < n / 4; ++i) check(1.0 - static_cast<double>(g() >> 40) * 0x1.0p-53);  // x near 1
    for (long i = 0; i < n / 4; ++i) check(static_cast<double>((g() >> 11) | 1) * 0x1.0p-53);  // x small
    for (int j = 1; j <= 53; ++j) check(std::ldexp(1.0, -j));
    check(1.0);
    check(1.0 - 0x1.0p-53);
    // the sampler's form: log(M 2^-53) with M = 2^53 - K an exact integer must equal log(1 - u)
    for (long i = 0; i < n / 4; ++i) {
        const uint64_t k = g() >> 11;
        const double a = fast_log(static_cast<double>((uint64_t{1} << 53) - k), -53, kTable, kPoly);
        const double b = fast_log(1.0 - static_cast<double>(k) * 0x1.0p-53, 0, kTable, kPoly);
        if (a != b) { std::printf("scaled form differs at K=%llu\n", (unsigned long long)k); std::exit(1); }
    }
    std::printf("%.4f %ld %a\n", worst, checked, worst_x);
    return 0;
}
