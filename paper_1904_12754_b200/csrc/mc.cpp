// Classical (single-level) Monte Carlo front end (mc.hpp / mc.cpp:42-113) over the GPU sampler:
// mc_single_entry, mc_forward_scalar and the pilot-driven mc_auto.  The sampling and the
// Welford reduction run in context.cu (mc_batch -> k_sample<Policy, Welford>).
#include <algorithm>
#include <cmath>

#include "internal.hpp"

using namespace expmc_b200;

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EXPMC_OK;
    } catch (const Status& s) {
        set_error(s.what());
        return s.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return EXPMC_EINTERNAL;
    }
}

}  // namespace

extern "C" {

int expmc_mc_batch(expmc_ctx* ctx, uint32_t lane, int64_t nreq, const expmc_mc_req* req, expmc_mc_result* out) {
    return guarded([&] {
        if (!ctx || nreq < 0 || (nreq > 0 && (!req || !out))) throw Status(EXPMC_EINVAL, "null argument");
        mc_batch(ctx, lane, req, nreq, out);
    });
}

int expmc_mc_single_entry(expmc_ctx* ctx, int64_t entry, double beta, double dt, uint64_t samples, uint64_t seed,
                          expmc_mc_result* out) {
    return guarded([&] {
        if (!ctx || !out) throw Status(EXPMC_EINVAL, "null argument");
        const expmc_mc_req r{entry, seed, samples, beta, dt};
        mc_batch(ctx, EXPMC_LANE_ENTRY, &r, 1, out);
    });
}

int expmc_mc_forward_scalar(expmc_ctx* ctx, double beta, double dt, uint64_t samples, uint64_t seed,
                            expmc_mc_result* out) {
    return guarded([&] {
        if (!ctx || !out) throw Status(EXPMC_EINVAL, "null argument");
        const expmc_mc_req r{0, seed, samples, beta, dt};
        mc_batch(ctx, EXPMC_LANE_FORWARD, &r, 1, out);
    });
}

int expmc_mc_auto(expmc_ctx* ctx, int64_t entry, double beta, double epsilon, uint64_t seed, expmc_mc_result* out) {
    return guarded([&] {
        if (!ctx || !out) throw Status(EXPMC_EINVAL, "null argument");
        if (!(epsilon > 0.0)) throw Status(EXPMC_EINVAL, "epsilon must be positive");
        constexpr uint64_t kPilot = 1000;  // mc.cpp:82
        expmc_ctx_info info{};
        if (expmc_ctx_get_info(ctx, &info) != EXPMC_OK) throw Status(EXPMC_EINVAL, "null context");
        // pilot step sizes (mc.cpp:84-93)
        int ka = 2;
        if (info.d_max > 0.0) {
            const int l0 = static_cast<int>(std::max<long>(0, std::lround(std::log2(2.0 * beta * info.d_max))));
            ka = std::max(ka, l0);
        }
        const double dt_a = beta / static_cast<double>(int64_t{1} << ka);
        const double dt_b = 0.5 * dt_a;
        const expmc_mc_req pilots[2] = {{entry, seed + 1, kPilot, beta, dt_a}, {entry, seed + 2, kPilot, beta, dt_b}};
        expmc_mc_result pr[2];
        mc_batch(ctx, EXPMC_LANE_ENTRY, pilots, 2, pr);  // both pilots in one pass
        // Richardson constant of the O(dt^2) splitting bias and the step count (mc.cpp:95-102)
        const double c = std::abs(pr[0].estimate - pr[1].estimate) / (dt_a * dt_a - dt_b * dt_b);
        int k = 0;
        while (true) {
            const double dt = beta / static_cast<double>(int64_t{1} << k);
            if (c * dt * dt <= epsilon / 2.0) break;
            ++k;
            if (k > 62) throw Status(EXPMC_EOVERFLOW, "epsilon requires more steps than a 64-bit count");
        }
        const double dt = beta / static_cast<double>(int64_t{1} << k);
        // sample count from the finer pilot's variance (mc.cpp:104-107)
        const double pilot_var = pr[1].std_error * pr[1].std_error * static_cast<double>(kPilot);
        const uint64_t m =
            std::max<uint64_t>(2, static_cast<uint64_t>(std::ceil(2.0 * pilot_var / (epsilon * epsilon))));
        const expmc_mc_req fin{entry, seed, m, beta, dt};
        mc_batch(ctx, EXPMC_LANE_ENTRY, &fin, 1, out);
        out->wall_cost += pr[0].wall_cost + pr[1].wall_cost;
    });
}

}  // extern "C"
