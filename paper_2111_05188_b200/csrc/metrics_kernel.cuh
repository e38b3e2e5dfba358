// metrics_kernel.cuh — evaluator backtest metrics of account-value curves.
//
// Method (§5.2 evaluation metrics; reading R#25), per env, float64:
//   rho_t = v_t / v_{t-1} - 1 (t = 1..T);  cumulative return (v_T - v_0) / v_0;
//   annual return (v_T / v_0)^(ppy / T) - 1;  annual volatility std_{n-1}(rho) sqrt(ppy);
//   Sharpe (mean(rho) - rf) / std_{n-1}(rho) sqrt(ppy) (NaN when std = 0 or T < 2);
//   max drawdown min_t (v_t / max_{s<=t} v_s - 1).
// B200 mapping: lane = env (coalesced rows of the time-major curve), two sequential passes over T
// (mean, then the centred sum of squares, as the definition reads); HBM-bound and tiny next to the
// rollout that produced the curve.
#pragma once
#include <cstdint>

namespace pod {

__global__ void __launch_bounds__(128) backtest_metrics_kernel(const double* __restrict__ v0,
                                                               const double* __restrict__ curve, int T, int N,
                                                               double ppy, double rf, double* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N) return;
    const double first = v0[e];
    double prev = first, peak = first, mdd = 0.0, s1 = 0.0;
    for (int t = 0; t < T; ++t) {
        const double v = curve[static_cast<int64_t>(t) * N + e];
        s1 = s1 + (v / prev - 1.0);
        peak = peak > v ? peak : v;
        const double dd = v / peak - 1.0;
        mdd = dd < mdd ? dd : mdd;
        prev = v;
    }
    const double last = prev;
    const double mean = s1 / T;
    double ss = 0.0;
    prev = first;
    for (int t = 0; t < T; ++t) {
        const double v = curve[static_cast<int64_t>(t) * N + e];
        const double d = (v / prev - 1.0) - mean;
        ss = ss + d * d;
        prev = v;
    }
    const double sd = T > 1 ? sqrt(ss / (T - 1)) : 0.0;
    out[e] = (last - first) / first;
    out[static_cast<int64_t>(N) + e] = pow(last / first, ppy / T) - 1.0;
    out[2 * static_cast<int64_t>(N) + e] = sd * sqrt(ppy);
    out[3 * static_cast<int64_t>(N) + e] = (T > 1 && sd > 0.0) ? (mean - rf) / sd * sqrt(ppy) : __longlong_as_double(0x7FF8000000000000ll);
    out[4 * static_cast<int64_t>(N) + e] = mdd;
}

}  // namespace pod
