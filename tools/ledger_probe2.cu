// Microbenchmark of the env step's buy pass on recorded steady-state ledger states (exp/dump_state.py:
// 8 steps x 32 envs of the C3 workload after the sell pass), one warp per launch, clock64 around the pass.
// Variants: 0 = per-ticker 5-op chain (round-1 kernel), 1 = affordability rounds (hits only), others below.
// Every variant's cash and holdings must equal variant 0's bit for bit.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/lp2 tools/ledger_probe2.cu
//   /tmp/lp2 exp/ledger_states.bin
#include <cuda_runtime.h>

#include <cstdint>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int NT = 100;
constexpr int CH = 16;
constexpr long long FR_LO = 0x3DD0000000000000ll, FR_HI = 0x3FEFFFFFFFF80000ll;

struct Rec {
    double unit[NT];
    short a[NT * 32];
    int h[NT * 32];
    double cash[32];
};

__device__ __forceinline__ void exact_fix(double cash_b, double unit, double ad, double& qd, double& cash) {
    double qmax = floor(__ddiv_rn(cash_b, unit));
    if (__dmul_rn(qmax, unit) > cash_b) qmax = __dadd_rn(qmax, -1.0);
    qd = ad < qmax ? ad : qmax;
    qd = qd < 0.0 ? 0.0 : qd;
    cash = __dadd_rn(cash_b, -__dmul_rn(qd, unit));
}

template <int V>
__global__ void probe(const Rec* recs, int nrec, double* cash_out, int* hold_out, long long* cyc, int w2) {
    // warp 0 and (when w2 > 0) warp w2 each run the pass on their own copy of the data; other warps exit
    __shared__ int hold_all[2][NT * 32];
    __shared__ short aint_all[2][NT * 32];
    __shared__ double unit_s[NT], rcp_s[NT];
    __shared__ float unit_f[NT];
    const int wid = threadIdx.x >> 5;
    if (wid != 0 && wid != w2) return;
    const int me = wid == 0 ? 0 : 1;
    int* hold_s = hold_all[me];
    short* aint_s = aint_all[me];
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < nrec; ++r) {
        const Rec& R = recs[r];
        if (me == 0) for (int i = lane; i < NT; i += 32) {
            unit_s[i] = R.unit[i];
            rcp_s[i] = __ddiv_rn(1.0, R.unit[i]);
            unit_f[i] = __double2float_rd(R.unit[i]);
        }
        for (int i = lane; i < NT * 32; i += 32) {
            hold_s[i] = R.h[i];
            aint_s[i] = R.a[i];
        }
        __syncthreads();
        double cash = R.cash[lane];
        const int n = NT;
        const int nch = (n + CH - 1) / CH;
        if (V != 0)   // post-sell holdings (variant 0 forms them inside its loop; the kernel in the trailing warps)
            for (int i = 0; i < n; ++i) {
                const int ai = aint_s[i * 32 + lane];
                if (ai < 0) hold_s[i * 32 + lane] -= min(hold_s[i * 32 + lane], -ai);
            }
        __syncwarp();
        int rounds = 0;
        long long t0 = clock64();
        if (V == 0) {
            for (int c = 0; c < nch; ++c) {
                const int i0 = c * CH, i1 = min(i0 + CH, n);
                const double cash_c0 = cash;
                bool unsure = false;
                int ai_n = aint_s[i0 * 32 + lane], h_n = hold_s[i0 * 32 + lane];
                double un_n = unit_s[i0], rc_n = rcp_s[i0];
#pragma unroll 8
                for (int i = i0; i < i1; ++i) {
                    const int ai = ai_n;
                    int h = h_n;
                    const double unit = un_n, rcp = rc_n;
                    if (i + 1 < i1) {
                        ai_n = aint_s[(i + 1) * 32 + lane];
                        h_n = hold_s[(i + 1) * 32 + lane];
                        un_n = unit_s[i + 1];
                        rc_n = rcp_s[i + 1];
                    }
                    if (ai < 0) h -= min(h, -ai);
                    const double ad = static_cast<double>(ai > 0 ? ai : 0);
                    const double y = __dmul_rn(cash, rcp);
                    const double fl = floor(y);
                    const double qd = fl < ad ? fl : ad;
                    const double cost = __dmul_rn(qd, unit);
                    const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                    unsure |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                                (frb >= FR_LO && frb <= FR_HI));
                    h += static_cast<int>(qd);
                    cash = __dadd_rn(cash, -cost);
                    hold_s[i * 32 + lane] = h;
                }
                if (__any_sync(0xffffffffu, unsure)) cash = cash_c0 - 1e300;   // (never on this data)
            }
        } else {
            for (int c = 0; c < nch; ++c) {
                const int i0 = c * CH;
                uint32_t cm = 0;
#pragma unroll
                for (int k = 0; k < CH; ++k) cm |= (i0 + k < n && aint_s[min(i0 + k, n - 1) * 32 + lane] > 0 ? 1u : 0u) << k;
                double uc[CH];   // V3: the chunk's unit prices in registers
                float ucf[CH];   // V4: rounded down to float32
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    if (V == 3) uc[k] = unit_s[min(i0 + k, n - 1)];
                    if (V == 4) ucf[k] = unit_f[min(i0 + k, n - 1)];
                }
                long long ub[CH];   // V5: the chunk's unit prices as (monotone) int64 bit patterns
#pragma unroll
                for (int k = 0; k < CH; ++k)
                    if (V == 5) ub[k] = __double_as_longlong(unit_s[min(i0 + k, n - 1)]);
                auto affordable = [&](double b_now) {
                    if (V == 5) {
                        const long long cb = __double_as_longlong(b_now);
                        uint32_t bit[CH];
#pragma unroll
                        for (int k = 0; k < CH; ++k) bit[k] = ub[k] <= cb ? (1u << k) : 0u;
#pragma unroll
                        for (int st = 1; st < CH; st *= 2)
#pragma unroll
                            for (int k = 0; k + st < CH; k += 2 * st) bit[k] |= bit[k + st];
                        return bit[0];
                    }
                    if (V == 3 || V == 4) {
                        const float bf = __double2float_ru(b_now);
                        uint32_t bit[CH];
#pragma unroll
                        for (int k = 0; k < CH; ++k)
                            bit[k] = (V == 3 ? uc[k] <= b_now : ucf[k] <= bf) ? (1u << k) : 0u;
#pragma unroll
                        for (int st = 1; st < CH; st *= 2)
#pragma unroll
                            for (int k = 0; k + st < CH; k += 2 * st) bit[k] |= bit[k + st];
                        return bit[0];
                    }
                    if (V == 1 || V == 6) {
                        uint32_t bit[CH];
#pragma unroll
                        for (int k = 0; k < CH; ++k) bit[k] = unit_s[min(i0 + k, n - 1)] <= b_now ? (1u << k) : 0u;
#pragma unroll
                        for (int st = 1; st < CH; st *= 2)
#pragma unroll
                            for (int k = 0; k + st < CH; k += 2 * st) bit[k] |= bit[k + st];
                        return bit[0];
                    } else {
                        // V2: float32 filter (unit rounded down): unit_f <= b_f is necessary for unit <= b
                        const float bf = __double2float_ru(b_now);
                        uint32_t bit[CH];
#pragma unroll
                        for (int k = 0; k < CH; ++k) bit[k] = unit_f[min(i0 + k, n - 1)] <= bf ? (1u << k) : 0u;
#pragma unroll
                        for (int st = 1; st < CH; st *= 2)
#pragma unroll
                            for (int k = 0; k + st < CH; k += 2 * st) bit[k] |= bit[k + st];
                        return bit[0];
                    }
                };
                uint32_t aff = affordable(cash);
                while (V == 6) {   // predicated round: every lane runs the hit code, lanes without a hit discard it
                    const uint32_t hits = cm & aff;
                    if (!__any_sync(0xffffffffu, hits != 0u)) break;
                    ++rounds;
                    const bool has = hits != 0u;
                    const int k = has ? __ffs(static_cast<int>(hits)) - 1 : 0;
                    const int i = i0 + k;
                    const double unit = unit_s[i];
                    const double rcp = rcp_s[i];
                    const int ai = aint_s[i * 32 + lane];
                    const int h = hold_s[i * 32 + lane];
                    const double ad = static_cast<double>(ai);
                    const double cash_b = cash;
                    const double y = __dmul_rn(cash, rcp);
                    const double fl = floor(y);
                    double qd = fl < ad ? fl : ad;
                    const double cost = __dmul_rn(qd, unit);
                    const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                    const bool unsure =
                        has && !(__double_as_longlong(fl) > __double_as_longlong(ad) || (frb >= FR_LO && frb <= FR_HI));
                    const double cn = __dadd_rn(cash, -cost);
                    cash = has ? cn : cash;
                    if (__any_sync(0xffffffffu, unsure)) {
                        if (unsure) exact_fix(cash_b, unit, ad, qd, cash);
                    }
                    if (has) {
                        hold_s[i * 32 + lane] = h + static_cast<int>(qd);
                        cm &= ~((2u << k) - 1u);
                    }
                    aff = affordable(cash);
                }
                int hu[CH];   // V7: high words of the chunk's unit prices (a necessary test: hi(unit) <= hi(b))
#pragma unroll
                for (int k = 0; k < CH; ++k) hu[k] = (V == 7) ? __double2hiint(unit_s[min(i0 + k, n - 1)]) : 0;
                auto aff_hi = [&](double b_now) {
                    const int hc = __double2hiint(b_now);
                    uint32_t bit[CH];
#pragma unroll
                    for (int k = 0; k < CH; ++k) bit[k] = (hu[k] <= hc) ? (1u << k) : 0u;
#pragma unroll
                    for (int st = 1; st < CH; st *= 2)
#pragma unroll
                        for (int k = 0; k + st < CH; k += 2 * st) bit[k] |= bit[k + st];
                    return bit[0];
                };
                if (V == 7) aff = aff_hi(cash);
                while (V == 7) {   // predicated rounds, integer affordability filter, floor by the 2^52 trick
                    const uint32_t hits = cm & aff;
                    if (!__any_sync(0xffffffffu, hits != 0u)) break;
                    ++rounds;
                    const bool has = hits != 0u;
                    const int k = has ? __ffs(static_cast<int>(hits)) - 1 : 0;
                    const int i = i0 + k;
                    const double unit = unit_s[i];
                    const double rcp = rcp_s[i];
                    const int ai = aint_s[i * 32 + lane];
                    const int h = hold_s[i * 32 + lane];
                    const double ad = static_cast<double>(ai);
                    const double cost_a = __dmul_rn(ad, unit);
                    const double cash_b = cash;
                    const double y = __dmul_rn(cash, rcp);
                    const double t52 = __dadd_rd(y, 4503599627370496.0);   // 2^52 + floor(y), exactly (0 <= y < 2^52)
                    const int m = __double2loint(t52);                      // floor(y)
                    const double fl = __dadd_rn(t52, -4503599627370496.0);
                    const bool clip = m < ai;
                    const double cost = clip ? __dmul_rn(fl, unit) : cost_a;
                    const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                    const bool unsure = has && !(m > ai || (frb >= FR_LO && frb <= FR_HI));
                    const double cn = __dadd_rn(cash, -cost);
                    cash = has ? cn : cash;
                    int q = clip ? m : ai;
                    if (__any_sync(0xffffffffu, unsure)) {
                        if (unsure) {
                            double qd;
                            exact_fix(cash_b, unit, ad, qd, cash);
                            q = static_cast<int>(qd);
                        }
                    }
                    if (has) {
                        hold_s[i * 32 + lane] = h + q;
                        cm &= ~((2u << k) - 1u);
                    }
                    aff = aff_hi(cash);
                }
                while (V != 6 && V != 7) {
                    uint32_t hits = cm & aff;
                    if (!__any_sync(0xffffffffu, hits != 0u)) break;
                    ++rounds;
                    if (hits) {
                        const int k = __ffs(static_cast<int>(hits)) - 1;
                        const int i = i0 + k;
                        cm &= ~((2u << k) - 1u);
                        const double unit = unit_s[i];
                        const int ai = aint_s[i * 32 + lane];
                        const int h = hold_s[i * 32 + lane];
                        if (V == 2 && !(unit <= cash)) {   // filtered candidate not affordable: q = 0
                            aff &= ~(1u << k);
                            continue;
                        }
                        if (V == 4 && !(unit <= cash)) {   // float filter passed, exact compare failed: q = 0
                            aff = affordable(cash) & ~((2u << k) - 1u);
                            continue;
                        }
                        const double ad = static_cast<double>(ai);
                        const double cash_b = cash;
                        const double y = __dmul_rn(cash, rcp_s[i]);
                        const double fl = floor(y);
                        double qd = fl < ad ? fl : ad;
                        double cost;
                        if (V == 5) {   // both candidate costs, selected after the products (off the compare)
                            const double cost_m = __dmul_rn(fl, unit), cost_a = __dmul_rn(ad, unit);
                            cost = fl < ad ? cost_m : cost_a;
                        } else {
                            cost = __dmul_rn(qd, unit);
                        }
                        const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                        const bool unsure =
                            !(__double_as_longlong(fl) > __double_as_longlong(ad) || (frb >= FR_LO && frb <= FR_HI));
                        cash = __dadd_rn(cash, -cost);
                        if (unsure) exact_fix(cash_b, unit, ad, qd, cash);
                        hold_s[i * 32 + lane] = h + static_cast<int>(qd);
                        aff = affordable(cash);
                    }
                }
            }
        }
        long long t1 = clock64();
        __syncwarp();
        if (me == 0) {
            cash_out[r * 32 + lane] = cash;
            for (int i = 0; i < n; ++i) hold_out[(r * NT + i) * 32 + lane] = hold_s[i * 32 + lane];
            if (lane == 0) cyc[r] = (t1 - t0) * 1000 + rounds;
        }
        __syncthreads();
    }
}

int main(int argc, char** argv) {
    FILE* f = fopen(argc > 1 ? argv[1] : "exp/ledger_states.bin", "rb");
    if (!f) { printf("no states\n"); return 1; }
    std::vector<Rec> recs;
    Rec r;
    while (fread(r.unit, 8, NT, f) == NT && fread(r.a, 2, NT * 32, f) == NT * 32 && fread(r.h, 4, NT * 32, f) == NT * 32 &&
           fread(r.cash, 8, 32, f) == 32)
        recs.push_back(r);
    fclose(f);
    const int nr = static_cast<int>(recs.size());
    Rec* d;
    cudaMalloc(&d, sizeof(Rec) * nr);
    cudaMemcpy(d, recs.data(), sizeof(Rec) * nr, cudaMemcpyHostToDevice);
    double* dc;
    int* dh;
    long long* dcy;
    cudaMalloc(&dc, 8 * 32 * nr);
    cudaMalloc(&dh, 4 * NT * 32 * nr);
    cudaMalloc(&dcy, 8 * nr);
    std::vector<double> c0(32 * nr), c1(32 * nr);
    std::vector<int> h0(NT * 32 * nr), h1(NT * 32 * nr);
    std::vector<long long> cy(nr);
    void (*ks[])(const Rec*, int, double*, int*, long long*, int) = {probe<0>, probe<1>, probe<2>, probe<3>, probe<4>, probe<5>, probe<6>, probe<7>};
    for (int v = 0; v < 8; ++v) {
        const int w2 = argc > 2 ? atoi(argv[2]) : 0;
        for (int rep = 0; rep < 3; ++rep) ks[v]<<<1, 32 * (w2 + 1)>>>(d, nr, dc, dh, dcy, w2);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(v ? c1.data() : c0.data(), dc, 8 * 32 * nr, cudaMemcpyDeviceToHost);
        cudaMemcpy(v ? h1.data() : h0.data(), dh, 4 * NT * 32 * nr, cudaMemcpyDeviceToHost);
        cudaMemcpy(cy.data(), dcy, 8 * nr, cudaMemcpyDeviceToHost);
        bool same = true;
        if (v) same = !memcmp(c0.data(), c1.data(), 8 * 32 * nr) && !memcmp(h0.data(), h1.data(), 4 * NT * 32 * nr);
        printf("variant %d: cycles per pass", v);
        long long s = 0;
        for (int i = 0; i < nr; ++i) { printf(" %lld(%lld)", cy[i] / 1000, cy[i] % 1000); s += cy[i] / 1000; }
        printf("  mean %lld  %s\n", s / nr, v ? (same ? "bit-identical" : "MISMATCH") : "(reference)");
    }
    return 0;
}
