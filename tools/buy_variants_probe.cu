// per-ticker buy pass variants: fp64 instruction count vs ALU work (see DESIGN §6 K2)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
constexpr int NT = 100;
constexpr long long FR_LO = 0x3DD0000000000000ll, FR_HI = 0x3FEFFFFFFFF80000ll;
struct Rec { double unit[NT]; short a[NT * 32]; int h[NT * 32]; double cash_after[32]; double p[NT]; double cash0[32]; };

// exact u32 -> double bits on the integer pipe
__device__ __forceinline__ long long u32_f64bits(uint32_t q) {
    if (q == 0) return 0;
    const int e = 31 - __clz(q);
    const unsigned long long mant = (static_cast<unsigned long long>(q) << (52 - e)) & 0xFFFFFFFFFFFFFull;
    return static_cast<long long>((static_cast<unsigned long long>(1023 + e) << 52) | mant);
}

template <int V>
__global__ void probe(const Rec* recs, int nrec, double* out, int* hout, long long* cyc) {
    __shared__ int hold_s[NT * 32];
    __shared__ short aint_s[NT * 32];
    __shared__ double unit_s[NT], rcp_s[NT];
    const int lane = threadIdx.x;
    for (int r = 0; r < nrec; ++r) {
        const Rec& R = recs[r];
        for (int i = lane; i < NT; i += 32) { unit_s[i] = R.unit[i]; rcp_s[i] = __ddiv_rn(1.0, R.unit[i]); }
        for (int i = lane; i < NT * 32; i += 32) { aint_s[i] = R.a[i]; const int a = R.a[i]; hold_s[i] = a < 0 ? R.h[i] - min(R.h[i], -a) : R.h[i]; }
        __syncwarp();
        double cash = R.cash_after[lane];
        bool unsure = false;
        long long t0 = clock64();
        if (V == 0) {
#pragma unroll 8
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                const double unit = unit_s[i], rcp = rcp_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp);
                const double fl = floor(y);
                const double qd = fl < ad ? fl : ad;
                const double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                unsure |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) || (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
            }
        } else if (V == 1) {   // integer compares / min, FRND kept
#pragma unroll 8
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const int ap = ai > 0 ? ai : 0;
                const double unit = unit_s[i], rcp = rcp_s[i];
                const long long adb = u32_f64bits(static_cast<uint32_t>(ap));
                const double y = __dmul_rn(cash, rcp);
                const double fl = floor(y);
                const long long flb = __double_as_longlong(fl);
                const bool clip = flb < adb;
                const double qd = __longlong_as_double(clip ? flb : adb);
                const double cost = __dmul_rn(qd, unit);
                // fr = y - fl >= 2^-34 and <= 1 - 2^-34, from the bits of y (y < 2^31 here, else no clip)
                const long long Y = __double_as_longlong(y);
                const int ex = static_cast<int>(Y >> 52) - 1023;
                bool frok;
                if (ex < 0) {
                    frok = Y >= FR_LO && Y <= FR_HI;
                } else {
                    const int s = 52 - ex;   // fractional bits
                    const long long F = Y & ((1ll << s) - 1);
                    const long long lo = s >= 34 ? (1ll << (s - 34)) : 1ll;
                    const long long hi = s >= 34 ? ((1ll << s) - (1ll << (s - 34))) : ((1ll << s) - 1);
                    frok = F >= lo && F <= hi;
                }
                unsure |= !(ap == 0 || flb > adb || frok);
                if (ap > 0) hold_s[i * 32 + lane] += static_cast<int>(clip ? static_cast<int>(fl) : ap);
                cash = __dadd_rn(cash, -cost);
            }
        } else if (V == 2) {   // floor from the bits of y as well (no FRND): 2 DMUL + 1 DADD per ticker
#pragma unroll 8
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const int ap = ai > 0 ? ai : 0;
                const double unit = unit_s[i], rcp = rcp_s[i];
                const long long adb = u32_f64bits(static_cast<uint32_t>(ap));
                const double y = __dmul_rn(cash, rcp);
                const long long Y = __double_as_longlong(y);
                const int ex = static_cast<int>(Y >> 52) - 1023;
                long long flb;
                int m;
                bool frok;
                if (ex < 0) {
                    flb = 0; m = 0;
                    frok = Y >= FR_LO && Y <= FR_HI;
                } else if (ex >= 31) {   // y >= 2^31 > any action: no clip
                    flb = 0x7FF0000000000000ll; m = 0x7fffffff; frok = true;
                } else {
                    const int s = 52 - ex;
                    const long long fmask = (1ll << s) - 1;
                    const long long F = Y & fmask;
                    flb = Y & ~fmask;
                    m = static_cast<int>(((Y & 0xFFFFFFFFFFFFFll) | (1ll << 52)) >> s);
                    const long long lo = s >= 34 ? (1ll << (s - 34)) : 1ll;
                    const long long hi = s >= 34 ? (fmask + 1 - (1ll << (s - 34))) : fmask;
                    frok = F >= lo && F <= hi;
                }
                const bool clip = m < ap;
                const double qd = __longlong_as_double(clip ? flb : adb);
                const double cost = __dmul_rn(qd, unit);
                unsure |= !(ap == 0 || m > ap || frok);
                if (ap > 0) hold_s[i * 32 + lane] += clip ? m : ap;
                cash = __dadd_rn(cash, -cost);
            }
        }
        long long t1 = clock64();
        if (__any_sync(0xffffffffu, unsure)) cash = -1.0;
        out[r * 32 + lane] = cash;
        for (int i = 0; i < NT; ++i) hout[(r * NT + i) * 32 + lane] = hold_s[i * 32 + lane];
        if (lane == 0) cyc[r] = t1 - t0;
        __syncwarp();
    }
}
int main() {
    FILE* f = fopen("exp/ledger_states.bin", "rb");
    std::vector<Rec> recs; Rec r;
    while (fread(r.unit, 8, NT, f) == NT && fread(r.a, 2, NT*32, f) == NT*32 && fread(r.h, 4, NT*32, f) == NT*32 &&
           fread(r.cash_after, 8, 32, f) == 32 && fread(r.p, 8, NT, f) == NT && fread(r.cash0, 8, 32, f) == 32) recs.push_back(r);
    int nr = recs.size();
    Rec* d; cudaMalloc(&d, sizeof(Rec) * nr); cudaMemcpy(d, recs.data(), sizeof(Rec) * nr, cudaMemcpyHostToDevice);
    double* o; int* ho; long long* c; cudaMalloc(&o, 8 * 32 * nr); cudaMalloc(&ho, 4 * NT * 32 * nr); cudaMalloc(&c, 8 * nr);
    void (*ks[])(const Rec*, int, double*, int*, long long*) = {probe<0>, probe<1>, probe<2>};
    std::vector<double> c0(32 * nr), c1(32 * nr); std::vector<int> h0(NT * 32 * nr), h1(NT * 32 * nr);
    for (int v = 0; v < 3; ++v) {
        for (int rep = 0; rep < 3; ++rep) ks[v]<<<1, 32>>>(d, nr, o, ho, c);
        cudaDeviceSynchronize();
        std::vector<long long> hc(nr);
        cudaMemcpy(v ? c1.data() : c0.data(), o, 8 * 32 * nr, cudaMemcpyDeviceToHost);
        cudaMemcpy(v ? h1.data() : h0.data(), ho, 4 * NT * 32 * nr, cudaMemcpyDeviceToHost);
        cudaMemcpy(hc.data(), c, 8 * nr, cudaMemcpyDeviceToHost);
        bool same = !v || (!memcmp(c0.data(), c1.data(), 8 * 32 * nr) && !memcmp(h0.data(), h1.data(), 4 * NT * 32 * nr));
        long long s = 0; for (auto x : hc) s += x;
        printf("buy variant %d: mean %lld cycles (%.1f per ticker) %s\n", v, s / nr, s / nr / 100.0, same ? "identical" : "MISMATCH");
    }
}
