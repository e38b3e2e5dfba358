#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
constexpr int NT = 100;
struct Rec { double unit[NT]; short a[NT * 32]; int h[NT * 32]; double cash_after[32]; double p[NT]; double cash0[32]; };
template <int V>
__global__ void probe(const Rec* recs, int nrec, double* out, long long* cyc) {
    __shared__ int hold_s[NT * 32];
    __shared__ short aint_s[NT * 32];
    __shared__ double p64[NT];
    const int lane = threadIdx.x;
    for (int r = 0; r < nrec; ++r) {
        const Rec& R = recs[r];
        for (int i = lane; i < NT; i += 32) p64[i] = R.p[i];
        for (int i = lane; i < NT * 32; i += 32) { hold_s[i] = R.h[i]; aint_s[i] = R.a[i]; }
        __syncwarp();
        double cash = R.cash0[lane];
        const double omc = __dadd_rn(1.0, -0.002);
        const int n = NT;
        long long t0 = clock64();
        if (V == 0) {
#pragma unroll 16
            for (int i = 0; i < n; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const int h = hold_s[i * 32 + lane];
                const int q = ai < 0 ? min(h, -ai) : 0;
                cash = __dadd_rn(cash, __dmul_rn(__dmul_rn(p64[i], static_cast<double>(q)), omc));
            }
        } else if (V == 1) {   // int -> double by the 2^52 trick
#pragma unroll 16
            for (int i = 0; i < n; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const int h = hold_s[i * 32 + lane];
                const int q = ai < 0 ? min(h, -ai) : 0;
                const double qd = __dadd_rn(__hiloint2double(0x43300000, q), -4503599627370496.0);
                cash = __dadd_rn(cash, __dmul_rn(__dmul_rn(p64[i], qd), omc));
            }
        } else if (V == 2) {   // all products first (registers), then the carried adds
            double pr[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const int h = hold_s[i * 32 + lane];
                const int q = ai < 0 ? min(h, -ai) : 0;
                pr[i] = __dmul_rn(__dmul_rn(p64[i], static_cast<double>(q)), omc);
            }
#pragma unroll
            for (int i = 0; i < NT; ++i) cash = __dadd_rn(cash, pr[i]);
        } else if (V == 3) {   // blocks of 20: products, then adds
#pragma unroll 1
            for (int i0 = 0; i0 < n; i0 += 20) {
                double pr[20];
#pragma unroll
                for (int k = 0; k < 20; ++k) {
                    const int i = i0 + k;
                    const int ai = aint_s[i * 32 + lane];
                    const int h = hold_s[i * 32 + lane];
                    const int q = ai < 0 ? min(h, -ai) : 0;
                    pr[k] = __dmul_rn(__dmul_rn(p64[i], static_cast<double>(q)), omc);
                }
#pragma unroll
                for (int k = 0; k < 20; ++k) cash = __dadd_rn(cash, pr[k]);
            }
        }
        long long t1 = clock64();
        out[r * 32 + lane] = cash;
        if (lane == 0) cyc[r] = t1 - t0;
        __syncwarp();
    }
}
int main(int argc, char** argv) {
    FILE* f = fopen("exp/ledger_states.bin", "rb");
    std::vector<Rec> recs; Rec r;
    while (fread(r.unit, 8, NT, f) == NT && fread(r.a, 2, NT*32, f) == NT*32 && fread(r.h, 4, NT*32, f) == NT*32 &&
           fread(r.cash_after, 8, 32, f) == 32 && fread(r.p, 8, NT, f) == NT && fread(r.cash0, 8, 32, f) == 32) recs.push_back(r);
    int nr = recs.size();
    Rec* d; cudaMalloc(&d, sizeof(Rec) * nr); cudaMemcpy(d, recs.data(), sizeof(Rec) * nr, cudaMemcpyHostToDevice);
    double* o; long long* c; cudaMalloc(&o, 8 * 32 * nr); cudaMalloc(&c, 8 * nr);
    void (*ks[])(const Rec*, int, double*, long long*) = {probe<0>, probe<1>, probe<2>, probe<3>};
    for (int v = 0; v < 4; ++v) {
        for (int rep = 0; rep < 3; ++rep) ks[v]<<<1, 32>>>(d, nr, o, c);
        cudaDeviceSynchronize();
        std::vector<double> ho(32 * nr); std::vector<long long> hc(nr);
        cudaMemcpy(ho.data(), o, 8 * 32 * nr, cudaMemcpyDeviceToHost); cudaMemcpy(hc.data(), c, 8 * nr, cudaMemcpyDeviceToHost);
        bool ok = true; for (int i = 0; i < nr; ++i) for (int l = 0; l < 32; ++l) ok &= ho[i*32+l] == recs[i].cash_after[l];
        long long s = 0; for (auto x : hc) s += x;
        printf("sell variant %d: mean %lld cycles  %s\n", v, s / nr, ok ? "exact" : "MISMATCH");
    }
}
