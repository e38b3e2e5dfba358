// Microbenchmark: cycles per ticker of the env-step buy loop and variants (one warp, smem data).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 100;
constexpr long long FR_LO = 0x3DD0000000000000ll, FR_HI = 0x3FEFFFFFFFF80000ll;
__global__ void probe(double* out, long long* cyc, int mode) {
    __shared__ int hold_s[NT * 32], hnew_s[NT * 32];
    __shared__ short aint_s[NT * 32];
    __shared__ double unit_s[NT], rcp_s[NT], p164[NT], dtab[128];
    const int lane = threadIdx.x;
    for (int i = lane; i < NT; i += 32) {
        unit_s[i] = 100.0 + i * 0.37;
        rcp_s[i] = 1.0 / unit_s[i];
        p164[i] = 100.5 + i * 0.37;
    }
    for (int i = lane; i < 128; i += 32) dtab[i] = i;
    for (int i = lane; i < NT * 32; i += 32) {
        hold_s[i] = (i * 7) % 50;
        aint_s[i] = static_cast<short>(((i * 13) % 201) - 100);
    }
    __syncwarp();
    double cash = 1e6 + lane, ph = 0.0;
    long long t0 = clock64();
    for (int rep = 0; rep < 10; ++rep) {
        if (mode == 0) {   // the kernel's loop
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                const bool safe = ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                                  (frb >= FR_LO && frb <= FR_HI);
                if (!safe) {
                    double qmax = floor(__ddiv_rn(cash, unit));
                    if (__dmul_rn(qmax, unit) > cash) qmax = __dadd_rn(qmax, -1.0);
                    qd = ad < qmax ? ad : qmax;
                    qd = qd < 0.0 ? 0.0 : qd;
                    cost = __dmul_rn(qd, unit);
                }
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
                ph = __dadd_rn(ph, __dmul_rn(p164[i], static_cast<double>(h)));
            }
        } else if (mode == 1) {   // no safety branch
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
                ph = __dadd_rn(ph, __dmul_rn(p164[i], static_cast<double>(h)));
            }
        } else if (mode == 2) {   // no safety, no ph/hold
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                cash = __dadd_rn(cash, -__dmul_rn(qd, unit));
            }
        } else if (mode == 4) {   // speculative: unsafe tickers only flagged (redo after the loop)
            bool bad = false;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                bad |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                         (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
                ph = __dadd_rn(ph, __dmul_rn(p164[i], static_cast<double>(h)));
            }
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 5) {   // speculative, ph accumulated in a second pass
            bool bad = false;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                bad |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                         (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
            }
#pragma unroll 8
            for (int i = 0; i < NT; ++i) ph = __dadd_rn(ph, __dmul_rn(p164[i], static_cast<double>(hold_s[i * 32 + lane])));
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 6) {   // speculative, no ph, table ad, magic-number q -> int
            bool bad = false;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = dtab[ai > 0 ? ai : 0];
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                bad |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                         (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(__double_as_longlong(__dadd_rn(qd, 6755399441055744.0)));
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
            }
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 7) {   // speculative, no ph (as the kernel now)
            bool bad = false;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                bad |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                         (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
            }
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 8) {   // chain with the min done on int bits, cost via table
            bool bad = false;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = dtab[ai > 0 ? ai : 0];
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                const bool lt = __double_as_longlong(fl) < __double_as_longlong(ad);
                const double qd = lt ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                bad |= !(ai <= 0 || !lt && fl != ad || (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(__double_as_longlong(__dadd_rn(qd, 6755399441055744.0)));
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
            }
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 9) {   // spec no ph, chunk of 16 loaded into registers first
            bool bad = false;
            for (int c0 = 0; c0 < NT; c0 += 16) {
                int aa[16], hh[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int i = c0 + k < NT ? c0 + k : NT - 1;
                    aa[k] = aint_s[i * 32 + lane];
                    hh[k] = hold_s[i * 32 + lane];
                }
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int i = c0 + k;
                    if (i < NT) {
                        const int ai = aa[k];
                        int h = hh[k];
                        if (ai < 0) h -= min(h, -ai);
                        const double unit = unit_s[i];
                        const double ad = static_cast<double>(ai > 0 ? ai : 0);
                        const double y = __dmul_rn(cash, rcp_s[i]);
                        const double fl = floor(y);
                        double qd = fl < ad ? fl : ad;
                        double cost = __dmul_rn(qd, unit);
                        const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                        bad |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                                 (frb >= FR_LO && frb <= FR_HI));
                        h += static_cast<int>(qd);
                        cash = __dadd_rn(cash, -cost);
                        hold_s[i * 32 + lane] = h;
                    }
                }
            }
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 10) {   // chain only + hold load/store
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                cash = __dadd_rn(cash, -__dmul_rn(qd, unit));
                hold_s[i * 32 + lane] = h + static_cast<int>(qd);
            }
        } else if (mode == 11) {   // chain + hold ld/st, magic-number conversion
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                cash = __dadd_rn(cash, -__dmul_rn(qd, unit));
                hold_s[i * 32 + lane] = h + static_cast<int>(__double_as_longlong(__dadd_rn(qd, 6755399441055744.0)));
            }
        } else if (mode == 12) {   // chain + F2I, no ld/st of hold
            int hs = 0;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                cash = __dadd_rn(cash, -__dmul_rn(qd, unit));
                hs += static_cast<int>(qd);
            }
            ph += hs;
        } else if (mode == 13) {   // chain + hold ld/st (no conversion: q from the int action bound)
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                const bool lt = fl < ad;
                double qd = lt ? fl : ad;
                cash = __dadd_rn(cash, -__dmul_rn(qd, unit));
                hold_s[i * 32 + lane] = h + (lt ? 0 : ai);
            }
        } else if (mode == 14) {   // spec no ph, results to a separate smem array
            bool bad = false;
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const double ad = static_cast<double>(ai > 0 ? ai : 0);
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                double qd = fl < ad ? fl : ad;
                double cost = __dmul_rn(qd, unit);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                bad |= !(ai <= 0 || __double_as_longlong(fl) > __double_as_longlong(ad) ||
                         (frb >= FR_LO && frb <= FR_HI));
                h += static_cast<int>(qd);
                cash = __dadd_rn(cash, -cost);
                hnew_s[i * 32 + lane] = h;
            }
            if (__any_sync(0xffffffffu, bad)) cash += 1.0;
        } else if (mode == 3) {   // kernel loop, min in integer domain (q int) and cost = fl(q unit)
#pragma unroll 4
            for (int i = 0; i < NT; ++i) {
                const int ai = aint_s[i * 32 + lane];
                int h = hold_s[i * 32 + lane];
                if (ai < 0) h -= min(h, -ai);
                const double unit = unit_s[i];
                const int ap = ai > 0 ? ai : 0;
                const double y = __dmul_rn(cash, rcp_s[i]);
                const double fl = floor(y);
                const long long flb = __double_as_longlong(fl);
                const long long frb = __double_as_longlong(__dadd_rn(y, -fl));
                // fl as integer (fl < 2^31 whenever it matters, i.e. fl <= ap)
                const int fi = flb > __double_as_longlong(static_cast<double>(ap)) ? ap + 1 : static_cast<int>(fl);
                int q = fi < ap ? fi : ap;
                double cost = __dmul_rn(static_cast<double>(q), unit);
                const bool safe = ai <= 0 || fi > ap || (frb >= FR_LO && frb <= FR_HI);
                if (!safe) {
                    double qmax = floor(__ddiv_rn(cash, unit));
                    if (__dmul_rn(qmax, unit) > cash) qmax = __dadd_rn(qmax, -1.0);
                    double qd = ap < qmax ? ap : qmax;
                    qd = qd < 0.0 ? 0.0 : qd;
                    q = static_cast<int>(qd);
                    cost = __dmul_rn(qd, unit);
                }
                h += q;
                cash = __dadd_rn(cash, -cost);
                hold_s[i * 32 + lane] = h;
                ph = __dadd_rn(ph, __dmul_rn(p164[i], static_cast<double>(h)));
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[mode] = t1 - t0;
    out[lane] = cash + ph + hnew_s[lane * 7 % (NT * 32)];
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 8 * 32); cudaMalloc(&c, 8 * 16);
    const char* nm[] = {"kernel buy loop", "no safety branch", "chain only", "int-domain min", "speculative", "spec + ph pass", "spec tab+magic", "spec no ph", "int-bit min", "spec regs chunk16", "chain + hold ld/st", "chain+ld/st magic", "chain + F2I", "chain + ld/st no cvt", "spec, separate out"};
    for (int m = 0; m < 15; ++m) {
        probe<<<1, 32>>>(d, c, m);
        probe<<<1, 32>>>(d, c, m);
    }
    long long h[16];
    cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
    for (int m = 0; m < 15; ++m) printf("%-22s %.1f cycles/ticker\n", nm[m], h[m] / 1000.0);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
