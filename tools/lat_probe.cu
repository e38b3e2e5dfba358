// Microbenchmark: dependent-chain latency (cycles per op) of fp64 / fp32 ops on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double x0, float f0) {
    double x = x0, y = x0 * 0.5;
    float f = f0;
    long long t0, t1;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, y);
    t1 = clock64(); cyc[0] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = __dmul_rn(x, 1.0000001);
    t1 = clock64(); cyc[1] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = __fma_rn(x, 0.9999999, y);
    t1 = clock64(); cyc[2] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = floor(x) + 0.5;
    t1 = clock64(); cyc[3] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = __ddiv_rn(x, 1.0000001);
    t1 = clock64(); cyc[4] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) f = __fadd_rn(f, 1.5f);
    t1 = clock64(); cyc[5] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = (x > y) ? __dadd_rn(x, -1.0) : x;
    t1 = clock64(); cyc[6] = t1 - t0;
    out[0] = x + f;
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 8); cudaMalloc(&c, 8 * 8);
    probe<<<1, 32>>>(d, c, 1.25, 1.0f);
    probe<<<1, 32>>>(d, c, 1.25, 1.0f);
    long long h[8];
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char* nm[] = {"DADD", "DMUL", "DFMA", "FRND+DADD", "DDIV", "FADD(f32)", "DSETP+sel+DADD"};
    for (int i = 0; i < 7; ++i) printf("%-16s %.1f cycles/op (incl. loop)\n", nm[i], h[i] / 1024.0);
    return 0;
}
