#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, double m, int* sm_in) {
    __shared__ double sd[64];
    __shared__ int si[64];
    sd[threadIdx.x] = threadIdx.x; sd[threadIdx.x+32] = threadIdx.x; si[threadIdx.x] = 0; si[threadIdx.x+32]=0;
    __syncwarp();
    double x = x0 + threadIdx.x;
    long long t0, t1;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = floor(x * m);   // dmul + frnd
    t1 = clock64(); cyc[0] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) { double y = x * m; x = (y < 1e300) ? y : x; }   // dmul + dsetp + fsel
    t1 = clock64(); cyc[1] = t1 - t0;
    int j = threadIdx.x;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) j = si[j & 63] + j;   // lds chain
    t1 = clock64(); cyc[2] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = (double)((int)x + 1);   // f2i + i2f
    t1 = clock64(); cyc[3] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) { x = x * m; if (__any_sync(0xffffffff, x > 1e300)) x = 0; }   // dmul + dsetp + vote + bra
    t1 = clock64(); cyc[4] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = __dadd_rd(x * m, 4503599627370496.0) - 4503599627370496.0;   // dmul + 2 dadd
    t1 = clock64(); cyc[5] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = x * m;
    t1 = clock64(); cyc[6] = t1 - t0;
    out[threadIdx.x] = x + j;
}
int main() {
    double* o; long long* c; int* s; cudaMalloc(&o, 8*64); cudaMalloc(&c, 128); cudaMalloc(&s, 256);
    k<<<1,32>>>(o, c, 1.5, 1.0000001, s); k<<<1,32>>>(o, c, 1.5, 1.0000001, s);
    long long h[7]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
    const char* nm[] = {"dmul+frnd", "dmul+dsetp+fsel", "lds", "f2i+i2f", "dmul+dsetp+vote+bra", "dmul+2dadd(floor trick)", "dmul"};
    for (int i = 0; i < 7; ++i) printf("%s: %.1f cycles/iter\n", nm[i], h[i] / 64.0);
}
