// Microbenchmark: cost of the actor epilogue's swizzled st.shared (8 warps x 4 atoms x 4 STS.128 per
// thread) alone and while (B) a TMA stream fills a 5-stage ring of 16 KB weight-like tiles, (C) a
// tcgen05.mma stream (M=128, N=256, K=16, SS) reads the activation buffer and the ring, (D) both.
// One 320-thread CTA per SM, 128 CTAs (the actor's C3 grid), smem laid out as the actor's.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2111_05188_b200/csrc/ptx.cuh"
using namespace pod;

constexpr int STAGES = 5;
constexpr int TILE = 16384;

__global__ void __launch_bounds__(320, 1) probe(const __grid_constant__ CUtensorMap map, int mode, int reps,
                                                unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    const uint32_t act = base;                       // 128 KB activation buffer (8 atoms of 16 KB)
    const uint32_t ring = base + 131072u;            // 5 x 16 KB
    const uint32_t bars = ring + STAGES * TILE;      // STAGES full barriers + done barrier + tmem slot
    const uint32_t done_b = bars + 8u * STAGES;
    const uint32_t tslot = done_b + 8u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s) mbar_init(bars + 8u * s, 1);
            mbar_init(done_b, 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(tslot, 256);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + (tslot - smem_u32(sm)));
    volatile int* stop = reinterpret_cast<volatile int*>(sm + (tslot + 4 - smem_u32(sm)));
    if (threadIdx.x == 0) *stop = 0;
    __syncthreads();
    if (warp == 0) {
        if (lane == 0 && (mode & 1)) {   // TMA stream into the ring until the epilogue is done
            uint32_t phase = 0;
            int s = 0, q = 0;
            while (!*stop) {
                if (q >= STAGES) mbar_wait(bars + 8u * s, phase ^ 1u);
                mbar_arrive_expect_tx(bars + 8u * s, TILE);
                tma_load_2d(ring + s * TILE, &map, 0, ((q + blockIdx.x * 3) % 96) * 256, bars + 8u * s);
                ++q;
                if (++s == STAGES) {
                    s = 0;
                    phase ^= 1u;
                }
            }
            // drain
            for (int k = 0; k < STAGES && k < q; ++k) {
                const int qq = q - 1 - k;
                mbar_wait(bars + 8u * (qq % STAGES), (qq / STAGES) & 1u);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && (mode & 2)) {   // MMA stream reading act + ring
            const uint64_t ad = sw128_desc(act), bd = sw64_desc(ring);
            const uint32_t idesc = idesc_bf16_f32(128, 256);
            int k = 0, nc = 0;
            while (!*stop) {
                mma_bf16(tmem, ad + ((k & 15) * 64 >> 4), bd + (((k % 5) * TILE) >> 4), idesc, k != 0);
                ++k;
                if ((k & 63) == 0) {   // keep the queue bounded
                    mma_commit(done_b);
                    mbar_wait(done_b, static_cast<uint32_t>(nc) & 1u);
                    ++nc;
                }
            }
            mma_commit(done_b);
            mbar_wait(done_b, static_cast<uint32_t>(nc) & 1u);
        }
    } else {
        // epilogue warps: 4 atoms x (4 STS.128) each, reps times
        const int ew = warp - 2, quad = warp & 3, hh = ew >> 2;
        const int r = quad * 32 + lane;
        uint32_t pk[16];
        for (int i = 0; i < 16; ++i) pk[i] = threadIdx.x * 16 + i;
        named_bar_sync(1, 256);
        unsigned long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int j = 0; j < 4; ++j) {
                const uint32_t atom = act + static_cast<uint32_t>(4 + j) * 16384u;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    st_shared_v4(atom + sw128_offset(static_cast<uint32_t>(r), static_cast<uint32_t>(hh * 4 + q)),
                                 pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                pk[0] += rep;
            }
        }
        named_bar_sync(1, 256);
        unsigned long long t1 = clock64();
        if (ew == 0 && lane == 0) {
            out[blockIdx.x] = t1 - t0;
            *stop = 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t rows = 96 * 256, cols = 32;
    void* d;
    cudaMalloc(&d, rows * cols * 2);
    cudaMemset(d, 0, rows * cols * 2);
    unsigned long long* out;
    cudaMalloc(&out, 256 * 8);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t str[1] = {cols * 2};
    cuuint32_t box[2] = {32, 256}, es[2] = {1, 1};
    ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 131072 + STAGES * TILE + 1024 + 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"STS alone", "STS + TMA stream", "STS + MMA stream", "STS + TMA + MMA"};
    const int reps = 64;
    for (int mode = 0; mode < 4; ++mode) {
        for (int k = 0; k < 2; ++k) probe<<<128, 320, smem>>>(map, mode, reps, out);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[128];
        cudaMemcpy(h, out, 128 * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 128; ++i) avg += h[i];
        avg /= 128;
        printf("%-20s %8.1f cycles per atom (16 KB, 256 threads)  %s\n", names[mode], avg / (reps * 4),
               cudaGetErrorString(e));
    }
    return 0;
}
