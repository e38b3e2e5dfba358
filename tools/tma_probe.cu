// Microbenchmark: per-SM streaming rate of 16 KB weight tiles from L2 into a
// 5-stage shared-memory ring, (a) 2-D tensor TMA box 128 rows x 128 B (SW128),
// (b) one contiguous cp.async.bulk of 16 KB, (c) two bulk copies of 8 KB.
// Grid = 128 CTAs (as the actor kernel at C3); each CTA streams `iters` tiles.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2111_05188_b200/csrc/ptx.cuh"
using namespace pod;

constexpr int STAGES = 5;
constexpr int TILE = 16384;

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                    const __grid_constant__ CUtensorMap map64, const char* src, int mode,
                                                    int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    const uint32_t bars = base + STAGES * TILE;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bars + 8 * s, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int tiles = 104;   // 1.7 MB of tiles cycled through (L2 resident)
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        // prologue: fill the ring
        for (int q = 0; q < iters + STAGES; ++q) {
            const int s = q % STAGES;
            if (q >= STAGES) mbar_wait(bars + 8 * s, ((q / STAGES) - 1) & 1);   // consumed (we just wait data)
            if (q >= iters) break;
            const int tile = (q + blockIdx.x * 7) % tiles;
            mbar_arrive_expect_tx(bars + 8 * s, TILE);
            if (mode == 3) {
                tma_load_2d(base + s * TILE, &map64, (tile % 16) * 32, (tile / 16) * 256, bars + 8 * s);
            } else if (mode == 0) {
                tma_load_2d(base + s * TILE, &map, (tile % 8) * 64, (tile / 8) * 128, bars + 8 * s);
            } else if (mode == 1) {
                bulk_g2s(base + s * TILE, src + static_cast<size_t>(tile) * TILE, TILE, bars + 8 * s);
            } else {
                bulk_g2s(base + s * TILE, src + static_cast<size_t>(tile) * TILE, TILE / 2, bars + 8 * s);
                bulk_g2s(base + s * TILE + TILE / 2, src + static_cast<size_t>(tile) * TILE + TILE / 2, TILE / 2, bars + 8 * s);
            }
        }
        mbar_wait(bars + 8 * ((iters - 1) % STAGES), ((iters - 1) / STAGES) & 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    // weights-like buffer: 13 row-chunks x 128 rows x 1 KB rows (512 bf16) = 1.7 MB
    const size_t bytes = 104 * TILE;
    char* d;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    unsigned long long* out;
    cudaMalloc(&out, 1024 * 8);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {512, 13 * 128};
    cuuint64_t str[1] = {1024};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap map64;
    cuuint32_t box64[2] = {32, 256};
    ((EncodeFn)fn)(&map64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = STAGES * TILE + 1024 + 64;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"tensor TMA 128x128B SW128", "bulk 16 KB contiguous", "bulk 2 x 8 KB", "tensor TMA 256x64B SW64"};
    for (int grid : {1, 128, 148}) {
        for (int mode = 0; mode < 4; ++mode) {
            const int iters = 200;
            for (int rep = 0; rep < 2; ++rep) stream_kernel<<<grid, 64, smem>>>(map, map64, d, mode, iters, out);
            cudaDeviceSynchronize();
            unsigned long long h[256];
            cudaMemcpy(h, out, 8 * grid, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += h[i];
            avg /= grid;
            printf("grid %3d  %-28s %7.1f cycles/tile  %6.1f B/clk/SM\n", grid, names[mode], avg / iters,
                   TILE * iters / avg);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
