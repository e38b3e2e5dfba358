// gemm_kernel.cuh — the PPO learner's layer contractions ("PPO"; R#26).
//
// Every contraction of the learner is written as one "TN" product over row-major, K-contiguous operands:
//     C[M][N] = sum_k A[M][K] B[N][K]          (fp32 accumulate)
//   forward     Z_l     = X_l W_l^T            A = X_l   [B][in],    B = W_l   [out][in]
//   weight grad dW_l    = delta_l^T X_l        A = d_l^T [out][B],   B = X_l^T [in][B]
//   input grad  dX_l    = delta_l W_l          A = d_l   [B][out],   B = W_l^T [in][out]
// so the forward epilogue stores each activation twice (row-major for the next forward product, transposed
// for the weight gradient) and the input-gradient epilogue does the same for delta; W_l^T is refreshed
// from the float32 master after every Adam step.  Two cores share the epilogue and the operand layouts:
//   * tc_gemm_kernel: bf16 x bf16 -> f32 on the 5th-generation tensor cores.  One 128 x BN tile per CTA;
//     one thread streams 128 x 64 and BN x 64 operand boxes with TMA (128-B swizzle) through a 4-stage
//     mbarrier ring, one thread issues tcgen05.mma (M = 128, N = BN, K = 16, four per box) into a TMEM
//     accumulator, then the four warps read their 32 TMEM lanes (rows) with tcgen05.ld in 32-column
//     chunks and run the epilogue.
//   * simt_gemm_f32_kernel: float32 operands, float32 FMA on the CUDA cores, the same thread = row mapping
//     and the same epilogue — the precision-reference mode of the learner (parity at float32 bars).
// Epilogues (per 32-column chunk of one row):
//   FWD_HIDDEN  x = act(acc + b)  -> out [row][c], out_t [c][row]          (rows >= M written as 0)
//   FWD_HEAD    z = acc + b       -> outf [row][c] (f32)
//   DW          g = acc           -> outf [row][c] (f32, the gradient segment of W_l)
//   DX          d = acc act'(x_l) -> out, out_t, and the column sums of the tile's 128 rows (the bias
//               gradient of the layer below, reduced later in a fixed order: deterministic)
// act' from the stored post-activation x: ReLU' = [x > 0], tanh' = 1 - x^2.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "ptx.cuh"

namespace pod {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_STAGES = 4;
enum GemmEpiMode : int { EPI_FWD_HIDDEN = 0, EPI_FWD_HEAD = 1, EPI_DW = 2, EPI_DX = 3 };

template <class T>
struct GemmEpi {
    int32_t mode;
    int32_t M;           // valid output rows
    int32_t N;           // valid output columns
    int32_t act;         // 0 = ReLU, 1 = tanh
    const float* bias;   // [N]                       (FWD modes)
    T* out;              // [rows][ld_out]            (FWD_HIDDEN, DX)
    T* out_t;            // [N][ld_out_t]             (FWD_HIDDEN, DX)
    float* outf;         // [rows][ld_outf]           (FWD_HEAD, DW)
    const T* xl;         // [rows][ld_xl]             (DX: the layer input, post-activation)
    float* bpart;        // [rows / 128][N]           (DX: per-tile column sums)
    int32_t ld_out, ld_out_t, ld_outf, ld_xl;
};

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
template <class T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

// 32 consecutive values of one row -> T, row-major (16-byte stores)
__device__ __forceinline__ void store_row32(float* dst, const float (&x)[32]) {
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
}
__device__ __forceinline__ void store_row32(__nv_bfloat16* dst, const float (&x)[32]) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        d[q] = make_uint4(pack_bf16x2(x[8 * q], x[8 * q + 1]), pack_bf16x2(x[8 * q + 2], x[8 * q + 3]),
                          pack_bf16x2(x[8 * q + 4], x[8 * q + 5]), pack_bf16x2(x[8 * q + 6], x[8 * q + 7]));
}
__device__ __forceinline__ void load_row32(const float* src, float (&x)[32]) {
    const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float4 v = s[q];
        x[4 * q] = v.x;
        x[4 * q + 1] = v.y;
        x[4 * q + 2] = v.z;
        x[4 * q + 3] = v.w;
    }
}
__device__ __forceinline__ void load_row32(const __nv_bfloat16* src, float (&x)[32]) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint4 v = s[q];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[8 * q + 2 * j] = __uint_as_float(w[j] << 16);
            x[8 * q + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
    }
}

// lane l ends with the sum over the warp's 32 lanes of v[l] (recursive halving: 31 shuffles)
__device__ __forceinline__ float warp_transpose_sum32(float (&v)[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
            const float send = upper ? v[j] : v[j + s];
            const float keep = upper ? v[j + s] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return v[0];
}

// the epilogue of one row's 32-column chunk [c0, c0 + 32); every lane of the warp calls it (row = the
// lane's row, rows of a warp consecutive); columns >= N are never stored
template <class T>
__device__ __forceinline__ void gemm_epilogue_chunk(const GemmEpi<T>& e, int row, int c0, float (&v)[32], int lane,
                                                    const float* bias_s, float* red_s) {
    const bool rv = row < e.M;
    const bool full = c0 + 32 <= e.N;
    if (e.mode == EPI_FWD_HIDDEN || e.mode == EPI_FWD_HEAD) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float x = v[j] + bias_s[j];   // the chunk's bias, staged in shared memory (0 beyond N)
            if (e.mode == EPI_FWD_HIDDEN) x = e.act == 0 ? fmaxf(x, 0.0f) : tanhf(x);
            v[j] = rv ? x : 0.0f;
        }
        if (e.mode == EPI_FWD_HEAD) {
            float* dst = e.outf + static_cast<int64_t>(row) * e.ld_outf + c0;
            if (full) {
                store_row32(dst, v);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (c0 + j < e.N) dst[j] = v[j];
            }
            return;
        }
    } else if (e.mode == EPI_DW) {
        if (!rv) return;
        float* dst = e.outf + static_cast<int64_t>(row) * e.ld_outf + c0;
        if (full) {
            store_row32(dst, v);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c0 + j < e.N) dst[j] = v[j];
        }
        return;
    } else {   // EPI_DX
        float x[32];
        load_row32(e.xl + static_cast<int64_t>(row) * e.ld_xl + c0, x);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float d = e.act == 0 ? (x[j] > 0.0f ? 1.0f : 0.0f) : (1.0f - x[j] * x[j]);
            v[j] = rv ? v[j] * d : 0.0f;
        }
    }
    // FWD_HIDDEN / DX: row-major and transposed copies (T); the padded rows carry zeros
    T* dst = e.out + static_cast<int64_t>(row) * e.ld_out + c0;
    if (full) {
        store_row32(dst, v);
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (c0 + j < e.N) dst[j] = from_f32<T>(v[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
        if (c0 + j < e.N) e.out_t[static_cast<int64_t>(c0 + j) * e.ld_out_t + row] = from_f32<T>(v[j]);
    if (e.mode == EPI_DX) {
        // the tile's column sums: each warp's 32 rows (transpose-reduce), then the 4 warps in order
        const int wq = (threadIdx.x >> 5) & 3;
        red_s[wq * 32 + lane] = warp_transpose_sum32(v, lane);   // column c0 + lane
        named_bar_sync(1, 128);
        if (wq == 0 && c0 + lane < e.N)
            e.bpart[static_cast<int64_t>(row >> 7) * e.N + c0 + lane] =
                ((red_s[lane] + red_s[32 + lane]) + red_s[64 + lane]) + red_s[96 + lane];
        named_bar_sync(1, 128);
    }
}

__host__ __device__ constexpr int gemm_smem_bytes(int BN) {
    return 1024 + GEMM_STAGES * (GEMM_BM * GEMM_BK * 2 + BN * GEMM_BK * 2) + 256 + 4 * BN + 512;
}

// bf16 x bf16 -> f32 on tcgen05; grid (M_rows / 128, ceil(N / BN)); K a multiple of 64
template <int BN>
__global__ void __launch_bounds__(128, 1) tc_gemm_kernel(const __grid_constant__ CUtensorMap ma,
                                                         const __grid_constant__ CUtensorMap mb,
                                                         const GemmEpi<__nv_bfloat16> ep, int K) {
    constexpr uint32_t A_BYTES = GEMM_BM * GEMM_BK * 2;
    constexpr uint32_t B_BYTES = BN * GEMM_BK * 2;
    constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    constexpr uint32_t TCOLS = BN < 32 ? 32 : BN;
    extern __shared__ __align__(1024) uint8_t gsm_raw[];
    uint8_t* gsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(gsm);
    const uint32_t bars = sbase + GEMM_STAGES * STAGE;   // full[S], empty[S], done
    const uint32_t full_b = bars, empty_b = bars + 8u * GEMM_STAGES, done_b = bars + 16u * GEMM_STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(gsm + GEMM_STAGES * STAGE + 16 * GEMM_STAGES + 8);
    float* bias_s = reinterpret_cast<float*>(gsm + GEMM_STAGES * STAGE + 256);   // [BN] (forward epilogues)
    float* red_s = bias_s + BN;                                                   // [4][32] (input-gradient)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc(smem_u32(tslot), TCOLS);
    if (tid == 32) {
        for (int s = 0; s < GEMM_STAGES; ++s) {
            mbar_init(full_b + 8u * s, 1);
            mbar_init(empty_b + 8u * s, 1);
        }
        mbar_init(done_b, 1);
        fence_mbar_init();
    }
    const int m0 = static_cast<int>(blockIdx.x) * GEMM_BM, n0 = static_cast<int>(blockIdx.y) * BN;
    if (ep.bias)
        for (int c = tid; c < BN; c += 128) bias_s[c] = n0 + c < ep.N ? ep.bias[n0 + c] : 0.0f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int KB = K / GEMM_BK;
    if (tid == 0) {
        prefetch_tmap(&ma);
        prefetch_tmap(&mb);
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % GEMM_STAGES;
            if (kb >= GEMM_STAGES) mbar_wait(empty_b + 8u * s, static_cast<uint32_t>((kb / GEMM_STAGES) & 1) ^ 1u);
            mbar_arrive_expect_tx(full_b + 8u * s, STAGE);
            tma_load_2d(sbase + s * STAGE, &ma, kb * GEMM_BK, m0, full_b + 8u * s);
            tma_load_2d(sbase + s * STAGE + A_BYTES, &mb, kb * GEMM_BK, n0, full_b + 8u * s);
        }
    } else if (tid == 32) {
        const uint32_t idesc = idesc_bf16_f32(GEMM_BM, BN);
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % GEMM_STAGES;
            mbar_wait(full_b + 8u * s, static_cast<uint32_t>((kb / GEMM_STAGES) & 1));
            tc_fence_after();
            const uint64_t ad = sw128_desc(sbase + s * STAGE), bd = sw128_desc(sbase + s * STAGE + A_BYTES);
#pragma unroll
            for (int kk = 0; kk < GEMM_BK / 16; ++kk)   // K = 16 per MMA: +32 B in the swizzled rows
                mma_bf16(tmem, ad + 2u * kk, bd + 2u * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
            mma_commit(empty_b + 8u * s);   // the stage is free once these MMAs have read it
        }
        mma_commit(done_b);
    }
    __syncwarp();
    mbar_wait(done_b, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
#pragma unroll 1
    for (int cc = 0; cc < BN / 32; ++cc) {
        if (n0 + cc * 32 >= ep.N) break;
        uint32_t r[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cc * 32), r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        gemm_epilogue_chunk(ep, row, n0 + cc * 32, v, lane, bias_s + cc * 32, red_s);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, TCOLS);
}

// float32 reference core: thread = row of the 128 x BN tile, K in chunks of 32 through shared memory.
// A [rowsA][lda], B [rowsB][ldb] (K-contiguous); rows beyond rowsA / rowsB read as zero.
template <int BN>
__global__ void __launch_bounds__(128) simt_gemm_f32_kernel(const float* __restrict__ A, int lda, int rowsA,
                                                            const float* __restrict__ B, int ldb, int rowsB, int K,
                                                            const GemmEpi<float> ep) {
    __shared__ float As[32][GEMM_BM + 1];
    __shared__ float Bs[32][BN];
    __shared__ float bias_s[BN];
    __shared__ float red_s[128];
    const int tid = threadIdx.x, lane = tid & 31;
    const int m0 = static_cast<int>(blockIdx.x) * GEMM_BM, n0 = static_cast<int>(blockIdx.y) * BN;
    if (ep.bias)
        for (int c = tid; c < BN; c += 128) bias_s[c] = n0 + c < ep.N ? ep.bias[n0 + c] : 0.0f;
    float acc[BN];
#pragma unroll
    for (int c = 0; c < BN; ++c) acc[c] = 0.0f;
    for (int k0 = 0; k0 < K; k0 += 32) {
        for (int idx = tid; idx < GEMM_BM * 32; idx += 128) {
            const int r = idx >> 5, kk = idx & 31;
            As[kk][r] = m0 + r < rowsA ? A[static_cast<int64_t>(m0 + r) * lda + k0 + kk] : 0.0f;
        }
        for (int idx = tid; idx < BN * 32; idx += 128) {
            const int c = idx >> 5, kk = idx & 31;
            Bs[kk][c] = n0 + c < rowsB ? B[static_cast<int64_t>(n0 + c) * ldb + k0 + kk] : 0.0f;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < 32; ++kk) {
            const float a = As[kk][tid];
#pragma unroll
            for (int c = 0; c < BN; ++c) acc[c] = fmaf(a, Bs[kk][c], acc[c]);
        }
        __syncthreads();
    }
    const int row = m0 + tid;
#pragma unroll
    for (int cc = 0; cc < BN / 32; ++cc) {
        if (n0 + cc * 32 >= ep.N) break;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = acc[cc * 32 + j];
        gemm_epilogue_chunk(ep, row, n0 + cc * 32, v, lane, bias_s + cc * 32, red_s);
    }
}

}  // namespace pod
