// gae_kernel.cuh — K3: segmented reverse-time GAE scan over [T][N].
//
// Method (R#11; PPO P:L472 needs it):
//   delta_t = r_t + gamma (1-d_t) V_{t+1} - V_t,   V_T = boot
//   A_t = delta_t + gamma lambda (1-d_t) A_{t+1},  A_T = 0,   R_t = A_t + V_t.
//
// B200 mapping: the recurrence is sequential in t and independent over envs,
// so lane = env and one warp owns 32 env columns.  The kernel is HBM-bound
// (17 algorithmic bytes per element), so what matters is bytes in flight:
// each warp streams its columns backwards through a STAGES-deep ring of
// [L time rows x 32 envs] chunks in shared memory.  Each chunk arrives as
// three 2-D TMA boxes ({32 envs x 32 steps} of r, V, d) issued by one lane
// (completion on an mbarrier with expect_tx; rows before t = 0 and columns
// past N are zero-filled by the TMA unit), so STAGES x L x 288 B per warp are
// in flight.  A chunk is read into registers, its stage refilled at once,
// the data-only part delta_t computed for all 32 rows, and the loop-carried
// chain reduced to one multiply-add per row; outputs are written with
// coalesced 128-B row stores.  Misaligned inputs (N % 16 != 0) use the
// plain-load path (same arithmetic, same order).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include <cuda.h>

#include "ptx.cuh"

namespace pod {

constexpr int GAE_L = 32;        // time rows per chunk
constexpr int GAE_STAGES = 6;    // chunks in flight per warp
constexpr int GAE_WARPS = 1;     // warps per block (small N: spread column groups over all SMs)

struct __align__(128) GaeStage {
    float r[GAE_L][32];
    float v[GAE_L][32];
    uint8_t d[GAE_L][32];
};

__device__ __forceinline__ void gae_row(float r, float v, uint8_t d, float gamma, float gl, float& v_next,
                                        float& a_next, float* adv, float* ret) {
    const float nd = d ? 0.0f : 1.0f;
    const float delta = (r + gamma * nd * v_next) - v;
    const float A = delta + gl * nd * a_next;
    *adv = A;
    *ret = A + v;
    a_next = A;
    v_next = v;
}

// per-buffer advantage statistics (R#23): this warp's sums of A and A^2, float64, one atomic pair
__device__ __forceinline__ void gae_stats_flush(double s1, double s2, double* stats) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_down_sync(0xffffffffu, s1, o);
        s2 += __shfl_down_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(stats, s1);
        atomicAdd(stats + 1, s2);
    }
}

struct GaeMaps {
    CUtensorMap r, v, d;   // 2-D [T][N], box {32, 32}
};

__global__ void __launch_bounds__(32 * GAE_WARPS)
    gae_kernel(const __grid_constant__ GaeMaps maps, const float* __restrict__ rew, const float* __restrict__ val,
               const uint8_t* __restrict__ done, const float* __restrict__ boot, int T, int N, float gamma,
               float lambda, float* __restrict__ adv, float* __restrict__ ret, int use_bulk,
               double* __restrict__ stats) {
    extern __shared__ __align__(128) uint8_t gsm[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int grp = blockIdx.x * GAE_WARPS + warp;
    const int e0 = grp * 32;
    if (e0 >= N) return;  // warp-uniform
    const int e = e0 + lane;
    const bool active = e < N;
    const float gl = gamma * lambda;
    float v_next = active ? boot[e] : 0.0f;
    float a_next = 0.0f;
    const int nchunks = (T + GAE_L - 1) / GAE_L;

    double s1 = 0.0, s2 = 0.0;   // advantage statistics (stats != null)
    const bool bulk = use_bulk != 0;
    if (!bulk) {
        for (int t = T - 1; t >= 0; --t) {
            if (active) {
                const int64_t i = static_cast<int64_t>(t) * N + e;
                gae_row(rew[i], val[i], done[i], gamma, gl, v_next, a_next, adv + i, ret + i);
                s1 += a_next;
                s2 += static_cast<double>(a_next) * a_next;
            }
        }
        if (stats) gae_stats_flush(s1, s2, stats);
        return;
    }

    GaeStage* st = reinterpret_cast<GaeStage*>(gsm + warp * (GAE_STAGES * sizeof(GaeStage) + 128));
    const uint32_t bars = smem_u32(reinterpret_cast<uint8_t*>(st) + GAE_STAGES * sizeof(GaeStage));
    if (lane == 0) {
        for (int s = 0; s < GAE_STAGES; ++s) mbar_init(bars + 8u * s, 1);
        fence_mbar_init();
    }
    __syncwarp();

    // chunk j covers rows [T - (j+1) L, T - j L) (rows < 0 arrive zero-filled; processed newest first)
    auto issue = [&](int j) {
        const int s = j % GAE_STAGES;
        const int t_hi = T - j * GAE_L;            // exclusive
        const uint32_t bar = bars + 8u * s;
        if (lane == 0) {
            mbar_arrive_expect_tx(bar, GAE_L * (128u + 128u + 32u));
            tma_load_2d(smem_u32(&st[s].r[0][0]), &maps.r, e0, t_hi - GAE_L, bar);
            tma_load_2d(smem_u32(&st[s].v[0][0]), &maps.v, e0, t_hi - GAE_L, bar);
            tma_load_2d(smem_u32(&st[s].d[0][0]), &maps.d, e0, t_hi - GAE_L, bar);
        }
    };

    for (int j = 0; j < GAE_STAGES && j < nchunks; ++j) issue(j);
    for (int j = 0; j < nchunks; ++j) {
        const int s = j % GAE_STAGES;
        const uint32_t parity = static_cast<uint32_t>(j / GAE_STAGES) & 1u;
        mbar_wait(bars + 8u * s, parity);
        // All 32 rows of the stage are processed (rows before t = 0 arrive zero-filled and come last in reverse
        // order, so they only disturb chain state that is never used again; their outputs are not stored).
        // delta_t depends only on data and V_{t+1}, so it is computed for every row first; the loop-carried
        // chain is then one multiply-add per row, A_t = delta_t + (gamma lambda (1-d_t)) A_{t+1}.
        const int t_base = T - (j + 1) * GAE_L;   // time of row q = 0 (may be negative in the last chunk)
        float delta[GAE_L], cgl[GAE_L], vv[GAE_L];
#pragma unroll
        for (int q = GAE_L - 1; q >= 0; --q) {
            const float r = st[s].r[q][lane];
            const float v = st[s].v[q][lane];
            const float nd = st[s].d[q][lane] ? 0.0f : 1.0f;
            delta[q] = (r + gamma * nd * v_next) - v;
            cgl[q] = gl * nd;
            vv[q] = v;
            v_next = v;
        }
        __syncwarp();
        fence_proxy_async_smem();   // order this stage's generic reads before the async refill
        if (j + GAE_STAGES < nchunks) issue(j + GAE_STAGES);
#pragma unroll
        for (int q = GAE_L - 1; q >= 0; --q) {
            const float A = delta[q] + cgl[q] * a_next;
            a_next = A;
            delta[q] = A;
        }
        if (active) {
#pragma unroll
            for (int q = GAE_L - 1; q >= 0; --q) {
                const int t = t_base + q;
                if (t >= 0) {
                    const int64_t i = static_cast<int64_t>(t) * N + e;
                    adv[i] = delta[q];
                    ret[i] = delta[q] + vv[q];
                    if (stats) {
                        s1 += delta[q];
                        s2 += static_cast<double>(delta[q]) * delta[q];
                    }
                }
            }
        }
    }
    if (stats) gae_stats_flush(s1, s2, stats);
}

inline size_t gae_smem_bytes() { return GAE_WARPS * (GAE_STAGES * sizeof(GaeStage) + 128); }

// ---------------------------------------------------------------- segmented variant (few env columns)
// With N / 32 column groups below a few per SM, the one-warp-per-group scan above leaves the SMs nearly empty
// and runs at the latency of one warp's 8K-instruction chain.  The segmented kernel gives each column group a
// block of SEG warps and splits time into SEG segments of CPW chunks (warp w owns chunks [w CPW, (w+1) CPW),
// counted from t = T backwards); the whole [T x 32] column slab stays resident in shared memory.
//   pass 1  each warp runs the recurrence over its segment from A = 0 and records the segment's local
//           advantage at its first row, a_loc, and the product of its coefficients, P = prod gamma lambda (1-d_t);
//   combine A at the end of segment w is A_in(w) = a_loc(w-1) + P(w-1) A_in(w-1), A_in(0) = 0 (exact affine
//           composition of the per-row maps A -> delta_t + c_t A);
//   pass 2  each warp reruns its segment from A_in(w) in the sequential order of the single-warp kernel, so only
//           A_in carries a differently rounded value (a few fp32 ulps of the magnitude recurrence).
constexpr int GAE_SEG_MAX = 16;      // warps per block
constexpr int GAE_CPW_MAX = 2;       // chunks per warp

struct GaeSegSum {
    float aloc[GAE_SEG_MAX][32];
    float prod[GAE_SEG_MAX][32];
};

inline size_t gae_seg_smem_bytes(int seg, int cpw) {
    return static_cast<size_t>(seg) * cpw * sizeof(GaeStage) + sizeof(GaeSegSum) + 8 * GAE_SEG_MAX * GAE_CPW_MAX + 128;
}

// NORM: the per-buffer normalisation (R#23) fused in — a cooperative launch (every block resident): block 0
// zeroes the statistics before a first grid barrier, pass 2 keeps A in shared memory (over r, no longer
// needed) instead of writing it, the float64 sums are flushed, a second grid barrier, and every block
// rewrites its own A as (A - m) / s — one launch and one pass over adv instead of three launches (memset,
// scan, normalisation) and a re-read.
template <bool NORM>
__global__ void __launch_bounds__(32 * GAE_SEG_MAX)
    gae_seg_kernel(const __grid_constant__ GaeMaps maps, const float* __restrict__ boot, int T, int N, float gamma,
                   float lambda, float* __restrict__ adv, float* __restrict__ ret, int cpw,
                   double* __restrict__ stats) {
    extern __shared__ __align__(128) uint8_t gsm[];
    const int seg = blockDim.x >> 5;
    const int w = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int e0 = blockIdx.x * 32;
    const int e = e0 + lane;
    const bool active = e < N;
    const float gl = gamma * lambda;
    const int nchunks = (T + GAE_L - 1) / GAE_L;
    GaeStage* st = reinterpret_cast<GaeStage*>(gsm);
    GaeSegSum* sum = reinterpret_cast<GaeSegSum*>(gsm + static_cast<size_t>(seg) * cpw * sizeof(GaeStage));
    const uint32_t bars = smem_u32(reinterpret_cast<uint8_t*>(sum) + sizeof(GaeSegSum));
    const int j0 = w * cpw;                                        // first (newest) chunk of this warp
    const int j1 = j0 + cpw < nchunks ? j0 + cpw : nchunks;        // exclusive
    if (lane == 0) {
        for (int j = j0; j < j0 + cpw; ++j) mbar_init(bars + 8u * j, 1);
        fence_mbar_init();
        for (int j = j0; j < j1; ++j) {
            const uint32_t bar = bars + 8u * j;
            mbar_arrive_expect_tx(bar, GAE_L * (128u + 128u + 32u));
            const int t_lo = T - (j + 1) * GAE_L;
            tma_load_2d(smem_u32(&st[j].r[0][0]), &maps.r, e0, t_lo, bar);
            tma_load_2d(smem_u32(&st[j].v[0][0]), &maps.v, e0, t_lo, bar);
            tma_load_2d(smem_u32(&st[j].d[0][0]), &maps.d, e0, t_lo, bar);
        }
    }
    __syncthreads();   // every warp's barrier initialisation is visible before anyone waits on it
    if (NORM) {   // zero the statistics before anyone adds to them (the loads above are in flight meanwhile)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            stats[0] = 0.0;
            stats[1] = 0.0;
        }
        cooperative_groups::this_grid().sync();
    }
    for (int j = j0; j < j1; ++j) mbar_wait(bars + 8u * j, 0u);
    // V at the row just after this segment (first row of the newer warp's oldest chunk) or the bootstrap
    float v_in = boot[active ? e : e0];
    if (w > 0) {
        mbar_wait(bars + 8u * (j0 - 1), 0u);
        v_in = st[j0 - 1].v[0][lane];
    }
    // pass 1: local recurrence from A = 0 over rows t >= 0 of this segment
    float a_loc = 0.f, prod = 1.f, v_next = v_in;
    for (int j = j0; j < j1; ++j) {
        const int t_base = T - (j + 1) * GAE_L;
        const int q_lo = t_base < 0 ? -t_base : 0;
#pragma unroll 8
        for (int q = GAE_L - 1; q >= q_lo; --q) {
            const float r = st[j].r[q][lane];
            const float v = st[j].v[q][lane];
            const float nd = st[j].d[q][lane] ? 0.0f : 1.0f;
            const float delta = (r + gamma * nd * v_next) - v;
            const float c = gl * nd;
            a_loc = delta + c * a_loc;
            prod = prod * c;
            v_next = v;
        }
    }
    sum->aloc[w][lane] = a_loc;
    sum->prod[w][lane] = prod;
    __syncthreads();
    // combine: A entering this segment from the newer side
    float a_next = 0.f;
    for (int u = 0; u < w; ++u) a_next = sum->aloc[u][lane] + sum->prod[u][lane] * a_next;
    // pass 2: sequential recurrence from the exact entry state, same arithmetic as gae_row
    double s1 = 0.0, s2 = 0.0;
    v_next = v_in;
    for (int j = j0; j < j1; ++j) {
        const int t_base = T - (j + 1) * GAE_L;
        const int q_lo = t_base < 0 ? -t_base : 0;
#pragma unroll 8
        for (int q = GAE_L - 1; q >= q_lo; --q) {
            const float r = st[j].r[q][lane];
            const float v = st[j].v[q][lane];
            const float nd = st[j].d[q][lane] ? 0.0f : 1.0f;
            const float delta = (r + gamma * nd * v_next) - v;
            const float A = delta + gl * nd * a_next;
            if (active) {
                const int64_t i = static_cast<int64_t>(t_base + q) * N + e;
                if (NORM) st[j].r[q][lane] = A;   // r of this row is not read again
                else adv[i] = A;
                ret[i] = A + v;
                s1 += A;
                s2 += static_cast<double>(A) * A;
            }
            a_next = A;
            v_next = v;
        }
    }
    if (stats) gae_stats_flush(s1, s2, stats);
    if (NORM) {
        cooperative_groups::this_grid().sync();
        const double count = static_cast<double>(T) * N;
        const double m = __ldcg(stats) / count;
        const double var = __ldcg(stats + 1) / count - m * m;
        const float mf = static_cast<float>(m);
        const float inv = var > 0.0 ? static_cast<float>(1.0 / sqrt(var)) : 0.0f;
        if (active)
            for (int j = j0; j < j1; ++j) {
                const int t_base = T - (j + 1) * GAE_L;
                const int q_lo = t_base < 0 ? -t_base : 0;
                for (int q = GAE_L - 1; q >= q_lo; --q)
                    adv[static_cast<int64_t>(t_base + q) * N + e] = (st[j].r[q][lane] - mf) * inv;
            }
    }
}

// advantage normalisation in place (R#23): A <- (A - m) / s, m = S1 / count, s^2 = S2 / count - m^2
__global__ void adv_normalize_kernel(float* __restrict__ adv, int64_t count, const double* __restrict__ stats,
                                     int vec4) {
    const double m = stats[0] / static_cast<double>(count);
    const double var = stats[1] / static_cast<double>(count) - m * m;
    const float mf = static_cast<float>(m);
    const float inv = var > 0.0 ? static_cast<float>(1.0 / sqrt(var)) : 0.0f;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n4 = vec4 ? count / 4 : 0;
    float4* a4 = reinterpret_cast<float4*>(adv);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 x = a4[i];
        x.x = (x.x - mf) * inv;
        x.y = (x.y - mf) * inv;
        x.z = (x.z - mf) * inv;
        x.w = (x.w - mf) * inv;
        a4[i] = x;
    }
    for (int64_t i = 4 * n4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        adv[i] = (adv[i] - mf) * inv;
}

}  // namespace pod
