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
// [L time rows x 32 envs] chunks in shared memory, every row fetched by one
// lane with cp.async.bulk (TMA engine, completion on an mbarrier with
// expect_tx), so STAGES x L x 288 B per warp are in flight while the lanes
// run the recurrence out of shared memory.  Outputs are written with
// coalesced 128-B row stores.  Each chunk arrives as three 2-D TMA boxes
// ({32 envs x 32 steps} of r, V, d) issued by one lane (rows before t = 0 and
// columns past N are zero-filled by the TMA unit); misaligned inputs
// (N % 16 != 0) use the plain-load path (same arithmetic, same order).
#pragma once
#include <cstdint>

#include <cuda.h>

#include "ptx.cuh"

namespace pod {

constexpr int GAE_L = 32;        // time rows per chunk
constexpr int GAE_STAGES = 4;    // chunks in flight per warp
constexpr int GAE_WARPS = 2;     // warps per block

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

struct GaeMaps {
    CUtensorMap r, v, d;   // 2-D [T][N], box {32, 32}
};

__global__ void __launch_bounds__(32 * GAE_WARPS)
    gae_kernel(const __grid_constant__ GaeMaps maps, const float* __restrict__ rew, const float* __restrict__ val,
               const uint8_t* __restrict__ done, const float* __restrict__ boot, int T, int N, float gamma,
               float lambda, float* __restrict__ adv, float* __restrict__ ret, int use_bulk) {
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

    const bool bulk = use_bulk != 0;
    if (!bulk) {
        for (int t = T - 1; t >= 0; --t) {
            if (active) {
                const int64_t i = static_cast<int64_t>(t) * N + e;
                gae_row(rew[i], val[i], done[i], gamma, gl, v_next, a_next, adv + i, ret + i);
            }
        }
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
        const int t_hi = T - j * GAE_L;
        const int t_lo = t_hi - GAE_L > 0 ? t_hi - GAE_L : 0;
        const int rows = t_hi - t_lo;
        for (int q = GAE_L - 1; q >= GAE_L - rows; --q) {
            const int t = t_lo + (q - (GAE_L - rows));
            const int64_t i = static_cast<int64_t>(t) * N + e;
            float A = 0.f, R = 0.f;
            gae_row(st[s].r[q][lane], st[s].v[q][lane], st[s].d[q][lane], gamma, gl, v_next, a_next, &A, &R);
            if (active) {
                adv[i] = A;
                ret[i] = R;
            }
        }
        __syncwarp();
        fence_proxy_async_smem();   // order this stage's generic reads before the async refill
        if (j + GAE_STAGES < nchunks) issue(j + GAE_STAGES);
    }
}

inline size_t gae_smem_bytes() { return GAE_WARPS * (GAE_STAGES * sizeof(GaeStage) + 128); }

}  // namespace pod
