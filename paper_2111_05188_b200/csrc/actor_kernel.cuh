// actor_kernel.cuh — K1: the actor MLP forward over a 128-env M-tile on the
// 5th-generation tensor cores, fused with the Gaussian sampling head.
//
// Method ("a policy network parameterised by theta maps a state to an
// action vector over n stocks"; Gaussian head with state-independent log-std,
// DESIGN.md R#12; hidden activation R#13; action map R#6; noise R#14):
//   h_0 = s_t,  h_{l+1} = act(W_l h_l + b_l),  mu = W_L h_L + b_L
//   raw = mu + exp(log_std) z,  logp = sum_i(-z_i^2/2 - log_std_i - ln(2 pi)/2),
//   u = tanh(raw),  a_i = sgn(u_i) floor(|u_i| h_max + 1/2).
//
// B200 design (one CTA per 128-row tile of envs, all layers fused on chip):
//   * warp 0 (one lane): TMA producer — the obs tile [128 x k_pad] bf16 into the
//     activation buffer, then every weight tile W_l[BN x 64] through a
//     STAGES-deep ring (128B-swizzled, 3-D tensor map over [agent][out][in]);
//   * warp 1 (one lane): tcgen05.mma issuer, M=128, N=BN<=256, K=16 steps,
//     A = activations in smem, B = weight ring, D = fp32 accumulator in TMEM;
//   * warps 2..5: epilogue — tcgen05.ld of their 32-lane TMEM quadrant, bias +
//     activation, bf16 pack, swizzled st.shared back into the activation buffer
//     (it becomes the A operand of the next layer: activations never leave the
//     SM), and for the head the sampling epilogue writing act/logp/mu and the
//     integer action a_t (ticker-major scratch for the env-step kernel).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "philox.cuh"
#include "ptx.cuh"

namespace pod {

constexpr int ACT_THREADS = 192;       // 6 warps
constexpr int ACT_STAGES = 3;          // weight ring depth
constexpr int ACT_MAX_LAYERS = 5;      // n_hidden <= 4

struct ActorArgs {
    int32_t N;               // envs
    int32_t per_agent;       // envs per agent
    int32_t tiles_per_agent; // ceil(per_agent / 128)
    int32_t n;               // stocks
    int32_t n_out_pad;       // head rows (n rounded to 16)
    int32_t k_pad;           // obs row width
    int32_t hidden;
    int32_t n_layers;        // n_hidden + 1
    int32_t act;             // 0 relu, 1 tanh
    int32_t h_max;
    int32_t deterministic;
    int32_t t;               // step within the rollout
    int32_t obs_row0;        // row of obs[t][0] in the obs tensor map = t * N
    int32_t bn_max;          // ring stage rows
    uint64_t seed;
    int64_t env_offset;
    const uint64_t* step_base;   // device step counter of the handle
    const char* params;          // [agents][param_bytes]
    uint64_t param_bytes;
    uint64_t b_off[ACT_MAX_LAYERS];
    uint64_t log_std_off;
    float* act_out;      // [N][n] at step t (raw)
    float* logp_out;     // [N]
    float* mu_out;       // [N][n] or null
    int16_t* aint;       // [n][N] scratch
    int16_t* dbg_aint;   // [N][n] or null
    uint32_t* err;
};

struct ActorMaps {
    CUtensorMap obs;                     // 2-D bf16 [rows][k_pad], box {64, 128}
    CUtensorMap w[ACT_MAX_LAYERS];       // 3-D bf16 [agents][out][in], box {64, BN_l, 1}
};

__device__ __forceinline__ float act_fn(float x, int act) { return act == 0 ? fmaxf(x, 0.0f) : tanhf(x); }

__global__ void __launch_bounds__(ACT_THREADS, 1)
    actor_forward_kernel(const __grid_constant__ ActorMaps maps, const ActorArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the swizzle atoms
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ka = (a.k_pad > a.hidden ? a.k_pad : a.hidden) / 64;   // activation atoms
    const uint32_t act_s = base_u32;                                  // ka * 16 KB
    const uint32_t ring_s = act_s + ka * 16384u;
    const uint32_t stage_bytes = static_cast<uint32_t>(a.bn_max) * 128u;
    const uint32_t bar_s = ring_s + ACT_STAGES * stage_bytes;        // 8-byte barriers
    const uint32_t full_b = bar_s;                                   // [STAGES]
    const uint32_t empty_b = bar_s + 8u * ACT_STAGES;                // [STAGES]
    const uint32_t obs_b = bar_s + 16u * ACT_STAGES;
    const uint32_t accum_b = obs_b + 8u;
    const uint32_t actrdy_b = obs_b + 16u;
    const uint32_t tslot_s = obs_b + 24u;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(base + (tslot_s - base_u32));

    const int agent = blockIdx.x / a.tiles_per_agent;
    const int tile_in_agent = blockIdx.x % a.tiles_per_agent;
    const int env0 = agent * a.per_agent + tile_in_agent * 128;
    int rows_valid = a.per_agent - tile_in_agent * 128;
    rows_valid = rows_valid > 128 ? 128 : rows_valid;

    uint32_t tcols = 32;
    {
        const int need = a.hidden > a.n_out_pad ? a.hidden : a.n_out_pad;
        while (tcols < static_cast<uint32_t>(need)) tcols <<= 1;
    }

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < ACT_STAGES; ++s) {
                mbar_init(full_b + 8u * s, 1);
                mbar_init(empty_b + 8u * s, 1);
            }
            mbar_init(obs_b, 1);
            mbar_init(accum_b, 1);
            mbar_init(actrdy_b, 128);
            fence_mbar_init();
            prefetch_tmap(&maps.obs);
            for (int l = 0; l < a.n_layers; ++l) prefetch_tmap(&maps.w[l]);
        }
        __syncwarp();
        tmem_alloc(tslot_s, tcols);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const int kb0 = a.k_pad / 64;
            mbar_arrive_expect_tx(obs_b, static_cast<uint32_t>(kb0) * 16384u);
            for (int kb = 0; kb < kb0; ++kb)
                tma_load_2d(act_s + kb * 16384u, &maps.obs, kb * 64, a.obs_row0 + env0, obs_b);
            int stage = 0;
            uint32_t phase = 0;
            for (int l = 0; l < a.n_layers; ++l) {
                const int K = l == 0 ? a.k_pad : a.hidden;
                const int Nl = l == a.n_layers - 1 ? a.n_out_pad : a.hidden;
                const int bn = Nl > 256 ? 256 : Nl;
                const int nchunks = Nl / bn;
                for (int c = 0; c < nchunks; ++c) {
                    for (int kb = 0; kb < K / 64; ++kb) {
                        mbar_wait(empty_b + 8u * stage, phase ^ 1u);
                        mbar_arrive_expect_tx(full_b + 8u * stage, static_cast<uint32_t>(bn) * 128u);
                        tma_load_3d(ring_s + stage * stage_bytes, &maps.w[l], kb * 64, c * bn, agent,
                                    full_b + 8u * stage);
                        if (++stage == ACT_STAGES) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            mbar_wait(obs_b, 0);
            tc_fence_after();
            int stage = 0;
            uint32_t phase = 0;
            for (int l = 0; l < a.n_layers; ++l) {
                if (l > 0) {
                    mbar_wait(actrdy_b, static_cast<uint32_t>(l - 1) & 1u);
                    tc_fence_after();
                }
                const int K = l == 0 ? a.k_pad : a.hidden;
                const int Nl = l == a.n_layers - 1 ? a.n_out_pad : a.hidden;
                const int bn = Nl > 256 ? 256 : Nl;
                const int nchunks = Nl / bn;
                const uint32_t idesc = idesc_bf16_f32(128, bn);
                for (int c = 0; c < nchunks; ++c) {
                    for (int kb = 0; kb < K / 64; ++kb) {
                        mbar_wait(full_b + 8u * stage, phase);
                        tc_fence_after();
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint64_t ad = sw128_desc(act_s + kb * 16384u + k * 32u);
                            const uint64_t bd = sw128_desc(ring_s + stage * stage_bytes + k * 32u);
                            mma_bf16(tmem + static_cast<uint32_t>(c * bn), ad, bd, idesc, (kb | k) != 0);
                        }
                        mma_commit(empty_b + 8u * stage);
                        if (++stage == ACT_STAGES) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                }
                mma_commit(accum_b);
            }
        }
        __syncwarp();
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int r = quad * 32 + lane;            // row of the tile == TMEM lane
        const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const int e = env0 + r;
        const bool valid = r < rows_valid && e < a.N;
        for (int l = 0; l < a.n_layers - 1; ++l) {
            mbar_wait(accum_b, static_cast<uint32_t>(l) & 1u);
            tc_fence_after();
            const float* bias = reinterpret_cast<const float*>(a.params + agent * a.param_bytes + a.b_off[l]);
            for (int cc = 0; cc < a.hidden / 32; ++cc) {
                uint32_t v[32];
                tmem_ld32(trow + static_cast<uint32_t>(cc * 32), v);
                tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float x0 = act_fn(__uint_as_float(v[2 * j]) + __ldg(bias + cc * 32 + 2 * j), a.act);
                    const float x1 = act_fn(__uint_as_float(v[2 * j + 1]) + __ldg(bias + cc * 32 + 2 * j + 1), a.act);
                    pk[j] = pack_bf16x2(x0, x1);
                }
                const uint32_t atom = act_s + static_cast<uint32_t>((cc * 32) / 64) * 16384u;
                const uint32_t c0 = static_cast<uint32_t>(((cc * 32) % 64) / 8);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    st_shared_v4(atom + sw128_offset(static_cast<uint32_t>(r), c0 + q), pk[4 * q], pk[4 * q + 1],
                                 pk[4 * q + 2], pk[4 * q + 3]);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(actrdy_b);
        }
        // ----- head: mean, Gaussian sample, log-prob, squash, integer action
        const int L = a.n_layers - 1;
        mbar_wait(accum_b, static_cast<uint32_t>(L) & 1u);
        tc_fence_after();
        const char* slab = a.params + agent * a.param_bytes;
        const float* bias = reinterpret_cast<const float*>(slab + a.b_off[L]);
        const float* log_std = reinterpret_cast<const float*>(slab + a.log_std_off);
        const uint64_t step = *a.step_base + static_cast<uint64_t>(a.t);
        const uint32_t eg = static_cast<uint32_t>(a.env_offset + e);
        float logp = 0.0f;
        bool bad = false;
        const float half_ln_2pi = 0.918938533204672742f;
        for (int cc = 0; cc * 32 < a.n; ++cc) {
            uint32_t v[32];
            __syncwarp();
            tmem_ld32(trow + static_cast<uint32_t>(cc * 32), v);   // warp-collective
            tmem_ld_wait();
            if (valid) {
            float raw[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                const int i0 = cc * 32 + q * 4;
                if (!a.deterministic && i0 < a.n) z = normals4(a.seed, eg, step, static_cast<uint32_t>(i0 / 4));
                const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int i = i0 + j;
                    const int jj = q * 4 + j;
                    if (i < a.n) {
                        const float mu = __uint_as_float(v[jj]) + __ldg(bias + i);
                        const float ls = __ldg(log_std + i);
                        bad |= !isfinite(mu);
                        raw[jj] = fmaf(expf(ls), zz[j], mu);
                        logp += (-0.5f * zz[j] * zz[j] - ls) - half_ln_2pi;
                        v[jj] = __float_as_uint(mu);
                        const float u = tanhf(raw[jj]);
                        const double m = floor(static_cast<double>(fabsf(u)) * static_cast<double>(a.h_max) + 0.5);
                        const int ai = u < 0.0f ? -static_cast<int>(m) : static_cast<int>(m);
                        a.aint[static_cast<int64_t>(i) * a.N + e] = static_cast<int16_t>(ai);
                        if (a.dbg_aint) a.dbg_aint[static_cast<int64_t>(e) * a.n + i] = static_cast<int16_t>(ai);
                    }
                }
            }
            float* arow = a.act_out + static_cast<int64_t>(e) * a.n + cc * 32;
            float* mrow = a.mu_out ? a.mu_out + static_cast<int64_t>(e) * a.n + cc * 32 : nullptr;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
                if (cc * 32 + jj < a.n) {
                    arow[jj] = raw[jj];
                    if (mrow) mrow[jj] = __uint_as_float(v[jj]);
                }
            }
            }
        }
        if (valid) {
            a.logp_out[e] = logp;
            if (bad) atomicOr(a.err, 1u);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, tcols);
    }
}

}  // namespace pod
