// actor_pair_kernel.cuh — K1 for agents whose envs fill M-tile PAIRS (per-agent
// env count a multiple of 256): the same method as actor_kernel.cuh (MLP chain
// + Gaussian head, R#6, R#12–R#14), mapped onto 4-CTA clusters that use
// the 2-SM tensor-core MMA.
//
//   cluster rank cr: mrow = cr & 1 (which of the cluster's two 128-env M-tiles),
//                    chalf = cr >> 1 (which half of every layer's output columns).
//   MMA pairs (0,1) and (2,3): tcgen05.mma.cta_group::2 with M = 256 (128 rows of
//   each M-tile, A from each CTA's own activation buffer), N = the column half,
//   B split across the pair (each CTA stages half of the weight rows).  Each SM
//   therefore reads only half of B per MMA: the shared-memory traffic per FLOP
//   that bounds the single-CTA (cta_group::1, SS) version halves, and each
//   weight byte fetched from L2 serves 256 rows.
//   Column halves exchange activation atoms through DSMEM bulk copies (cr ^ 2),
//   exactly as in actor_kernel.cuh; the pair's leader (mrow = 0) issues the MMAs
//   once both CTAs of the pair report their atoms ready (remote mbarrier arrives).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "actor_kernel.cuh"
#include "ptx.cuh"

namespace pod {

constexpr int AP_STAGES = 10;                       // 8 KB stages (this CTA's half of a 256 x 32 tile)
constexpr uint32_t AP_STAGE_BYTES = 128 * ACT_BK * 2;

inline size_t actor_pair_smem_bytes(int k_pad, int hidden) {
    const int ka = (k_pad > hidden ? k_pad : hidden) / 64;
    return 1024 + static_cast<size_t>(ka) * 16384 + static_cast<size_t>(AP_STAGES) * AP_STAGE_BYTES + ACT_BIAS_FLOATS * 4 +
           4 * 128 * 4 + 512;
}

__global__ void __launch_bounds__(ACT_THREADS, 1)
    actor_pair_kernel(const __grid_constant__ ActorMaps maps, const ActorArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t cr = cluster_ctarank();
    const uint32_t mrow = cr & 1u;                      // M-tile within the cluster / role in the MMA pair
    const uint32_t chalf = cr >> 1;                     // column half
    const uint32_t xpart = cr ^ 2u;                     // same M-tile, other column half
    const uint32_t leader = cr & ~1u;                   // MMA-issuing CTA of this pair
    const bool is_leader = mrow == 0;
    const uint16_t pair_mask = static_cast<uint16_t>(3u << leader);
    const int ka = (a.k_pad > a.hidden ? a.k_pad : a.hidden) / 64;
    const uint32_t act_s = base_u32;
    const uint32_t ring_s = act_s + ka * 16384u;
    const uint32_t bias_off = ka * 16384u + AP_STAGES * AP_STAGE_BYTES;
    float* bias_s = reinterpret_cast<float*>(base + bias_off);
    float* logp_s = bias_s + ACT_BIAS_FLOATS;                                  // [4][128]
    const uint32_t bar_s = base_u32 + bias_off + ACT_BIAS_FLOATS * 4 + 4 * 128 * 4;
    const uint32_t full_b = bar_s;                                   // [STAGES] (leader)
    const uint32_t empty_b = bar_s + 8u * AP_STAGES;                 // [STAGES]
    const uint32_t obs_b = bar_s + 16u * AP_STAGES;                  // (leader)
    const uint32_t accum_b = obs_b + 8u;
    const uint32_t ownrdy_b = obs_b + 16u;       // [4] local atom written (256 arrivals)
    const uint32_t ownpair_b = obs_b + 48u;      // [4] (leader) the non-leader's atom written
    const uint32_t peerrdy_b = obs_b + 80u;      // [4] the other column half's atom landed here
    const uint32_t peerpair_b = obs_b + 112u;    // [4] (leader) ... landed in the non-leader
    const uint32_t tslot_s = obs_b + 144u;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(base + (tslot_s - base_u32));

    const int mtile = a.mtile0 + 2 * static_cast<int>(blockIdx.x >> 2) + static_cast<int>(mrow);
    const int agent = mtile / a.tiles_per_agent;
    const int tile_in_agent = mtile % a.tiles_per_agent;
    const int env0 = agent * a.per_agent + tile_in_agent * 128;
    const int rows_valid = 128;                      // per-agent env count is a multiple of 256

    const int hid_half = a.hidden / 2;
    const int head_half = a.n_out_pad / 2;
    const int na = hid_half / 64;                    // activation atoms per column half
    const uint32_t tbuf = static_cast<uint32_t>(hid_half > head_half ? hid_half : head_half);
    uint32_t tcols = 32;
    while (tcols < 2 * tbuf) tcols <<= 1;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < AP_STAGES; ++s) {
                mbar_init(full_b + 8u * s, 1);
                mbar_init(empty_b + 8u * s, 1);
            }
            mbar_init(obs_b, 1);
            mbar_init(accum_b, 2);        // one commit from each pair's leader
            for (int j = 0; j < 4; ++j) {
                mbar_init(ownrdy_b + 8u * j, 256);
                mbar_init(ownpair_b + 8u * j, 1);
                mbar_init(peerrdy_b + 8u * j, 1);
                mbar_init(peerpair_b + 8u * j, 1);
            }
            fence_mbar_init();
            prefetch_tmap(&maps.obs);
            for (int l = 0; l < a.n_layers; ++l) prefetch_tmap(&maps.w[l]);
        }
        __syncwarp();
        tmem_alloc_cta2(tslot_s, tcols);
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    unsigned long long* tr = a.trace ? a.trace + blockIdx.x * 64 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = clock64();

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            const int kbo = a.k_pad / 64;
            const uint32_t obs_lead = mapa_shared(obs_b, leader);
            if (is_leader) mbar_arrive_expect_tx(obs_b, 2u * static_cast<uint32_t>(kbo) * 16384u);
            for (int kb = 0; kb < kbo; ++kb)
                tma_load_2d_cta2(act_s + kb * 16384u, &maps.obs, kb * 64, a.obs_row0 + env0, obs_lead);
            int stage = 0;
            uint32_t phase = 0;
            for (int l = 0; l < a.n_layers; ++l) {
                const int K = l == 0 ? a.k_pad : a.hidden;
                const int half = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad) / 2;
                const int rows = half / 2;                                  // this CTA's share of B
                const int KB = K / ACT_BK;
                const int kb0 = l == 0 ? 0 : static_cast<int>(chalf) * na * 2;
                for (int j = 0; j < KB; ++j) {
                    const int kb = (j + kb0) % KB;
                    mbar_wait(empty_b + 8u * stage, phase ^ 1u);
                    if (is_leader) mbar_arrive_expect_tx(full_b + 8u * stage, 2u * static_cast<uint32_t>(rows) * (ACT_BK * 2));
                    tma_load_3d_cta2(ring_s + stage * AP_STAGE_BYTES, &maps.w[l], kb * ACT_BK,
                                     static_cast<int>(chalf) * half + static_cast<int>(mrow) * rows, agent,
                                     mapa_shared(full_b + 8u * stage, leader));
                    if (++stage == AP_STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            if (is_leader) {
                // ===================== MMA issuer (pair leader) =====================
                mbar_wait(obs_b, 0);
                tc_fence_after();
                if (tr) tr[1] = clock64();
                const uint64_t adesc0 = sw128_desc(act_s);
                const uint64_t bdesc0 = sw64_desc(ring_s);
                int stage = 0;
                uint32_t phase = 0;
                for (int l = 0; l < a.n_layers; ++l) {
                    const int K = l == 0 ? a.k_pad : a.hidden;
                    const int half = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad) / 2;
                    const uint32_t idesc = idesc_bf16_f32(256, static_cast<uint32_t>(half));
                    const int KB = K / ACT_BK;
                    const int kb0 = l == 0 ? 0 : static_cast<int>(chalf) * na * 2;
                    const uint32_t par = static_cast<uint32_t>(l - 1) & 1u;
                    if (tr) tr[2 + 4 * l] = clock64();
                    for (int j = 0; j < KB; ++j) {
                        const int kb = j + kb0 < KB ? j + kb0 : j + kb0 - KB;
                        if (l > 0 && (j & 1) == 0) {
                            const int ja = j >> 1;
                            if (ja < na) {          // own column half: written by both CTAs' epilogues
                                mbar_wait(ownrdy_b + 8u * ja, par);
                                mbar_wait_cluster(ownpair_b + 8u * ja, par);
                            } else {                // other column half: DSMEM copies into both CTAs
                                mbar_arrive_expect_tx(peerrdy_b + 8u * (ja - na), 16384u);
                                mbar_wait(peerrdy_b + 8u * (ja - na), par);
                                mbar_wait_cluster(peerpair_b + 8u * (ja - na), par);
                            }
                            tc_fence_after();
                        }
                        mbar_wait(full_b + 8u * stage, phase);
                        tc_fence_after();
                        if (tr && l == 0 && j < 16) tr[32 + j] = clock64();
                        const uint64_t ad = adesc0 + (((kb >> 1) * 16384u + (kb & 1) * 64u) >> 4);
                        const uint64_t bd = bdesc0 + ((stage * AP_STAGE_BYTES) >> 4);
                        const uint32_t dt = tmem + (static_cast<uint32_t>(l) & 1u) * tbuf;
                        mma_bf16_cta2(dt, ad, bd, idesc, j != 0);
                        mma_bf16_cta2(dt, ad + 2, bd + 2, idesc, 1u);
                        mma_commit_cta2_mc(empty_b + 8u * stage, pair_mask);
                        if (++stage == AP_STAGES) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    if (tr) tr[3 + 4 * l] = clock64();
                    mma_commit_cta2_mc(accum_b, 0xF);     // every CTA of the cluster
                }
            } else {
                // ===== non-leader: forward "the other half's atom landed here" to the leader
                for (int l = 1; l < a.n_layers; ++l) {
                    const uint32_t par = static_cast<uint32_t>(l - 1) & 1u;
                    for (int ja = 0; ja < na; ++ja) {
                        mbar_arrive_expect_tx(peerrdy_b + 8u * ja, 16384u);
                        mbar_wait(peerrdy_b + 8u * ja, par);
                        mbar_arrive_remote(mapa_shared(peerpair_b + 8u * ja, leader));
                    }
                }
            }
        }
        __syncwarp();
    } else {
        // ===================== epilogue (warps 2..9) =====================
        const int ew = warp - 2;
        const int etid = ew * 32 + lane;
        const int quad = warp & 3;
        const int hh = ew >> 2;
        const int r = quad * 32 + lane;
        const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const int e = env0 + r;
        const bool valid = r < rows_valid && e < a.N;
        const char* slab = a.params + agent * a.param_bytes;
        {
            int off = 0;
            for (int l = 0; l < a.n_layers; ++l) {
                const int half = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad) / 2;
                const float* b = reinterpret_cast<const float*>(slab + a.b_off[l]) + chalf * half;
                for (int j = etid; j < half; j += 256) bias_s[off + j] = b[j];
                off += half;
            }
            const float* ls = reinterpret_cast<const float*>(slab + a.log_std_off) + chalf * head_half;
            for (int j = etid; j < head_half; j += 256) {
                bias_s[off + j] = ls[j];
                bias_s[off + head_half + j] = expf(ls[j]);
            }
        }
        const int hq = head_half / 2;
        float zr[ACT_MAX_HQ];
#pragma unroll
        for (int q = 0; q < ACT_MAX_HQ; ++q) {
            const int i = static_cast<int>(chalf) * head_half + hh * hq + q;
            zr[q] = (q < hq && valid && i < a.n && !a.deterministic) ? a.znoise[static_cast<int64_t>(i) * a.N + e] : 0.0f;
        }
        named_bar_sync(1, 256);
        int boff = 0;
        for (int l = 0; l < a.n_layers - 1; ++l) {
            mbar_wait_cluster(accum_b, static_cast<uint32_t>(l) & 1u);   // both pairs done reading h_l
            tc_fence_after();
            if (tr && etid == 0) tr[4 + 4 * l] = clock64();
            for (int j = 0; j < na; ++j) {
                const int tc = j * 64 + hh * 32;
                uint32_t v[32];
                tmem_ld32(trow + (static_cast<uint32_t>(l) & 1u) * tbuf + static_cast<uint32_t>(tc), v);
                tmem_ld_wait();
                const float4* b4 = reinterpret_cast<const float4*>(bias_s + boff + tc);
                uint32_t pk[16];
                epi_pack(v, b4, a.act, pk);
                const int atom_g = static_cast<int>(chalf) * na + j;
                const uint32_t atom = act_s + static_cast<uint32_t>(atom_g) * 16384u;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    st_shared_v4(atom + sw128_offset(static_cast<uint32_t>(r), static_cast<uint32_t>(hh * 4 + q)),
                                 pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(ownrdy_b + 8u * j);
                if (etid == 0) {
                    mbar_wait(ownrdy_b + 8u * j, static_cast<uint32_t>(l) & 1u);
                    // the atom to the other column half of this M-tile ...
                    bulk_s2peer(mapa_shared(atom, xpart), atom, 16384u, mapa_shared(peerrdy_b + 8u * j, xpart));
                    // ... and "written" to this pair's MMA issuer
                    if (!is_leader) mbar_arrive_remote(mapa_shared(ownpair_b + 8u * j, leader));
                }
            }
            boff += hid_half;
            if (tr && etid == 0) tr[5 + 4 * l] = clock64();
        }
        // ----- head
        const int L = a.n_layers - 1;
        mbar_wait_cluster(accum_b, static_cast<uint32_t>(L) & 1u);
        tc_fence_after();
        if (tr && etid == 0) tr[24] = clock64();
        const float* bias = bias_s + boff;
        const float* log_std = bias_s + boff + head_half;
        const float* sigma = bias_s + boff + 2 * head_half;
        float logp = 0.0f;
        bool bad = false;
        const float half_ln_2pi = 0.918938533204672742f;
        const bool vec = (a.n % 4) == 0;
#pragma unroll
        for (int cc = 0; cc < ACT_MAX_HQ / 8; ++cc) {
            if (cc >= hq / 8) break;
            const int tc = hh * hq + cc * 8;
            const int i0 = static_cast<int>(chalf) * head_half + tc;
            uint32_t hv[8];
            __syncwarp();
            tmem_ld8(trow + (static_cast<uint32_t>(L) & 1u) * tbuf + static_cast<uint32_t>(tc), hv);
            tmem_ld_wait();
            if (valid && i0 < a.n) {
                float raw[8], mu[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int i = i0 + jj;
                    mu[jj] = __uint_as_float(hv[jj]) + bias[tc + jj];
                    raw[jj] = mu[jj];
                    if (i < a.n) {
                        const float z = zr[cc * 8 + jj];
                        const float ls = log_std[tc + jj];
                        bad |= !isfinite(mu[jj]);
                        raw[jj] = fmaf(sigma[tc + jj], z, mu[jj]);
                        logp += (-0.5f * z * z - ls) - half_ln_2pi;
                        const float u = tanh_sfu(raw[jj]);
                        const double m = floor(static_cast<double>(fabsf(u)) * static_cast<double>(a.h_max) + 0.5);
                        const int ai = u < 0.0f ? -static_cast<int>(m) : static_cast<int>(m);
                        a.aint[static_cast<int64_t>(i) * a.N + e] = static_cast<int16_t>(ai);
                        if (a.dbg_aint) a.dbg_aint[static_cast<int64_t>(e) * a.n + i] = static_cast<int16_t>(ai);
                    }
                }
                float* arow = a.act_out + static_cast<int64_t>(e) * a.n + i0;
                float* mrow_p = a.mu_out ? a.mu_out + static_cast<int64_t>(e) * a.n + i0 : nullptr;
                if (vec && i0 + 8 <= a.n) {
                    reinterpret_cast<float4*>(arow)[0] = make_float4(raw[0], raw[1], raw[2], raw[3]);
                    reinterpret_cast<float4*>(arow)[1] = make_float4(raw[4], raw[5], raw[6], raw[7]);
                    if (mrow_p) {
                        reinterpret_cast<float4*>(mrow_p)[0] = make_float4(mu[0], mu[1], mu[2], mu[3]);
                        reinterpret_cast<float4*>(mrow_p)[1] = make_float4(mu[4], mu[5], mu[6], mu[7]);
                    }
                } else {
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        if (i0 + jj < a.n) {
                            arow[jj] = raw[jj];
                            if (mrow_p) mrow_p[jj] = mu[jj];
                        }
                    }
                }
            }
        }
        if (bad && valid) atomicOr(a.err, 1u);
        if (tr && etid == 0) tr[25] = clock64();
        // log-prob partial (chalf, hh) of row r -> logp_s of this M-tile's column-half-0 CTA (rank mrow)
        st_cluster_f32(mapa_shared(smem_u32(logp_s + (chalf * 2 + hh) * 128 + r), mrow), logp);
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp >= 2 && chalf == 0) {
        const int ew = warp - 2;
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        const int e = env0 + r;
        if ((ew >> 2) == 0 && r < rows_valid && e < a.N)
            a.logp_out[e] = ((logp_s[r] + logp_s[128 + r]) + logp_s[256 + r]) + logp_s[384 + r];
    }
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_cta2(tmem, tcols);
    }
    if (tr && threadIdx.x == 0) tr[26] = clock64();
}

}  // namespace pod
