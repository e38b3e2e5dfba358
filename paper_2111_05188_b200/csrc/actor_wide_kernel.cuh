// actor_wide_kernel.cuh — K1 on 2-CTA clusters with the 2-SM tensor-core MMA and NO column split:
// the same method as actor_kernel.cuh (MLP chain + Gaussian head, R#6, R#12–R#14, critic R#22).
//
//   cluster rank mrow (0 = leader): which of the pair's two 128-env M-tiles this CTA holds.
//   Every layer: tcgen05.mma.cta_group::2 with M = 256 (A = each CTA's own activation buffer), N = the
//   whole layer width in chunks of <= 256 columns (TMEM columns [c cw, (c+1) cw) of both CTAs), B split
//   across the pair (each CTA stages half of each chunk's weight rows).  So each CTA streams the same
//   weight bytes as a CTA of the column-split kernel but for twice the rows, and no activation leaves
//   the CTA (no DSMEM exchange).  The epilogue of a CTA writes all of h_{l+1} for its 128 rows.
//   TMEM holds one layer (up to 512 fp32 columns): layer l+1's first chunk overwrites the columns the
//   epilogue of layer l reads first, so its MMAs start once those atoms are read (atom by atom after).
//   The leader issues the MMAs once both CTAs report an atom written (local + remote mbarrier arrivals).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "actor_kernel.cuh"
#include "ptx.cuh"

namespace pod {

constexpr int AW_STAGES = 10;                         // 8 KB stages (this CTA's half of a 256 x 32 tile)
constexpr uint32_t AW_STAGE_BYTES = 128 * ACT_BK * 2;
constexpr int AW_BIAS_FLOATS = 2048;                  // all biases + log-std + sigma of one agent
constexpr int AW_MAX_ATOMS = 8;                       // hidden <= 512

inline size_t actor_wide_smem_bytes(int k_pad, int hidden) {
    const int ka = (k_pad > hidden ? k_pad : hidden) / 64;
    return 1024 + static_cast<size_t>(ka) * 16384 + static_cast<size_t>(AW_STAGES) * AW_STAGE_BYTES +
           AW_BIAS_FLOATS * 4 + 4 * 128 * 4 + 512;
}
// eligible shapes: per-agent env count a multiple of 256 (pairs never straddle agents), hidden a multiple
// of 128 up to 512, every bias of the agent staged at once
inline bool actor_wide_ok(int per_agent, int n_hidden, int hidden, int n_out_pad) {
    return per_agent % 256 == 0 && hidden % 128 == 0 && hidden <= 512 && n_out_pad <= 128 &&
           n_hidden * hidden + 3 * n_out_pad <= AW_BIAS_FLOATS;
}
__host__ __device__ inline int actor_wide_cw(int out) { return out < 256 ? out : 256; }

__global__ void __launch_bounds__(ACT_THREADS, 1)
    actor_wide_kernel(const __grid_constant__ ActorMaps maps, const ActorArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t mrow = cluster_ctarank();            // M-tile of the pair / role in the MMA pair
    const bool is_leader = mrow == 0;
    const uint16_t pair_mask = 3u;
    const int ka = (a.k_pad > a.hidden ? a.k_pad : a.hidden) / 64;
    const uint32_t act_s = base_u32;
    const uint32_t ring_s = act_s + ka * 16384u;
    const uint32_t bias_off = ka * 16384u + AW_STAGES * AW_STAGE_BYTES;
    float* bias_s = reinterpret_cast<float*>(base + bias_off);
    float* logp_s = bias_s + AW_BIAS_FLOATS;                                   // [4 quarters][128]
    const uint32_t bar_s = base_u32 + bias_off + AW_BIAS_FLOATS * 4 + 4 * 128 * 4;
    const uint32_t full_b = bar_s;                                   // [STAGES] (leader: both CTAs' bytes)
    const uint32_t empty_b = bar_s + 8u * AW_STAGES;                 // [STAGES]
    const uint32_t obs_b = bar_s + 16u * AW_STAGES;                  // (leader)
    const uint32_t accum_b = obs_b + 8u;                             // a layer's MMAs complete (both CTAs)
    const uint32_t ownrdy_b = obs_b + 16u;                           // [8] local atom written (256 arrivals)
    const uint32_t ownpair_b = ownrdy_b + 8u * AW_MAX_ATOMS;         // [8] (leader) the other CTA's atom
    const uint32_t tslot_s = ownpair_b + 8u * AW_MAX_ATOMS;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(base + (tslot_s - base_u32));

    const int mtile = a.mtile0 + 2 * static_cast<int>(blockIdx.x >> 1) + static_cast<int>(mrow);
    const int agent = mtile / a.tiles_per_agent;
    const int tile_in_agent = mtile % a.tiles_per_agent;
    const int env0 = agent * a.per_agent + tile_in_agent * 128;
    const int na = a.hidden / 64;                    // activation atoms of a hidden layer
    constexpr uint32_t tcols = 512;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < AW_STAGES; ++s) {
                mbar_init(full_b + 8u * s, 1);
                mbar_init(empty_b + 8u * s, 1);
            }
            mbar_init(obs_b, 1);
            mbar_init(accum_b, 1);
            for (int j = 0; j < AW_MAX_ATOMS; ++j) {
                mbar_init(ownrdy_b + 8u * j, 256);
                mbar_init(ownpair_b + 8u * j, 1);
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
    if (threadIdx.x == 0) pdl_launch_dependents();   // the env step may be scheduled (see env_kernel.cuh)
    const uint32_t tmem = *tslot;
    unsigned long long* tr = a.trace ? a.trace + blockIdx.x * 64 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = clock64();

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            const int kbo = a.k_pad / 64;
            const uint32_t obs_lead = mapa_shared(obs_b, 0);
            if (is_leader) mbar_arrive_expect_tx(obs_b, 2u * static_cast<uint32_t>(kbo) * 16384u);
            for (int kb = 0; kb < kbo; ++kb)
                tma_load_2d_cta2(act_s + kb * 16384u, &maps.obs, kb * 64, a.obs_row0 + env0, obs_lead);
            int stage = 0;
            uint32_t phase = 0;
            for (int l = 0; l < a.n_layers; ++l) {
                const int K = l == 0 ? a.k_pad : a.hidden;
                const int out = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad);
                const int cw = actor_wide_cw(out);
                const int rows = cw / 2;                                    // this CTA's share of B
                const int KB = K / ACT_BK;
                for (int c = 0; c < out / cw; ++c) {
                    for (int j = 0; j < KB; ++j) {
                        mbar_wait(empty_b + 8u * stage, phase ^ 1u);
                        if (is_leader)
                            mbar_arrive_expect_tx(full_b + 8u * stage, 2u * static_cast<uint32_t>(rows) * (ACT_BK * 2));
                        tma_load_3d_cta2(ring_s + stage * AW_STAGE_BYTES, &maps.w[l], j * ACT_BK,
                                         c * cw + static_cast<int>(mrow) * rows, agent,
                                         mapa_shared(full_b + 8u * stage, 0));
                        if (++stage == AW_STAGES) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0 && is_leader) {
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
                const int out = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad);
                const int cw = actor_wide_cw(out);
                const uint32_t idesc = idesc_bf16_f32(256, static_cast<uint32_t>(cw));
                const int KB = K / ACT_BK;
                const uint32_t par = static_cast<uint32_t>(l - 1) & 1u;
                // h_l atoms whose TMEM columns (of layer l-1) the first chunk overwrites
                const int first = ((cw + 63) / 64 < na) ? (cw + 63) / 64 : na;   // >= 1 (narrow heads too)
                if (tr) tr[2 + 4 * l] = clock64();
                for (int c = 0; c < out / cw; ++c) {
                    for (int j = 0; j < KB; ++j) {
                        if (l > 0 && c == 0 && (j & 1) == 0) {
                            const int ja = j >> 1;
                            if (ja == 0) {
                                for (int q = 0; q < first; ++q) {
                                    mbar_wait(ownrdy_b + 8u * q, par);
                                    mbar_wait_cluster(ownpair_b + 8u * q, par);
                                }
                            } else if (ja >= first) {
                                mbar_wait(ownrdy_b + 8u * ja, par);
                                mbar_wait_cluster(ownpair_b + 8u * ja, par);
                            }
                            tc_fence_after();
                        }
                        mbar_wait(full_b + 8u * stage, phase);
                        tc_fence_after();
                        if (tr && l == 0 && j < 16) tr[32 + j] = clock64();
                        const uint64_t ad = adesc0 + (((j >> 1) * 16384u + (j & 1) * 64u) >> 4);
                        const uint64_t bd = bdesc0 + ((stage * AW_STAGE_BYTES) >> 4);
                        const uint32_t dt = tmem + static_cast<uint32_t>(c * cw);
                        mma_bf16_cta2(dt, ad, bd, idesc, j != 0);
                        mma_bf16_cta2(dt, ad + 2, bd + 2, idesc, 1u);
                        mma_commit_cta2_mc(empty_b + 8u * stage, pair_mask);
                        if (++stage == AW_STAGES) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                }
                if (tr) tr[3 + 4 * l] = clock64();
                mma_commit_cta2_mc(accum_b, pair_mask);
            }
        } else if (lane == 0) {
            // non-leader: forward "atom j of h_l written here" to the leader's MMA issuer, so no epilogue
            // thread blocks on the whole-CTA barrier
            for (int l = 1; l < a.n_layers; ++l) {
                const uint32_t par = static_cast<uint32_t>(l - 1) & 1u;
                for (int j = 0; j < na; ++j) {
                    mbar_wait(ownrdy_b + 8u * j, par);
                    mbar_arrive_remote(mapa_shared(ownpair_b + 8u * j, 0));
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
        const bool valid = e < a.N;
        const char* slab = a.params + agent * a.param_bytes;
        const int nop = a.n_out_pad;
        {
            int off = 0;
            for (int l = 0; l < a.n_layers; ++l) {
                const int out = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad);
                const float* b = reinterpret_cast<const float*>(slab + a.b_off[l]);
                for (int j = etid; j < out; j += 256) bias_s[off + j] = b[j];
                off += out;
            }
            const float* ls = reinterpret_cast<const float*>(slab + a.log_std_off);
            for (int j = etid; j < nop; j += 256) {
                bias_s[off + j] = ls[j];
                bias_s[off + nop + j] = expf(ls[j]);
            }
        }
        const int nq = nop / 32;                       // 32-column quarters of the head (<= 4)
        // head noise of this thread's first quarter (q = hh), prefetched long before the head
        float zr[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const int i = hh * 32 + q;
            zr[q] = (hh < nq && valid && i < a.n && !a.deterministic) ? a.znoise[static_cast<int64_t>(i) * a.N + e]
                                                                       : 0.0f;
        }
        named_bar_sync(1, 256);
        int boff = 0;
        for (int l = 0; l < a.n_layers - 1; ++l) {
            mbar_wait_cluster(accum_b, static_cast<uint32_t>(l) & 1u);   // the pair's MMAs of layer l are done
            tc_fence_after();
            if (tr && etid == 0) tr[4 + 4 * l] = clock64();
            // TMEM loads one atom ahead: atom j+1's tcgen05.ld is in flight while atom j is packed
            // and stored (tcgen05.wait::ld waits for every outstanding load, so it is issued after the
            // wait for atom j)
            uint32_t v[32], vn[32];
            tmem_ld32(trow + static_cast<uint32_t>(hh * 32), v);
            for (int j = 0; j < na; ++j) {
                const int tc = j * 64 + hh * 32;
                tmem_ld_wait();
                if (j + 1 < na) tmem_ld32(trow + static_cast<uint32_t>(tc + 64), vn);
                const float4* b4 = reinterpret_cast<const float4*>(bias_s + boff + tc);
                uint32_t pk[16];
                epi_pack(v, b4, a.act, pk);
                const uint32_t atom = act_s + static_cast<uint32_t>(j) * 16384u;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    st_shared_v4(atom + sw128_offset(static_cast<uint32_t>(r), static_cast<uint32_t>(hh * 4 + q)),
                                 pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(ownrdy_b + 8u * j);
#pragma unroll
                for (int q = 0; q < 32; ++q) v[q] = vn[q];
            }
            tmem_ld_wait();
            boff += a.hidden;
            if (tr && etid == 0) tr[5 + 4 * l] = clock64();
        }
        // ----- head: quarters q = hh (pass 0) and q = hh + 2 (pass 1) of the n_out_pad columns
        const int L = a.n_layers - 1;
        mbar_wait_cluster(accum_b, static_cast<uint32_t>(L) & 1u);
        tc_fence_after();
        if (tr && etid == 0) tr[24] = clock64();
        const float* bias = bias_s + boff;
        const float* log_std = bias_s + boff + nop;
        const float* sigma = bias_s + boff + 2 * nop;
        const float half_ln_2pi = 0.918938533204672742f;
        const bool vec = (a.n % 4) == 0;
        bool bad = false;
        for (int pass = 0; pass < 2; ++pass) {
            const int q4 = 2 * pass + hh;
            float logp = 0.0f;
            if (pass == 1) {
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int i = q4 * 32 + q;
                    zr[q] = (q4 < nq && valid && i < a.n && !a.deterministic)
                                ? a.znoise[static_cast<int64_t>(i) * a.N + e]
                                : 0.0f;
                }
            }
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int tc = q4 * 32 + cc * 8;             // TMEM column == global ticker
                const int i0 = tc;
                uint32_t hv[8];
                __syncwarp();
                if (q4 < nq) {
                    tmem_ld8(trow + static_cast<uint32_t>(tc), hv);
                    tmem_ld_wait();
                }
                if (q4 >= nq) continue;
                if (valid && i0 <= a.n && a.val_out && a.n < i0 + 8) {
                    float vh = 0.0f;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if (i0 + jj == a.n) vh = __uint_as_float(hv[jj]);
                    a.val_out[e] = vh + bias[tc + (a.n - i0)];
                }
                if (valid && i0 < a.n && !a.value_only) {
                    float raw[8], mu[8];
                    int16_t ai8[8];
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        mu[jj] = __uint_as_float(hv[jj]) + bias[tc + jj];
                        raw[jj] = mu[jj];
                    }
                    auto sample = [&](int jj) {
                        const float z = zr[cc * 8 + jj];
                        const float ls = log_std[tc + jj];
                        bad |= !isfinite(mu[jj]);
                        raw[jj] = fmaf(sigma[tc + jj], z, mu[jj]);
                        logp += (-0.5f * z * z - ls) - half_ln_2pi;
                        const float u = tanh_sfu(raw[jj]);
                        const double m = floor(static_cast<double>(fabsf(u)) * static_cast<double>(a.h_max) + 0.5);
                        ai8[jj] = static_cast<int16_t>(u < 0.0f ? -static_cast<int>(m) : static_cast<int>(m));
                        a.aint[static_cast<int64_t>(i0 + jj) * a.N + e] = ai8[jj];
                    };
                    if (i0 + 8 <= a.n) {
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) sample(jj);
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            if (i0 + jj < a.n) sample(jj);
                    }
                    if (a.dbg_aint) {
                        for (int jj = 0; jj < 8 && i0 + jj < a.n; ++jj)
                            a.dbg_aint[static_cast<int64_t>(e) * a.n + i0 + jj] = ai8[jj];
                    }
                    float* arow = a.act_out + static_cast<int64_t>(e) * a.n + i0;
                    float* mrowp = a.mu_out ? a.mu_out + static_cast<int64_t>(e) * a.n + i0 : nullptr;
                    if (vec && i0 + 8 <= a.n) {
                        reinterpret_cast<float4*>(arow)[0] = make_float4(raw[0], raw[1], raw[2], raw[3]);
                        reinterpret_cast<float4*>(arow)[1] = make_float4(raw[4], raw[5], raw[6], raw[7]);
                        if (mrowp) {
                            reinterpret_cast<float4*>(mrowp)[0] = make_float4(mu[0], mu[1], mu[2], mu[3]);
                            reinterpret_cast<float4*>(mrowp)[1] = make_float4(mu[4], mu[5], mu[6], mu[7]);
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            if (i0 + jj < a.n) {
                                arow[jj] = raw[jj];
                                if (mrowp) mrowp[jj] = mu[jj];
                            }
                        }
                    }
                }
            }
            logp_s[q4 * 128 + r] = logp;
        }
        if (bad && valid) atomicOr(a.err, 1u);
        if (tr && etid == 0) tr[25] = clock64();
        named_bar_sync(1, 256);
        // the quarters in the column-split kernel's order: ((q0 + q1) + q2) + q3
        if (hh == 0 && valid && a.logp_out) {
            float s = logp_s[r];
            for (int q = 1; q < nq; ++q) s += logp_s[q * 128 + r];
            a.logp_out[e] = s;
        }
    }

    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_cta2(tmem, tcols);
    }
    if (tr && threadIdx.x == 0) tr[26] = clock64();
}

}  // namespace pod
