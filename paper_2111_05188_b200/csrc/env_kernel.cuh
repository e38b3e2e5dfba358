// env_kernel.cuh — K2: the fused stock-trading environment step.
//
// Method (Eqs. 3–4 transition, Eq. 2 reward, P:L220–226
// state; readings DESIGN.md R#1–R#5, R#8–R#10, R#17, R#18):
//   sells, tickers ascending:  q = min(h_i, -a_i); h_i -= q; b += (p_i q)(1 - c)
//   buys,  tickers ascending:  unit = p_i (1 + c); q = floor(b / unit), minus one
//                              if q unit > b; q = max(0, min(a_i, q));
//                              h_i += q; b -= q unit
//   v' = b + sum_i p_{t+1,i} h_i;  r = scale (v' - v);  J-accumulator
//   disc += gamma^k r;  k += 1;  done = (k == H) or (t+1 == T_data - 1);
//   on done: ep_ret = disc and auto-reset (b = C0, h = 0, k = 0, t = s);
//   s_{t+1} = [b/C0, h_i p_i/C0, p_i/p0_i, feat[t][c][i], 0-pad]  (bf16).
//
// B200 mapping: one 128-thread block per env tile (32 envs that share an
// episode start row, hence the same market rows).  The tile's holdings and
// actions ([n][32], ticker-major in HBM) arrive as two 2-D TMA boxes, the
// market rows with one round of independent loads; warp 0 (lane = env) then
// runs ONLY the sequential float64 ledger, in exactly the order written
// above (explicit __dmul_rn / __dadd_rn / __ddiv_rn, no FMA contraction), so
// cash, account value, reward and the integer holdings are bit-identical to a
// sequential float64 implementation — a parallel prefix over tickers would
// reassociate the cash sums and could flip a floor() at a near tie.  All four
// warps then write the new holdings (coalesced 128-B rows), build the per-env
// part of s_{t+1} and store the 32 observation rows with 16-B vector stores
// (512 contiguous bytes per warp instruction).  Warp 1 also sums the actor's four log-prob partials
// of each env into traj.logp (fixed order), and the idle warps draw the next step's actor noise.
//
// The tile body (env_step_tile) serves two callers: env_step_kernel (one block per tile, the separate
// launches) and the fused rollout kernel (actor_kernel.cuh, rollout_fused_kernel), where a 128-thread group of
// the actor CTA's epilogue warps runs it every step with the tile's header, ledger state and market rows kept
// in shared memory across steps (EnvPersist layout below), the actions and log-prob partials delivered by the
// actor's head through DSMEM, and the tile-shared part of s_{t+1} written while the ledger runs.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "philox.cuh"
#include "ptx.cuh"

namespace pod {

constexpr int ENV_MAX_STOCKS = 128;
constexpr int ENV_MAX_KPAD = 512;
constexpr int ENV_THREADS = 128;      // 4 warps per env tile
constexpr int ENV_BUY_CHUNKS = 7;     // buy-pass chunks released to the trailing warps (one mbarrier each)
constexpr int ENV_MAX_MARKET = 3 * ENV_MAX_STOCKS + ENV_MAX_KPAD;   // p_t, p_1, p_0, indicators

struct EnvArgs {
    int32_t N;
    int32_t n;
    int32_t f;
    int32_t k_pad;
    int32_t obs_dim;
    int32_t horizon;
    int32_t n_tiles;
    int32_t mode;             // 0 = step, 1 = write obs of the current state, 2 = reset + obs
    int32_t tma_ok;           // hold / aint tiles may be fetched with the 2-D tensor maps
    int32_t gen_noise;        // also draw the actor's N(0,1) noise for step *step_base + noise_t
    int32_t noise_t;
    int32_t tile0;            // first env tile of this launch (env groups)
    uint64_t seed;
    int64_t env_offset;
    const uint64_t* step_base;
    float* znoise;            // [n][N] noise output
    unsigned long long* trace;   // diagnostics: [n_tiles][8] clock64 stamps, or null
    int64_t T_data;
    double C0;
    double cost;
    double scale;
    double gamma;
    const float* close;       // [T_data][n]
    const float* feat;        // [T_data][f][n]
    int32_t* hold;            // [n][N]
    const int16_t* aint;      // [n][N]
    double* cash;             // [N]
    double* asset;            // [N]
    double* disc;             // [N]
    double* ep_ret;           // [N]
    int32_t* tile_start;      // [n_tiles]
    int32_t* tile_k;          // [n_tiles]
    double* tile_gpow;        // [n_tiles]
    float* rew;               // [N] slice of step t
    uint8_t* done;            // [N] slice of step t
    uint16_t* obs_out;        // [N][k_pad] bf16 slice (s_{t+1}, or s_t for mode 1/2), may be null
    int32_t* dbg_hold;        // [N][n] slice or null
    double* dbg_cash;         // [N] slice or null
    double* equity;           // [N] slice of step t: v_{t+1} before any reset, or null
    uint32_t* err;
    int32_t pdl;              // 1: launched as a programmatic dependent of the actor (see the kernel)
    const float* logp_parts;  // [4][N] the actor's log-prob partials of this step, or null
    float* logp_out;          // [N] slice of step t: ((p0 + p1) + p2) + p3 written here
};

struct EnvMaps {
    CUtensorMap hold;   // 2-D int32 [n][N], box {32, n}
    CUtensorMap aint;   // 2-D uint16 [n][N], box {32, n}
};

// shared memory of one block (one tile), TMA destinations 128-B aligned:
//   [hold_s n*32 i32 | aint_s n*32 i16 (pad 128) | unit, p_t, p_1, 1/unit n f64 each (pad 16) |
//    p_t, p_1, p_0 n f32 (pad 16) | tmpl k_pad bf16 | stg 32 x e_pad bf16 | mbar]
__host__ __device__ inline int env_e_pad(int n) { return (1 + n + 7) / 8 * 8; }
struct EnvSmemLayout {
    int aint, unit, p, tmpl, stg, ph, bar, total;
};
__host__ __device__ inline EnvSmemLayout env_smem_layout(int n, int k_pad) {
    EnvSmemLayout L;
    L.aint = n * 128;
    L.unit = L.aint + (n * 64 + 127) / 128 * 128;
    L.p = L.unit + (4 * n * 8 + 15) / 16 * 16;
    L.tmpl = L.p + (3 * n * 4 + 15) / 16 * 16;
    L.stg = L.tmpl + k_pad * 2;
    L.ph = (L.stg + 32 * env_e_pad(n) * 2 + 7) / 8 * 8;
    L.bar = L.ph + 32 * 8;
    L.total = L.bar + 8 + 8 * ENV_BUY_CHUNKS;   // TMA barrier, then one per buy chunk
    return L;
}
__host__ __device__ inline int env_smem_bytes(int n, int k_pad) { return env_smem_layout(n, k_pad).total; }

__device__ __forceinline__ uint16_t f2bf(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// SELL_UNROLL / BUY_UNROLL: unroll depths of the ledger's two ticker loops (16 / 8 for many tickers,
// 8 / 4 for few: the deeper unroll is +1.5 % at n = 100 and -3 % at n = 30)
// the per-step outputs of one env step (slices of the trajectory at step t)
struct EnvStep {
    float* rew;
    uint8_t* done;
    uint16_t* obs_out;
    int32_t* dbg_hold;
    double* dbg_cash;
    double* equity;
    float* logp_out;
    int32_t gen_noise;
    int32_t noise_t;
};

// Fused rollout (EnvPersist): an env tile's state kept in the CTA's shared memory across the T steps (outside the activation
// buffer the per-step tile area lives in): the tile header, its 32 envs' ledger state, and the next step's market
// rows, which TMA bulk copies bring in during the actor phase.  Byte offsets; `mkt` holds three 16-byte aligned
// windows, [p_t | p_{t+1}], [p_0], [feat[t_obs]] ((3 + f) n floats), each starting up to 3 floats before its row
// (bulk copies move whole 16-byte units); the header records where each row starts.
constexpr int ENVP_HDR = 0;       // int64 s, int32 k, pad, double gpow, uint16 row offsets (floats) of p_t, p_0, feat
constexpr int ENVP_LEDGER = 32;   // double cash[32], asset[32], disc[32]
constexpr int ENVP_MKT = 800;
__host__ __device__ inline int env_persist_bytes(int n, int f) {
    return (ENVP_MKT + (3 + f) * n * 4 + 3 * 16 + 127) / 128 * 128;
}
// one row range [src, src + bytes) as a whole-16-byte window at smem dst; returns the window's bytes, and the
// row's offset inside it in floats
__device__ __forceinline__ uint32_t env_mkt_window(uint32_t dst, const float* src, uint32_t bytes, uint32_t bar,
                                                   uint16_t* off) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(src);
    const uintptr_t p0 = p & ~static_cast<uintptr_t>(15);
    const uint32_t w = static_cast<uint32_t>((p + bytes - p0 + 15) & ~static_cast<uintptr_t>(15));
    bulk_g2s(dst, reinterpret_cast<const void*>(p0), w, bar);
    *off = static_cast<uint16_t>((p - p0) >> 2);
    return w;
}
// the market rows of the step with episode start s and step k: bulk copies onto `bar`, which this arms (the copies
// may read up to 12 bytes outside a row, inside the close / feat arrays' 16-byte-aligned allocation units)
__device__ __forceinline__ void env_mkt_issue(const EnvArgs& a, uint8_t* pst, int64_t s, int k, uint32_t bar) {
    const int n = a.n;
    const int64_t t = s + k;
    const bool done = (k + 1 == a.horizon) || (t + 1 == a.T_data - 1);
    const int64_t t_obs = done ? s : t + 1;
    const uint32_t m = smem_u32(pst + ENVP_MKT);
    uint16_t* off = reinterpret_cast<uint16_t*>(pst + ENVP_HDR + 24);
    auto span = [](const float* p, uint32_t bytes) {
        const uintptr_t q = reinterpret_cast<uintptr_t>(p);
        return static_cast<uint32_t>((q + bytes - (q & ~static_cast<uintptr_t>(15)) + 15) & ~static_cast<uintptr_t>(15));
    };
    const float* r0 = a.close + t * n;
    const float* r1 = a.close + s * n;
    const float* r2 = a.feat + t_obs * a.f * n;
    const uint32_t b0 = static_cast<uint32_t>(2 * n * 4), b1 = static_cast<uint32_t>(n * 4);
    const uint32_t b2 = static_cast<uint32_t>(a.f * n * 4);
    const uint32_t w0 = span(r0, b0), w1 = span(r1, b1), w2 = span(r2, b2);
    mbar_arrive_expect_tx(bar, w0 + w1 + w2);
    env_mkt_window(m, r0, b0, bar, off);                  // p_t, p_{t+1}
    env_mkt_window(m + w0, r1, b1, bar, off + 1);         // p_0
    env_mkt_window(m + w0 + w1, r2, b2, bar, off + 2);    // indicators at t_obs
    off[1] = static_cast<uint16_t>(off[1] + (w0 >> 2));
    off[2] = static_cast<uint16_t>(off[2] + ((w0 + w1) >> 2));
}

// One env tile (32 envs) on 128 threads (tid 0..127).  sync_id 0: the tile is a whole block (__syncthreads,
// the block initialises its own mbarriers at `bar`); sync_id > 0: the tile is a 128-thread group of a larger
// block (the fused rollout kernel) synchronised with named barrier sync_id, whose mbarriers at `bar` were
// initialised once and complete once per step (wait parity `par`).  With `pst` (fused, n % 4 == 0) the tile header,
// ledger state and market rows come from the persistent state (the rows on mkt_bar, one completion per step), and
// the tile issues the next step's row copies at its end when `issue_next`.  With `in_bar` (fused) the caller has
// issued the holdings TMA (n x 128 bytes on `bar`), and the actor's heads deliver the actions into aint_s and the
// four log-prob partials of each env into the first 512 bytes of stg ([4][32] float) by st.async on in_bar.
// StepT: EnvStep, or EnvArgs itself (the standalone kernel reads its step slices straight from the parameters)
template <int SELL_UNROLL, int BUY_UNROLL, typename StepT>
__device__ __forceinline__ void env_step_tile(const EnvMaps& maps, const EnvArgs a, const StepT st, const int tile,
                                              const int tid, uint8_t* env_smem, const uint32_t bar_in, const uint32_t par,
                                              const int sync_id, uint8_t* pst = nullptr, const uint32_t mkt_bar = 0,
                                              const bool issue_next = false, const uint32_t in_bar = 0) {
    auto sync = [sync_id] {
        if (sync_id == 0) __syncthreads();
        else named_bar_sync(static_cast<uint32_t>(sync_id), ENV_THREADS);
    };
    const int warp = tid >> 5;
    const int lane = tid & 31;
    unsigned long long* trc = (a.trace && a.mode == 0 && sync_id == 0) ? a.trace + tile * 8 : nullptr;
    if (trc && tid == 0) trc[0] = clock64();
#ifdef POD_EXP_GTIME
    if (sync_id == 0 && tid == 0 && a.mode == 0 && st.noise_t - 1 < 1024) atomicMin(&g_gtime[st.noise_t - 1][2], gtimer());
#endif
    const int n = a.n;
    const int e_pad = env_e_pad(n);
    const EnvSmemLayout SL = env_smem_layout(n, a.k_pad);
    int32_t* hold_s = reinterpret_cast<int32_t*>(env_smem);                                     // [n][32]
    int16_t* aint_s = reinterpret_cast<int16_t*>(env_smem + SL.aint);                           // [n][32]
    double* unit_s = reinterpret_cast<double*>(env_smem + SL.unit);   // [n] p_t (1 + c)
    double* p_t64 = unit_s + n;                                           // [n] p_t as float64
    double* p_164 = unit_s + 2 * n;                                       // [n] p_{t+1} as float64
    double* rcp_s = unit_s + 3 * n;                                       // [n] fl(1 / unit)
    const uint16_t* poff = reinterpret_cast<const uint16_t*>(pst + ENVP_HDR + 24);
    float* p_t = pst ? reinterpret_cast<float*>(pst + ENVP_MKT) + poff[0] : reinterpret_cast<float*>(env_smem + SL.p);
    float* p_1 = p_t + n;
    float* p_0 = pst ? reinterpret_cast<float*>(pst + ENVP_MKT) + poff[1] : p_1 + n;
    uint16_t* tmpl = reinterpret_cast<uint16_t*>(env_smem + SL.tmpl);
    uint16_t* stg = reinterpret_cast<uint16_t*>(env_smem + SL.stg);                           // [32][e_pad]
    double* ph_s = reinterpret_cast<double*>(env_smem + SL.ph);                               // [32]
    // (computed here, not by the caller: an early smem address kept live costs the ledger 8 registers)
    const uint32_t bar = sync_id == 0 ? smem_u32(env_smem + SL.bar) : bar_in;

    const int e = tile * 32 + lane;                 // this lane's env (all four warps)
    const bool active = e < a.N;
    const int64_t N = a.N;
    const bool full_tile = (tile + 1) * 32 <= a.N;
    const bool stepping = a.mode == 0;
    const bool need_hold = a.mode != 2;
    const bool tma = need_hold && full_tile && a.tma_ok;

    // ---- 1. fetch the tile's holdings h_t[n][32] and actions a_t[n][32]: two 2-D TMA boxes
    const uint32_t chunk_bar = bar + 8u;   // [ENV_BUY_CHUNKS] buy chunk c released by warp 0 (32 arrivals)
    if (sync_id == 0 && tid == 0 && stepping) {
        for (int c = 0; c < ENV_BUY_CHUNKS; ++c) mbar_init(chunk_bar + 8u * c, 32);
        if (!tma) fence_mbar_init();
    }
    // Launched as a programmatic dependent of the actor (when a.pdl): everything up to the actions
    // (holdings, ledger state, market rows, tile constants) is loaded while the actor grid is still
    // running; griddepcontrol.wait precedes the first read of the actor's outputs (the actions) and the
    // first write the actor could observe (the next step's noise).
    if (in_bar) {
        mbar_wait(in_bar, par);   // the actions and log-prob partials of this step have landed
        if (warp == 1 && stepping && a.logp_parts && st.logp_out && active) {
            // summed in the actor's own order; read before anything rewrites stg
            const float* pp = reinterpret_cast<const float*>(stg) + lane;
            st.logp_out[e] = ((pp[0] + pp[32]) + pp[64]) + pp[96];
        }
    }
    if (!in_bar && tma && tid == 0) {
        if (sync_id == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
        }
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(n) * (stepping ? 192u : 128u));
        tma_load_2d(smem_u32(hold_s), &maps.hold, tile * 32, 0, bar);
        if (stepping && !a.pdl) tma_load_2d(smem_u32(aint_s), &maps.aint, tile * 32, 0, bar);
    }
    // per-env ledger state (warp 0 owns the ledger)
    double cash0 = 0.0, v0 = 0.0, disc0 = 0.0;
    const double* pled = reinterpret_cast<const double*>(pst + ENVP_LEDGER);
    if (pst) {
        if (warp == 0) {
            cash0 = pled[lane];
            v0 = pled[32 + lane];
            disc0 = pled[64 + lane];
        }
    } else if (warp == 0 && active && a.mode != 2) {
        cash0 = a.cash[e];
        if (stepping) {
            v0 = a.asset[e];
            disc0 = a.disc[e];
        }
    }
    const int64_t s = pst ? *reinterpret_cast<const int64_t*>(pst + ENVP_HDR) : a.tile_start[tile];
    const int k = pst ? *reinterpret_cast<const int32_t*>(pst + ENVP_HDR + 8)
                      : (a.mode == 2 ? 0 : a.tile_k[tile]);
    const double gpow = pst ? *reinterpret_cast<const double*>(pst + ENVP_HDR + 16)
                            : (a.mode == 2 ? 1.0 : a.tile_gpow[tile]);
    const int64_t t = s + k;
    const bool done = stepping && ((k + 1 == a.horizon) || (t + 1 == a.T_data - 1));
    const int64_t t_obs = stepping ? (done ? s : t + 1) : t;   // market row of the next observation
    if (stepping) {
        // the next step reads close[t'+1] and feat[t'+1] (t' = this step's next row) for the first time:
        // pull them into L2 now, so the next launch's dependent market loads do not go to HBM
        const int64_t tn = t_obs + 1;
        const int lc = (n * 4 + 127) / 128, lf = (a.f * n * 4 + 127) / 128;
        if (tn < a.T_data && tid < lc + lf) {
            const char* row = tid < lc ? reinterpret_cast<const char*>(a.close + tn * n) + tid * 128
                                       : reinterpret_cast<const char*>(a.feat + tn * a.f * n) + (tid - lc) * 128;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
        }
    }

    if (need_hold && !tma) {   // ragged tile: cooperative plain loads
        for (int i = warp; i < n; i += 4) {
            hold_s[i * 32 + lane] = active ? a.hold[i * N + e] : 0;
            if (stepping && !a.pdl) aint_s[i * 32 + lane] = active ? a.aint[i * N + e] : 0;
        }
    }
    // ---- 2. market rows: every thread issues all of its loads before using any
    if (pst) {   // already in shared memory (the copies issued during the actor phase)
        mbar_wait(mkt_bar, par);
        const float* feat_s = reinterpret_cast<const float*>(pst + ENVP_MKT) + poff[2];
        for (int j = tid; j < a.f * n; j += ENV_THREADS) tmpl[1 + 2 * n + j] = f2bf(feat_s[j]);
    } else {
        const int total = 3 * n + a.f * n;
        constexpr int PER = (ENV_MAX_MARKET + ENV_THREADS - 1) / ENV_THREADS;
        float vals[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + ENV_THREADS * q;
            float x = 0.0f;
            if (idx < total) {
                const float* src;
                if (idx < n) src = a.close + t * n + idx;
                else if (idx < 2 * n) src = a.close + (stepping ? t + 1 : t) * n + (idx - n);
                else if (idx < 3 * n) src = a.close + s * n + (idx - 2 * n);
                else src = a.feat + t_obs * a.f * n + (idx - 3 * n);
                x = __ldg(src);
            }
            vals[q] = x;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + ENV_THREADS * q;
            if (idx < 3 * n) p_t[idx] = vals[q];
            else if (idx < total) tmpl[1 + 2 * n + (idx - 3 * n)] = f2bf(vals[q]);
        }
    }
    sync();
    // ---- 3. per-tile constants: unit price p_t (1 + c), p/p0 at t_obs, zero pad
    const double opc = __dadd_rn(1.0, a.cost);
    for (int i = tid; i < n; i += ENV_THREADS) {
        unit_s[i] = __dmul_rn(static_cast<double>(p_t[i]), opc);
        rcp_s[i] = __ddiv_rn(1.0, unit_s[i]);
        p_t64[i] = static_cast<double>(p_t[i]);
        p_164[i] = static_cast<double>(p_1[i]);
    }
    for (int c = tid; c < a.k_pad; c += ENV_THREADS) {
        if (c >= 1 + n && c < 1 + 2 * n) {
            const int i = c - 1 - n;
            const float p = t_obs == s ? p_0[i] : (t_obs == t ? p_t[i] : p_1[i]);
            tmpl[c] = f2bf(p / p_0[i]);
        } else if (c >= a.obs_dim || c < 1 + n) {
            tmpl[c] = 0;
        }
    }
    if (a.pdl) {
        pdl_wait();
        if (stepping) {
            if (tma && tid == 0) tma_load_2d(smem_u32(aint_s), &maps.aint, tile * 32, 0, bar);
            if (!tma)
                for (int i = warp; i < n; i += 4) aint_s[i * 32 + lane] = active ? a.aint[i * N + e] : 0;
        }
    }
    if (tma) mbar_wait(bar, par);
    sync();
    if (trc && tid == 0) trc[1] = clock64();
#ifdef POD_EXP_GTIME
    if (sync_id == 3 && tid == 0 && blockIdx.x == 0 && st.noise_t - 1 < 1024) g_ftime[st.noise_t - 1][6] = gtimer();
#endif
    if (!in_bar && warp == 1 && stepping && a.logp_parts && st.logp_out && active) {
        // the actor's four log-prob partials of this env, summed in the actor's own order
        const float* pp = a.logp_parts + e;
        if (sync_id == 0) {
            st.logp_out[e] = ((pp[0] + pp[N]) + pp[2 * N]) + pp[3 * N];
        } else {   // L2 loads: the peer CTA of the fused rollout wrote half of them
            st.logp_out[e] = ((__ldcg(pp) + __ldcg(pp + N)) + __ldcg(pp + 2 * N)) + __ldcg(pp + 3 * N);
        }
    }

    // ---- 4. the float64 ledger, warp 0, lane = env, in exactly the order of
    //         Eqs. 3-4 under R#3/R#4 (sells, then greedy buys, tickers ascending)
    double cash = cash0;
    // buy pass in chunks of CH tickers: after each chunk warp 0 releases mbarrier c,
    // and warps 1-3 (done with the noise) trail it: warp 1 carries the revaluation sum
    // sum_i p_{t+1,i} h_i (tickers ascending, as the oracle), warps 2-3 write the holdings out
    // and their part of s_{t+1}, so only the ledger's own chain is left on warp 0
    const int CH = ((n + ENV_BUY_CHUNKS - 1) / ENV_BUY_CHUNKS + 3) & ~3;   // multiple of the 4-way unroll
    const int nch = (n + CH - 1) / CH;
    const float inv_c0 = static_cast<float>(1.0 / a.C0);
    if (warp == 0) {
        if (a.mode == 2) {
            cash = a.C0;
            if (active) {
                a.cash[e] = a.C0;
                a.asset[e] = a.C0;
                a.disc[e] = 0.0;
                a.ep_ret[e] = 0.0;
            }
        } else if (stepping) {
            const double omc = __dadd_rn(1.0, -a.cost);
            // selling set (Eq. 3 "+ (p^S)^T k^S"), tickers ascending.  Branch-free: a
            // non-sell adds +0.0, which leaves the (never negative-zero) cash unchanged.
            // Only cash is carried: the post-sell holdings are recomputed in the buy pass.
            // unrolled SELL_UNROLL deep: the loads and products of that many tickers are scheduled ahead of
            // their carried adds (n = 100: 8 -> 4.2K cycles per tile for the sells, 16 -> 3.9K)
#pragma unroll SELL_UNROLL
            for (int i = 0; i < n; ++i) {
                const int ai = aint_s[i * 32 + lane];
                const int h = hold_s[i * 32 + lane];
                const int q = ai < 0 ? min(h, -ai) : 0;
                cash = __dadd_rn(cash, __dmul_rn(__dmul_rn(p_t64[i], static_cast<double>(q)), omc));
            }
            if (trc && lane == 0) trc[2] = clock64();
#ifdef POD_EXP_GTIME
            if (sync_id == 3 && lane == 0 && blockIdx.x == 0 && st.noise_t - 1 < 1024) g_ftime[st.noise_t - 1][11] = gtimer();
#endif
            // buying set (Eq. 3 "- (p^B)^T k^B"), tickers ascending.
            // The oracle computes qmax = floor(fl(b / unit)) (minus one if fl(qmax unit) > b),
            // q = max(0, min(a, qmax)), b -= fl(q unit).  Here, with y = fl(b fl(1/unit)) and
            // m = floor(y) (y = b/unit (1 +- 2^-51), fl(b/unit) = b/unit (1 +- 2^-53)):
            //   q = min(m, a+), cost = fl(q unit)         (5 dependent float64 ops)
            // equals the oracle whenever
            //   (i)  m > a+: b/unit >= (a+1)(1 - 2^-51) > a, so the oracle's qmax >= a too; or
            //   (ii) fr = y - m (exact) lies in [2^-34, 1 - 2^-34]: y < 2^15 here (else (i)),
            //        so |y - fl(b/unit)| <= y 2^-51 < 2^-36 while y is at least 2^-34 from both
            //        neighbouring integers: fl(b/unit) has the same floor m, and
            //        m unit < b - 2^-35 unit: the post-check cannot fire.
            // fr and m are non-negative doubles, compared through their bit patterns (integer
            // compares).  The test is kept off the carried chain: a ticker that fails it (b/unit
            // within ~2^-34 of an integer: rare) only sets a flag, and if any lane of the warp
            // raised it the chunk is redone with the oracle's own expressions before its release.
            constexpr long long FR_LO = 0x3DD0000000000000ll;   // 2^-34
            constexpr long long FR_HI = 0x3FEFFFFFFFF80000ll;   // 1 - 2^-34
            for (int c = 0; c < nch; ++c) {
                const int i0 = c * CH;
                const int i1 = i0 + CH < n ? i0 + CH : n;
                const double cash_c0 = cash;
                bool unsure = false;
                // one-deep prefetch: ticker i+1's shared-memory operands are loaded before ticker i's
                // holdings store (which would otherwise keep the compiler from hoisting them)
                int ai_n = aint_s[i0 * 32 + lane], h_n = hold_s[i0 * 32 + lane];
                double un_n = unit_s[i0], rc_n = rcp_s[i0];
                // unrolled BUY_UNROLL deep (n = 100: 4 -> 13.4K cycles per tile for the buys, 8 -> 12.9K;
                // 72 registers, still 7 tiles per SM, the shared-memory limit)
#pragma unroll BUY_UNROLL
                for (int i = i0; i < i1; ++i) {
                    const int ai = ai_n;
                    int h = h_n;
                    const double unit = un_n, rcp = rc_n;
                    if (i + 1 < i1) {
                        ai_n = aint_s[(i + 1) * 32 + lane];
                        h_n = hold_s[(i + 1) * 32 + lane];
                        un_n = unit_s[i + 1];
                        rc_n = rcp_s[i + 1];
                    }
                    if (ai < 0) h -= min(h, -ai);                      // post-sell holdings
                    // q = min(floor(y), a+) in the biased domain: fl(y + 2^52, rounded down) = 2^52 + floor(y)
                    // exactly (0 <= y < 2^52; larger y, never reached, still compares above), and 2^52 + a+ is
                    // built from the integer; both are positive doubles, so their bit patterns order as their
                    // values and an integer min replaces FRND / I2F / DSETP / F2I on the float64 pipe.  The
                    // min's low word is q; one exact DADD takes q back to a double for the cost
                    const long long ab = 0x4330000000000000ll | static_cast<long long>(ai > 0 ? ai : 0);
                    const double y = __dmul_rn(cash, rcp);
                    const long long tb = __double_as_longlong(__dadd_rd(y, 4503599627370496.0));
                    const bool cut = tb > ab;                           // floor(y) > a+: q = a+
                    const long long mb = cut ? ab : tb;
                    const double qd = __dadd_rn(__longlong_as_double(mb), -4503599627370496.0);
                    const double cost = __dmul_rn(qd, unit);
                    const long long frb = __double_as_longlong(__dadd_rn(y, -qd));   // y - floor(y) unless cut
                    unsure |= !(ai <= 0 || cut || (frb >= FR_LO && frb <= FR_HI));
                    h += static_cast<int>(static_cast<unsigned>(mb));
                    cash = __dadd_rn(cash, -cost);
                    hold_s[i * 32 + lane] = h;
                }
                if (__any_sync(0xffffffffu, unsure)) {
                    // redo the chunk: replay the pass above to recover each ticker's post-sell
                    // holdings, and run the oracle's expressions alongside
                    double bf = cash_c0;
                    cash = cash_c0;
                    for (int i = i0; i < i1; ++i) {
                        const int ai = aint_s[i * 32 + lane];
                        const double unit = unit_s[i];
                        const double ad = static_cast<double>(ai > 0 ? ai : 0);
                        const double yf = __dmul_rn(bf, rcp_s[i]);
                        const double flf = floor(yf);
                        const double qf = flf < ad ? flf : ad;
                        bf = __dadd_rn(bf, -__dmul_rn(qf, unit));
                        const int h_sold = hold_s[i * 32 + lane] - static_cast<int>(qf);
                        double qmax = floor(__ddiv_rn(cash, unit));
                        if (__dmul_rn(qmax, unit) > cash) qmax = __dadd_rn(qmax, -1.0);
                        double qd = ad < qmax ? ad : qmax;
                        qd = qd < 0.0 ? 0.0 : qd;
                        cash = __dadd_rn(cash, -__dmul_rn(qd, unit));
                        hold_s[i * 32 + lane] = h_sold + static_cast<int>(qd);
                    }
                }
                mbar_arrive(chunk_bar + 8u * c);   // release: this lane's holdings of the chunk
            }
            if (trc && lane == 0) trc[3] = clock64();
#ifdef POD_EXP_GTIME
            if (sync_id == 3 && lane == 0 && blockIdx.x == 0 && st.noise_t - 1 < 1024) g_ftime[st.noise_t - 1][10] = gtimer();
#endif
        }
    } else {
        if (st.gen_noise) {
            // the actor's Gaussian noise for the next actor launch (R#14: Philox4x32-10 keyed on
            // (global env, global step, ticker quad)), drawn while warp 0 runs the ledger
            const uint64_t step = *a.step_base + static_cast<uint64_t>(st.noise_t);
            const int nq = (n + 3) / 4;
            for (int idx = tid - 32; idx < 32 * nq; idx += ENV_THREADS - 32) {
                const int el = idx & 31;
                const int qd = idx >> 5;
                const int ee = tile * 32 + el;
                if (ee < a.N) {
                    const float4 z = normals4(a.seed, static_cast<uint32_t>(a.env_offset + ee), step, static_cast<uint32_t>(qd));
                    const float zz[4] = {z.x, z.y, z.z, z.w};
                    float* zp = a.znoise + static_cast<int64_t>(4 * qd) * N + ee;
                    if (4 * qd + 4 <= n) {   // full quad: four unconditional row stores
                        zp[0] = zz[0];
                        zp[N] = zz[1];
                        zp[2 * N] = zz[2];
                        zp[3 * N] = zz[3];
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (4 * qd + j < n) zp[static_cast<int64_t>(j) * N] = zz[j];
                    }
                }
            }
        }
        if (stepping) {
            uint16_t* my = stg + lane * e_pad;
            if (warp == 1) {
                for (int c = 1 + n; c < e_pad; ++c) my[c] = tmpl[c];
            }
            if (sync_id != 0 && st.obs_out) {
                // fused: the tile-shared part of the 32 rows of s_{t+1} (16-byte chunks from e_pad on: p/p0,
                // indicators, pad — the same for every env of the tile) leaves now, while the ledger runs; the
                // tail writes only the per-env chunks
                const int c0 = e_pad / 8, nc = a.k_pad / 8 - c0;
                const int rows = min(32, a.N - tile * 32);
                uint4* dst0 = reinterpret_cast<uint4*>(st.obs_out + static_cast<int64_t>(tile) * 32 * a.k_pad);
                for (int idx = tid - 32; idx < rows * nc; idx += ENV_THREADS - 32) {
                    const int row = idx / nc, c = c0 + idx % nc;
                    dst0[static_cast<int64_t>(row) * (a.k_pad / 8) + c] = *reinterpret_cast<const uint4*>(tmpl + c * 8);
                }
            }
            double ph = 0.0;
            for (int c = 0; c < nch; ++c) {
                mbar_wait_parked(chunk_bar + 8u * c, par);
                const int i0 = c * CH;
                const int i1 = i0 + CH < n ? i0 + CH : n;
                if (warp == 1) {
                    for (int i = i0; i < i1; ++i)
                        ph = __dadd_rn(ph, __dmul_rn(p_164[i], static_cast<double>(hold_s[i * 32 + lane])));
                } else {
                    // holdings out (one coalesced row per ticker; the row pointer steps by 2 N) and the
                    // per-env holdings entries of s_{t+1}
                    const int ib = i0 + (warp - 2);
                    int32_t* hrow = a.hold + static_cast<int64_t>(ib) * N + e;
                    const int64_t N2 = 2 * N;
                    const int hkeep = done ? 0 : 1;
                    for (int i = ib; i < i1; i += 2, hrow += N2) {
                        const int h = hold_s[i * 32 + lane];
                        if (active) *hrow = h * hkeep;
                        my[1 + i] = f2bf(static_cast<float>(h * hkeep) * p_1[i] * inv_c0);
                    }
                    if (st.dbg_hold && active)
                        for (int i = ib; i < i1; i += 2) st.dbg_hold[static_cast<int64_t>(e) * n + i] = hold_s[i * 32 + lane];
                }
            }
            if (warp == 1) ph_s[lane] = ph;
        }
    }
    if (tid == 0 && stepping) {
        a.tile_k[tile] = done ? 0 : k + 1;
        a.tile_gpow[tile] = done ? 1.0 : __dmul_rn(gpow, a.gamma);
    }
    if (tid == 0 && a.mode == 2) {
        a.tile_k[tile] = 0;
        a.tile_gpow[tile] = 1.0;
    }
    sync();
    if (trc && tid == 0) trc[4] = clock64();
#ifdef POD_EXP_GTIME
    if (sync_id == 3 && tid == 0 && blockIdx.x == 0 && st.noise_t - 1 < 1024) g_ftime[st.noise_t - 1][7] = gtimer();
#endif
    if (stepping) {
        // revalue at p_{t+1} (Eq. 2 reward), episode bookkeeping, and the cash entry of s_{t+1}
        if (warp == 0) {
            const double v1 = __dadd_rn(cash, ph_s[lane]);
            const double r = __dmul_rn(a.scale, __dadd_rn(v1, -v0));
            double disc = __dadd_rn(disc0, __dmul_rn(gpow, r));
            double v = v1;
            if (active) {
                st.rew[e] = static_cast<float>(r);
                st.done[e] = done ? 1 : 0;
                if (st.dbg_cash) st.dbg_cash[e] = cash;
                if (st.equity) st.equity[e] = v1;
                if (!isfinite(v1)) atomicOr(a.err, 2u);
                if (done) a.ep_ret[e] = disc;
            }
            if (done) {
                cash = a.C0;
                v = a.C0;
                disc = 0.0;
            }
            if (active) {
                a.cash[e] = cash;
                a.asset[e] = v;
                a.disc[e] = disc;
            }
            if (pst) {
                double* pl = reinterpret_cast<double*>(pst + ENVP_LEDGER);
                pl[lane] = cash;
                pl[32 + lane] = v;
                pl[64 + lane] = disc;
            }
            stg[lane * e_pad] = f2bf(static_cast<float>(cash / a.C0));
        }
    } else {
        // ---- 5. (reset / observe) holdings out and the per-env part of s_t, 4 warps
        const float* p_obs = p_t;
        uint16_t* my = stg + lane * e_pad;
        if (warp == 0) {
            my[0] = f2bf(static_cast<float>(cash / a.C0));
            for (int c = 1 + n; c < e_pad; ++c) my[c] = tmpl[c];
        }
#pragma unroll 5
        for (int i = warp; i < n; i += 4) {
            const int h = a.mode == 2 ? 0 : hold_s[i * 32 + lane];
            if (active && a.mode == 2) a.hold[i * N + e] = 0;
            my[1 + i] = a.mode == 2 ? 0 : f2bf(static_cast<float>(h) * p_obs[i] * inv_c0);
        }
    }
    sync();
    if (trc && tid == 0) trc[5] = clock64();
#ifdef POD_EXP_GTIME
    if (sync_id == 3 && tid == 0 && blockIdx.x == 0 && st.noise_t - 1 < 1024) g_ftime[st.noise_t - 1][8] = gtimer();
#endif
    // ---- 6. write s_{t+1}: env rows spread over the 4 warps, 16-B chunks (512 B per instruction)
    if (st.obs_out) {
        const int chunks = a.k_pad / 8;
        const int rows = min(32, a.N - tile * 32);
        if (sync_id != 0 && stepping) {
            // fused: only the per-env chunks are left (the rest left while the ledger ran), one 16-byte chunk
            // per thread and pass
            const int cpr = e_pad / 8;
            uint4* dst0 = reinterpret_cast<uint4*>(st.obs_out + static_cast<int64_t>(tile) * 32 * a.k_pad);
            for (int idx = tid; idx < rows * cpr; idx += ENV_THREADS) {
                const int row = idx / cpr, c = idx - row * cpr;
                dst0[static_cast<int64_t>(row) * chunks + c] = *reinterpret_cast<const uint4*>(stg + row * e_pad + c * 8);
            }
        } else {
            // (no unroll pragma: measured faster at C5 than the former 4-deep unroll of this loop)
            for (int row = warp; row < rows; row += 4) {
                uint4* dst = reinterpret_cast<uint4*>(st.obs_out + (static_cast<int64_t>(tile) * 32 + row) * a.k_pad);
                for (int c = lane; c < chunks; c += 32) {
                    const uint4 val = c * 8 < e_pad ? *reinterpret_cast<const uint4*>(stg + row * e_pad + c * 8)
                                                    : *reinterpret_cast<const uint4*>(tmpl + c * 8);
                    dst[c] = val;
                }
            }
        }
    }
    sync();
    if (trc && tid == 0) trc[6] = clock64();
#ifdef POD_EXP_GTIME
    if (sync_id == 3 && tid == 0 && blockIdx.x == 0 && st.noise_t - 1 < 1024) g_ftime[st.noise_t - 1][9] = gtimer();
#endif
    if (pst && stepping && tid == 0) {
        // the next step's header, and (issue_next) its market rows, which land during the next actor phase; every
        // thread of the tile is done reading the rows (the sync above)
        const int k1 = done ? 0 : k + 1;
        *reinterpret_cast<int32_t*>(pst + ENVP_HDR + 8) = k1;
        *reinterpret_cast<double*>(pst + ENVP_HDR + 16) = done ? 1.0 : __dmul_rn(gpow, a.gamma);
        if (issue_next) {
            fence_proxy_async_smem();
            env_mkt_issue(a, pst, s, k1, mkt_bar);
        }
    }
#ifdef POD_EXP_GTIME
    if (sync_id == 0 && tid == 0 && a.mode == 0 && st.noise_t - 1 < 1024) atomicMax(&g_gtime[st.noise_t - 1][3], gtimer());
#endif
}

template <int SELL_UNROLL, int BUY_UNROLL>
__global__ void __launch_bounds__(ENV_THREADS) env_step_kernel(const __grid_constant__ EnvMaps maps,
                                                                  const EnvArgs a) {
    extern __shared__ __align__(128) uint8_t env_smem[];
    env_step_tile<SELL_UNROLL, BUY_UNROLL>(maps, a, a, a.tile0 + static_cast<int>(blockIdx.x),
                                           static_cast<int>(threadIdx.x), env_smem, 0u, 0u, 0);
}

// injected actions: a[i][e] = sgn(u) floor(|u| h_max + 1/2)  (R#6)
__global__ void inject_map_kernel(const float* __restrict__ u, int N, int n, int h_max, int16_t* __restrict__ aint,
                                  int16_t* __restrict__ dbg_aint, int e0, int e1) {
    const int64_t idx = static_cast<int64_t>(e0) * n + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(e1) * n) return;
    const int e = static_cast<int>(idx / n);
    const int i = static_cast<int>(idx % n);
    const float x = u[idx];
    const double m = floor(static_cast<double>(fabsf(x)) * static_cast<double>(h_max) + 0.5);
    const int ai = x < 0.0f ? -static_cast<int>(m) : static_cast<int>(m);
    aint[static_cast<int64_t>(i) * N + e] = static_cast<int16_t>(ai);
    if (dbg_aint) dbg_aint[idx] = static_cast<int16_t>(ai);
}

// market validation at env creation: bit 0 = a close price that is not finite and > 0 (the unit
// price p (1 + c) and its reciprocal must be positive and finite), bit 1 = a non-finite indicator
__global__ void market_check_kernel(const float* __restrict__ close, int64_t n_close, const float* __restrict__ feat,
                                    int64_t n_feat, uint32_t* __restrict__ flags) {
    uint32_t f = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_close; i += stride) {
        const float p = close[i];
        if (!(p > 0.0f && p < INFINITY)) f |= 1u;
    }
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_feat; i += stride)
        if (!isfinite(feat[i])) f |= 2u;
    f = __reduce_or_sync(0xffffffffu, f);
    if (f && (threadIdx.x & 31) == 0) atomicOr(flags, f);
}

// J_a = (sum over agent a's envs of ep_ret) / per_agent, one 1024-thread block per agent
__global__ void __launch_bounds__(1024) fitness_kernel(const double* __restrict__ ep_ret, int per_agent,
                                                       double* __restrict__ out) {
    __shared__ double red[32];
    const int agent = blockIdx.x;
    const double* src = ep_ret + static_cast<int64_t>(agent) * per_agent;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int i = threadIdx.x;
    for (; i + 3 * 1024 < per_agent; i += 4 * 1024) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += src[i + q * 1024];
    }
    for (; i < per_agent; i += 1024) acc[0] += src[i];
    double v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) out[agent] = v / static_cast<double>(per_agent);
    }
}

// hold [n][N] -> out [N][n]
__global__ void hold_transpose_kernel(const int32_t* __restrict__ hold, int N, int n, int32_t* __restrict__ out) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(N) * n) return;
    const int e = static_cast<int>(idx / n);
    const int i = static_cast<int>(idx % n);
    out[idx] = hold[static_cast<int64_t>(i) * N + e];
}

__global__ void bump_step_kernel(uint64_t* step, uint64_t by) { *step += by; }

}  // namespace pod
