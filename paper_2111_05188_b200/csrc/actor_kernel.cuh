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
// B200 design.  A CLUSTER OF 2 CTAs owns one 128-env M-tile and splits every
// layer's output columns between its two CTAs (CTA r computes columns
// [r N/2, (r+1) N/2)), so twice as many SMs work on the chain and each SM
// streams only half of every weight matrix from L2.  Per CTA:
//   * warp 0 (one lane): TMA producer — the obs tile [128 x k_pad] bf16 into the
//     activation buffer (128B-swizzled K-major atoms), then this CTA's half of
//     every weight matrix W_l[BN x 64] through a STAGES-deep ring;
//   * warp 1 (one lane): tcgen05.mma issuer (M=128, N=BN, K=16 steps), A =
//     activations in smem, B = weight ring, D = fp32 accumulator in TMEM;
//     each layer's completion is committed to the accumulator barrier of BOTH
//     CTAs (multicast commit), so each side knows when the pair is done reading
//     the current activations;
//   * warps 2..9: epilogue, 2 warps per 32-lane TMEM quadrant, each half of
//     the columns — tcgen05.ld, bias + activation (biases staged in smem), bf16
//     pack, swizzled st.shared into the local activation buffer, then ONE
//     bulk copy (TMA engine, DSMEM) of this CTA's new activation atoms into the
//     peer's buffer, completing on the peer's activation-ready barrier.  The
//     activations never leave the cluster.
//   * the next layer's MMAs start on the CTA's own half of K while the peer's
//     half is still in flight (per-rank K order: own half first);
//   * head: each CTA samples its half of the tickers with noise z that the
//     previous env-step launch generated in its otherwise idle warps; the per-row
//     log-prob partials go to a [4][N] scratch that the next env step sums in a fixed order.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "env_kernel.cuh"
#include "philox.cuh"
#include "ptx.cuh"

namespace pod {

constexpr int ACT_THREADS = 320;       // 10 warps
#ifndef POD_ACT_BK
#define POD_ACT_BK 32
#endif
// weight ring: ACT_STAGES stages of [ACT_BN rows x ACT_BK K] bf16 (80 KB either way)
constexpr int ACT_STAGES = POD_ACT_BK == 16 ? 10 : 5;
constexpr int ACT_BN = POD_ACT_BK == 64 ? 128 : 256;   // weight rows per ring stage (max): one N = ACT_BN MMA
constexpr int ACT_BK = POD_ACT_BK;     // K per ring stage (32: 64-byte swizzled rows, 16: 32-byte)
constexpr int ACT_KPA = 64 / ACT_BK;   // K blocks per 64-column activation atom
constexpr int ACT_BAR_BYTES = 640;     // mbarrier region
constexpr int ACT_MAX_LAYERS = 5;      // n_hidden <= 4
constexpr int ACT_BIAS_FLOATS = 1792;  // per-CTA staged biases + log-std + sigma
constexpr int ACT_MAX_HQ = 32;         // head tickers per epilogue thread (n_out_pad <= 128)
constexpr int ACT_MAX_NA = 4;          // activation atoms per CTA half (hidden <= 512)

struct ActorArgs {
    int32_t N;               // envs
    int32_t per_agent;       // envs per agent
    int32_t tiles_per_agent; // ceil(per_agent / 128)
    int32_t n;               // stocks
    int32_t n_out_pad;       // head rows (n rounded to 32)
    int32_t k_pad;           // obs row width
    int32_t hidden;
    int32_t n_layers;        // n_hidden + 1
    int32_t act;             // 0 relu, 1 tanh
    int32_t h_max;
    int32_t deterministic;
    int32_t t;               // step within the rollout
    int32_t obs_row0;        // row of obs[t][0] in the obs tensor map = t * N
    int32_t mtile0;          // first 128-env M-tile of this launch (env groups)
    int32_t mtiles;          // M-tiles of this launch; cluster c processes mtile0 + c, + c + nclusters, ...
    int32_t mc;              // 0, or G = 2 / 4: clusters of 2G CTAs (G M-tiles) share weight tiles by TMA multicast
    int32_t value_only;      // 1: only the critic V (head row n) is written (bootstrap pass over obs[T])
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
    const float* znoise; // [n][N] N(0,1) noise for this step (written by the previous env-step launch)
    float* val_out;      // [N] critic V(s_t) = head row n (R#22), or null
    uint32_t* err;
    unsigned long long* trace;   // diagnostics: [grid][32] clock64 stamps, or null
    float* logp_parts;           // [4][N] log-prob partials (rank, half) for the env step to combine (required)
    uint32_t kpb_pack;           // K blocks per ring stage of layer l in bits [5l, 5l+5) (0/1: one 3-D box)
    // the weights re-tiled in ring-stage order (actor_retile_kernel): each stage one contiguous, pre-swizzled
    // block fetched with a 1-D bulk copy; null: the tensor maps
    const char* wt;
    uint64_t wt_agent_bytes;
    uint64_t wt_layer_off[ACT_MAX_LAYERS];
};


struct ActorMaps {
    CUtensorMap obs;                     // 2-D bf16 [rows][k_pad], box {64, 128}
    // 3-D bf16 [agents][out][in], box {32, BN_l, 1}; a narrow layer (kpb > 1): 4-D view
    // [agents][in / 32][out][32], box {32, BN_l, kpb, 1} — kpb K blocks per ring stage, one TMA
    CUtensorMap w[ACT_MAX_LAYERS];
};

// column split of layer l: this CTA's half (rows of W_l) and the ring tile height
__host__ __device__ inline int actor_layer_out(int l, int n_layers, int hidden, int n_out_pad) {
    return l == n_layers - 1 ? n_out_pad : hidden;
}
__host__ __device__ inline int actor_bn(int half) { return half < ACT_BN ? half : ACT_BN; }
// K blocks (32 wide) per ring stage of a narrow layer (bn < 256 weight rows: the C3 head, every C2 layer):
// kpb blocks per 16 KB stage in one 4-D TMA box keep as many bytes in flight as a wide layer's stage (the
// weight stream is latency-bound: ~1.5K cycles per TMA round trip under load, five stages; 4 KB stages
// ran the C3 head at ~2.2K cycles per stage).  The largest divisor of KB (of KB / 2 under the
// own-half-first rotation of layers l > 0) with kpb bn <= 256; at most 31 (5-bit field).
inline int actor_kpb(int KB, int bn, bool rotated) {
    const int kb = rotated ? KB / 2 : KB;
    int cap = ACT_BN / bn;
    if (cap > kb) cap = kb;
    if (cap > 31) cap = 31;
    if (cap < 1) cap = 1;
    while (kb % cap) --cap;
    return cap;
}
constexpr uint32_t ACT_STAGE_BYTES = ACT_BN * ACT_BK * 2;   // 16 KB

// Re-tiled weights: per agent, per layer, per CTA half r, per column chunk c, per ring stage s (natural K order),
// the stage's [bn rows x kp K blocks x 32 K] bf16 image exactly as the SWIZZLE_64B tensor-map load lands it in
// shared memory (16-byte chunk q of row p of a [bn x 64 B] sub-tile at p*64 + ((q ^ ((p >> 1) & 3)) << 4)).
struct RetileArgs {
    const char* params;
    uint64_t param_bytes;
    int32_t n_layers;
    uint64_t w_off[ACT_MAX_LAYERS];
    int32_t rows[ACT_MAX_LAYERS], cols[ACT_MAX_LAYERS], kp[ACT_MAX_LAYERS];
    uint64_t layer_off[ACT_MAX_LAYERS];
    uint64_t agent_bytes;
    char* wt;
};
__global__ void __launch_bounds__(256) actor_retile_kernel(const RetileArgs ra) {
    // one thread per 16-byte chunk of one layer (blockIdx.y = layer, blockIdx.z = agent)
    const int l = blockIdx.y, ag = blockIdx.z;
    if (l >= ra.n_layers) return;
    const int R = ra.rows[l], K = ra.cols[l], kp = ra.kp[l] > 1 ? ra.kp[l] : 1;
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c8n = K / 8;
    if (idx >= static_cast<int64_t>(R) * c8n) return;
    const int o = static_cast<int>(idx / c8n), c8 = static_cast<int>(idx % c8n);
    const int half = R / 2, bn = actor_bn(half);
    const int r = o / half, oh = o % half, c = oh / bn, p = oh % bn;
    const int kb = c8 / (ACT_BK / 8), q = c8 % (ACT_BK / 8);
    const int s = kb / kp, sub = kb % kp;
    const uint64_t stage_bytes = static_cast<uint64_t>(bn) * kp * ACT_BK * 2;
    const uint64_t dst = ra.agent_bytes * ag + ra.layer_off[l] + static_cast<uint64_t>(r) * half * K * 2 +
                         static_cast<uint64_t>(c) * bn * K * 2 + static_cast<uint64_t>(s) * stage_bytes +
                         static_cast<uint64_t>(sub) * bn * ACT_BK * 2 + static_cast<uint64_t>(p) * ACT_BK * 2 +
                         (static_cast<uint64_t>(q ^ ((p >> 1) & 3)) << 4);
    const uint4 v = *reinterpret_cast<const uint4*>(ra.params + ra.param_bytes * ag + ra.w_off[l] +
                                                    (static_cast<uint64_t>(o) * K + static_cast<uint64_t>(c8) * 8) * 2);
    *reinterpret_cast<uint4*>(ra.wt + dst) = v;
}

inline size_t actor_smem_bytes(int k_pad, int hidden) {
    const int ka = (k_pad > hidden ? k_pad : hidden) / 64;
    return 1024 + static_cast<size_t>(ka) * 16384 + static_cast<size_t>(ACT_STAGES) * ACT_STAGE_BYTES +
           ACT_BIAS_FLOATS * 4 + ACT_BAR_BYTES;   // + barriers
}

// The fused rollout (rollout_fused_kernel): one cluster per 128-env M-tile runs the actor AND the env step
// of its 128 envs for all T steps.  The env part of step t (4 env tiles of 32 envs: two per CTA, one per
// 4-warp half of the epilogue warps) runs in the activation buffer, which is idle between the head's MMAs
// and the next observation.
struct FusedEnvArgs {
    EnvArgs env;        // the env-step arguments with the step-0 slices (rew, done, obs_out = obs[1], ...)
    int32_t T;          // steps; iteration T (when val_out is set) is the critic bootstrap pass over obs[T]
    int32_t sampling;   // the env step of step t draws the actor noise of step t+1 (t + 1 < T)
    int32_t env_stride; // bytes between the two env tiles' shared-memory areas inside the activation buffer
    int32_t k_pad;
    int32_t persist;    // bytes of each env tile's persistent state (env_persist_bytes; 0: none, n % 4 != 0) after
                        // the barrier region (the launch adds 2 x persist to the actor's shared memory)
};
struct FusedMaps {
    ActorMaps am;
    EnvMaps em;
};
// per TMEM quadrant: the head's staged actions [64 tickers][32 envs] int16 and log-prob partials [2][32] float
constexpr int FUSED_QUAD_STAGE = 2 * ACT_MAX_HQ * 64 + 256;
// Fused rollout: the env-tile thread index of CTA warp w (2..9) — tile 0 on warps 2-5, tile 1 on warps 6-9 — with
// the roles placed on sub-partitions (warp w runs on sub-partition w % 4): the two ledger warps (env warp 0) on
// sub-partitions 2 and 3 (warps 2, 7), the two revaluation warps (env warp 1, float64 too) on 1 and 0 (warps 5, 8),
// away from each other and from the TMA / MMA threads' sub-partitions where possible
__device__ __forceinline__ int env_role_tid(int w, int lane) {
    // env warp of CTA warps 2..9 = {0, 2, 3, 1, 2, 0, 1, 3}, two bits each (a table would live in local memory)
    return static_cast<int>((0xD278u >> (2 * (w - 2))) & 3u) * 32 + lane;
}
// shared memory of the two env tiles of a CTA, and the head's four quadrant stages after them, fit in the
// activation buffer
inline bool fused_env_fits(int n, int k_pad, int hidden) {
    const int ka = (k_pad > hidden ? k_pad : hidden) / 64;
    const int es = (env_smem_bytes(n, k_pad) + 127) / 128 * 128;
    return 2 * es + 4 * FUSED_QUAD_STAGE <= ka * 16384;
}

// tanh(x) = 1 - 2 / (e^{2x} + 1) on the SFU (ex2.approx, approximate reciprocal): absolute error
// <~ 4e-7 over the whole range (saturates to +-1 exactly), i.e. < 1e-4 of one share of h_max <= 100
// in the action map floor(|u| h_max + 1/2), the bound the sampled-rollout parity test allows.
__device__ __forceinline__ float tanh_sfu(float x) {
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));   // 2 log2(e)
    return 1.0f - __fdividef(2.0f, e + 1.0f);
}
// 32 accumulator columns + bias -> activation -> 16 packed bf16 pairs.  The activation is CTA-uniform:
// one branch around two straight-line bodies (a per-element select issued both the ReLU and the SFU
// tanh sequence, with a branch per element, for every element: 2.5x the epilogue's cost)
__device__ __forceinline__ void epi_pack(const uint32_t (&v)[32], const float4* b4, int act, uint32_t (&pk)[16]) {
    if (act == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 b = b4[q];
            pk[2 * q] = pack_bf16x2(fmaxf(__uint_as_float(v[4 * q]) + b.x, 0.0f),
                                    fmaxf(__uint_as_float(v[4 * q + 1]) + b.y, 0.0f));
            pk[2 * q + 1] = pack_bf16x2(fmaxf(__uint_as_float(v[4 * q + 2]) + b.z, 0.0f),
                                        fmaxf(__uint_as_float(v[4 * q + 3]) + b.w, 0.0f));
        }
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 b = b4[q];
            pk[2 * q] = pack_bf16x2(tanh_sfu(__uint_as_float(v[4 * q]) + b.x), tanh_sfu(__uint_as_float(v[4 * q + 1]) + b.y));
            pk[2 * q + 1] =
                pack_bf16x2(tanh_sfu(__uint_as_float(v[4 * q + 2]) + b.z), tanh_sfu(__uint_as_float(v[4 * q + 3]) + b.w));
        }
    }
}

// FUSED: the rollout kernel (one M-tile per cluster, iteration it = step it, see FusedEnvArgs); else the
// actor forward of one step over M-tiles mtile0 + c, + c + nclusters, ...
template <bool FUSED, int SELL_UNROLL, int BUY_UNROLL>
__device__ __forceinline__ void actor_body(const ActorMaps& maps, const ActorArgs& a, const EnvMaps* emaps,
                                           const FusedEnvArgs* fe) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t cr = cluster_ctarank();              // rank in the cluster (2 or 4 CTAs)
    const uint32_t rank = cr & 1u;                      // column half of this CTA
    const uint32_t peer = cr ^ 1u;                      // same M-tile, other column half
    const uint32_t partner = cr ^ 2u;                   // other M-tile, same column half (a.mc)
    const uint16_t pair_mask = static_cast<uint16_t>((1u << cr) | (1u << peer));
    uint16_t share_mask = static_cast<uint16_t>((1u << cr) | (1u << partner));
    if (a.mc > 2) {   // every CTA of this column half in the cluster
        share_mask = 0;
        for (int gq = 0; gq < a.mc; ++gq) share_mask |= static_cast<uint16_t>(1u << (2 * gq + rank));
    }
    const int ka = (a.k_pad > a.hidden ? a.k_pad : a.hidden) / 64;   // activation atoms
    const uint32_t act_s = base_u32;                                  // ka * 16 KB
    const uint32_t ring_s = act_s + ka * 16384u;
    const uint32_t stage_bytes = ACT_STAGE_BYTES;
    const uint32_t bias_off = ka * 16384u + ACT_STAGES * stage_bytes;
    float* bias_s = reinterpret_cast<float*>(base + bias_off);                 // [ACT_BIAS_FLOATS]
    const uint32_t bar_s = base_u32 + bias_off + ACT_BIAS_FLOATS * 4;
    const uint32_t full_b = bar_s;                                   // [STAGES]
    const uint32_t empty_b = bar_s + 8u * ACT_STAGES;                // [STAGES]
    const uint32_t obs_b = bar_s + 16u * ACT_STAGES;
    const uint32_t accum_b = obs_b + 8u;
    const uint32_t ownrdy_b = obs_b + 16u;     // [4] atom j of this CTA's half of h_{l+1} written (256 arrivals)
    const uint32_t peerrdy_b = obs_b + 48u;    // [4] atom j of the peer's half landed (expect_tx)
    const uint32_t actfree_b = obs_b + 80u;    // this CTA's MMAs of a tile are done reading act_s (commit)
    const uint32_t tslot_s = obs_b + 112u;
    const uint32_t accl_b = obs_b + 120u;      // this CTA's MMAs of a layer are complete (local commit)
    // FUSED: both CTAs' env steps of step t are done (s_{t+1}, holdings and noise written; 2 arrivals), and the
    // env tiles' own mbarriers
    const uint32_t envdone_b = obs_b + 136u;
    static_assert(1 + ENV_BUY_CHUNKS <= 8, "the env tiles' mbarriers take 8 slots per tile below");
    const uint32_t envbar_b = obs_b + 144u;    // [2 tiles][1 + ENV_BUY_CHUNKS]
    const uint32_t envmkt_b = obs_b + 272u;    // [2 tiles] the next step's market rows landed (bulk copies)
    const uint32_t envin_b = obs_b + 288u;     // [2 tiles] both CTAs' heads' actions + log-prob partials landed
    const uint32_t obsa_b = obs_b + 304u;      // FUSED: [8] obs atom kb landed (layer 0 starts on the first atom)
    uint8_t* const env_pst = base + bias_off + ACT_BIAS_FLOATS * 4 + ACT_BAR_BYTES;   // [2 tiles][persist] (FUSED)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(base + (tslot_s - base_u32));

    // persistent over M-tiles: cluster c (one CTA pair per M-tile) takes tiles mtile0 + c + it * nclusters
    const int cid = static_cast<int>(blockIdx.x >> 1);
    const int ncl = static_cast<int>(gridDim.x >> 1);
    struct Tile {
        int agent, env0, rows_valid;
    };
    // FUSED: iterations 0..T-1 are the steps, T the critic bootstrap pass (when val_out is set)
    const int n_iter = FUSED ? fe->T + (a.val_out ? 1 : 0) : 0;
    auto tile_of = [&](int it, Tile& tl) -> bool {
        if (FUSED && it >= n_iter) return false;
        const int k = FUSED ? cid : cid + it * ncl;
        if (k >= a.mtiles) return false;
        const int mtile = a.mtile0 + k;
        tl.agent = mtile / a.tiles_per_agent;
        const int tile_in_agent = mtile % a.tiles_per_agent;
        tl.env0 = tl.agent * a.per_agent + tile_in_agent * 128;
        const int rv = a.per_agent - tile_in_agent * 128;
        tl.rows_valid = rv > 128 ? 128 : rv;
        return true;
    };

    const int hid_half = a.hidden / 2;
    const int head_half = a.n_out_pad / 2;
    // TMEM: two accumulator buffers (layer l uses buffer l & 1), so layer l+1's MMAs can
    // start while the epilogue is still reading layer l's accumulator
    const uint32_t tbuf = static_cast<uint32_t>(hid_half > head_half ? hid_half : head_half);
    uint32_t tcols = 32;
    while (tcols < 2 * tbuf) tcols <<= 1;

    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < ACT_STAGES; ++s) {
                mbar_init(full_b + 8u * s, 1);
                mbar_init(empty_b + 8u * s, a.mc ? a.mc : 1);   // every consumer of a shared tile
            }
            mbar_init(obs_b, 1);
            mbar_init(accum_b, 2);        // one multicast commit from each CTA of the pair
            mbar_init(accl_b, 1);
            mbar_init(actfree_b, 1);
            for (int j = 0; j < 4; ++j) {
                mbar_init(ownrdy_b + 8u * j, 256);   // the 256 epilogue threads
                mbar_init(peerrdy_b + 8u * j, 1);    // the MMA thread's expect_tx + the peer's bytes
            }
            if (FUSED) {
                mbar_init(envdone_b, 2);
                mbar_init(envmkt_b, 1);
                mbar_init(envmkt_b + 8u, 1);
                mbar_init(envin_b, 1);        // the tile's own expect_tx arrival + the heads' bulk-copy bytes
                mbar_init(envin_b + 8u, 1);
                for (int kb = 0; kb < 8; ++kb) mbar_init(obsa_b + 8u * kb, 1);
                for (int g = 0; g < 2; ++g) {
                    mbar_init(envbar_b + 64u * g, 1);   // the env tile's TMA barrier
                    for (int c = 0; c < ENV_BUY_CHUNKS; ++c) mbar_init(envbar_b + 64u * g + 8u * (c + 1), 32);
                }
            }
            fence_mbar_init();
            prefetch_tmap(&maps.obs);
            for (int l = 0; l < a.n_layers; ++l) prefetch_tmap(&maps.w[l]);
        }
        __syncwarp();
        tmem_alloc(tslot_s, tcols);
    }
    tc_fence_before();
    cluster_sync_all();          // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    // the env-step grid that follows may be scheduled now (its blocks stage their inputs on free SMs and
    // wait for this grid's completion before reading the actions); a no-op without a dependent
    if (!FUSED && threadIdx.x == 0) pdl_launch_dependents();
    const uint32_t tmem = *tslot;
    unsigned long long* tr = (a.trace && !FUSED) ? a.trace + blockIdx.x * 64 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = clock64();
#ifdef POD_EXP_GTIME
    if (!FUSED && threadIdx.x == 0 && a.t < 1024) atomicMin(&g_gtime[a.t][0], gtimer());
#endif

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0, seq = 0;
            uint32_t phase = 0;
            Tile tl;
            for (int it = 0; tile_of(it, tl); ++it) {
                // the obs tile goes into act_s once this CTA's MMAs of the previous tile are done with it
                // (FUSED: and both CTAs' env steps of the previous step, which write s_{t+1} and use act_s
                // as their shared memory, are done; the first ring stages of layer 0 are issued before that
                // wait, so the weight stream of step t+1 starts during the env step of step t)
                bool obs_issued = false;
                int pre = it > 0 ? ACT_STAGES : 0;
                auto issue_obs = [&] {
                    if (it > 0) mbar_wait(actfree_b, static_cast<uint32_t>(it - 1) & 1u);
                    if (FUSED && it > 0) mbar_wait_cluster(envdone_b, static_cast<uint32_t>(it - 1) & 1u);
                    const int kb0 = a.k_pad / 64;
                    const int row0 = FUSED ? it * a.N : a.obs_row0;
                    if constexpr (FUSED) {   // one barrier per atom: layer 0's MMAs start as the first atom lands
                        for (int kb = 0; kb < kb0; ++kb) {
                            mbar_arrive_expect_tx(obsa_b + 8u * kb, 16384u);
                            tma_load_2d(act_s + kb * 16384u, &maps.obs, kb * 64, row0 + tl.env0, obsa_b + 8u * kb);
                        }
                    } else {
                        mbar_arrive_expect_tx(obs_b, static_cast<uint32_t>(kb0) * 16384u);
                        for (int kb = 0; kb < kb0; ++kb)
                            tma_load_2d(act_s + kb * 16384u, &maps.obs, kb * 64, row0 + tl.env0, obs_b);
                    }
                    obs_issued = true;
                };
                auto before_stage = [&](int l) {
                    if constexpr (FUSED) {
                        if (l == 0 && !obs_issued && pre-- == 0) issue_obs();
                    }
                };
                if constexpr (!FUSED) issue_obs();
                for (int l = 0; l < a.n_layers; ++l) {
                    if constexpr (FUSED) {
                        if (l == 1 && !obs_issued) issue_obs();
                    }
                    const int K = l == 0 ? a.k_pad : a.hidden;
                    const int half = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad) / 2;
                    const int bn = actor_bn(half);
                    const int KB = K / ACT_BK;                                          // 32-wide K blocks
                    const int kbo = l == 0 ? 0 : static_cast<int>(rank) * (KB / 2);   // own half of h_l first
                    const int kp = static_cast<int>((a.kpb_pack >> (5 * l)) & 31u);
                    if (__builtin_expect(kp > 1, 0)) {
                        // narrow layer: kp K blocks per stage, one 4-D box (half == bn here)
                        const int ns = KB / kp;
                        const int kso = l == 0 ? 0 : static_cast<int>(rank) * (ns / 2);
                        for (int j = 0; j < ns; ++j) {
                            const int ks = (j + kso) % ns;
                            before_stage(l);
                            mbar_wait(empty_b + 8u * stage, phase ^ 1u);
                            const uint32_t sbytes = static_cast<uint32_t>(bn * kp) * (ACT_BK * 2);
                            mbar_arrive_expect_tx(full_b + 8u * stage, sbytes);
                            if (a.wt)
                                bulk_g2s(ring_s + stage * stage_bytes,
                                         a.wt + a.wt_agent_bytes * tl.agent + a.wt_layer_off[l] +
                                             static_cast<uint64_t>(rank) * half * K * 2 + static_cast<uint64_t>(ks) * sbytes,
                                         sbytes, full_b + 8u * stage);
                            else
                                tma_load_4d(ring_s + stage * stage_bytes, &maps.w[l], 0, static_cast<int>(rank) * half,
                                            ks * kp, tl.agent, full_b + 8u * stage);
                            ++seq;
                            if (++stage == ACT_STAGES) {
                                stage = 0;
                                phase ^= 1u;
                            }
                        }
                        continue;
                    }
                    for (int c = 0; c < half / bn; ++c) {
                        for (int j = 0; j < KB; ++j) {
                            const int kb = (j + kbo) % KB;
                            before_stage(l);
                            mbar_wait(empty_b + 8u * stage, phase ^ 1u);
                            mbar_arrive_expect_tx(full_b + 8u * stage, static_cast<uint32_t>(bn) * (ACT_BK * 2));
                            if (a.wt) {
                                const uint32_t sbytes = static_cast<uint32_t>(bn) * (ACT_BK * 2);
                                bulk_g2s(ring_s + stage * stage_bytes,
                                         a.wt + a.wt_agent_bytes * tl.agent + a.wt_layer_off[l] +
                                             static_cast<uint64_t>(rank) * half * K * 2 + static_cast<uint64_t>(c) * bn * K * 2 +
                                             static_cast<uint64_t>(kb) * sbytes,
                                         sbytes, full_b + 8u * stage);
                            } else if (!a.mc) {
                                tma_load_3d(ring_s + stage * stage_bytes, &maps.w[l], kb * ACT_BK,
                                            static_cast<int>(rank) * half + c * bn, tl.agent, full_b + 8u * stage);
                            } else if ((seq & (a.mc - 1)) == static_cast<int>(cr >> 1)) {
                                // round robin over the M-tiles: this CTA fetches the stage for all of them
                                tma_load_3d_mc(ring_s + stage * stage_bytes, &maps.w[l], kb * ACT_BK,
                                               static_cast<int>(rank) * half + c * bn, tl.agent, full_b + 8u * stage,
                                               share_mask);
                            }
                            if (tr && seq < 16) tr[48 + seq] = clock64();
                            ++seq;
                            if (++stage == ACT_STAGES) {
                                stage = 0;
                                phase ^= 1u;
                            }
                        }
                    }
                }
                if constexpr (FUSED) {
                    if (!obs_issued) issue_obs();
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint64_t adesc0 = sw128_desc(act_s);
            const uint64_t bdesc0 = ACT_BK == 16 ? sw32_desc(ring_s) : (ACT_BK == 64 ? sw128_desc(ring_s) : sw64_desc(ring_s));
            int stage = 0;
            uint32_t phase = 0;
            const int na = a.hidden / 128;           // activation atoms (64 cols) per CTA half
            Tile tl;
            for (int it = 0; tile_of(it, tl); ++it) {
                if constexpr (!FUSED) {
                    mbar_wait(obs_b, static_cast<uint32_t>(it) & 1u);
                    tc_fence_after();
                }

                if (tr && it == 0) tr[1] = clock64();
                for (int l = 0; l < a.n_layers; ++l) {
                    const int g = it * a.n_layers + l;                 // layer count over tiles: TMEM buffer g & 1
                    if (tr && it == 0) tr[2 + 4 * l] = clock64();
                    const int K = l == 0 ? a.k_pad : a.hidden;
                    const int half = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad) / 2;
                    const int bn = actor_bn(half);
                    const uint32_t idesc = idesc_bf16_f32(128, static_cast<uint32_t>(bn));
                    const int KB = K / ACT_BK;                 // 32-wide K blocks (two per activation atom)
                    const int kbo = l == 0 ? 0 : static_cast<int>(rank) * na * ACT_KPA;   // own atoms of h_l first
                    // phase of the atom barriers: one completion per hidden epilogue, over tiles
                    const uint32_t par = static_cast<uint32_t>(it * (a.n_layers - 1) + l - 1) & 1u;
                    const int kp = static_cast<int>((a.kpb_pack >> (5 * l)) & 31u);
                    if (__builtin_expect(kp > 1, 0)) {
                        // narrow layer: kp K blocks per stage (sub-tiles of bn x 64 B, consecutive)
                        const uint32_t sub16 = static_cast<uint32_t>(bn) * (ACT_BK * 2) >> 4;
                        const uint32_t dt = tmem + (static_cast<uint32_t>(g) & 1u) * tbuf;
                        for (int j0 = 0; j0 < KB; j0 += kp) {
                            for (int q = 0; q < kp; ++q) {
                                const int j = j0 + q;
                                const int kb = j + kbo < KB ? j + kbo : j + kbo - KB;
                                if (FUSED && l == 0 && (j % ACT_KPA) == 0) {
                                    mbar_wait(obsa_b + 8u * (j / ACT_KPA), static_cast<uint32_t>(it) & 1u);
                                    tc_fence_after();
                                }
#ifdef POD_EXP_GTIME
                                // fused rollout, CTA 0: [step][obs atom 0 landed, head accumulator ready, ...]
                                if (FUSED && l == 0 && j == 0 && blockIdx.x == 0 && it < 1024) g_ftime[it][0] = gtimer();
#endif
                                if (l > 0 && (j % ACT_KPA) == 0) {
                                    const int ja = j / ACT_KPA;
                                    if (ja < na) {
                                        mbar_wait(ownrdy_b + 8u * ja, par);
                                    } else {
                                        mbar_arrive_expect_tx(peerrdy_b + 8u * (ja - na), 16384u);
                                        mbar_wait(peerrdy_b + 8u * (ja - na), par);
                                    }
                                    tc_fence_after();
                                }
                                if (q == 0) {
                                    mbar_wait(full_b + 8u * stage, phase);
                                    tc_fence_after();
                                }
                                const uint64_t ad =
                                    adesc0 + (((kb / ACT_KPA) * 16384u + (kb % ACT_KPA) * (ACT_BK * 2u)) >> 4);
                                const uint64_t bd = bdesc0 + ((stage * stage_bytes) >> 4) + static_cast<uint32_t>(q) * sub16;
    #pragma unroll
                                for (int h = 0; h < ACT_BK / 16; ++h)
                                    mma_bf16(dt, ad + 2 * h, bd + 2 * h, idesc, (j != 0 || h > 0) ? 1u : 0u);
                            }
                            mma_commit(empty_b + 8u * stage);
                            if (++stage == ACT_STAGES) {
                                stage = 0;
                                phase ^= 1u;
                            }
                        }
                    } else
                    for (int c = 0; c < half / bn; ++c) {
                        for (int j = 0; j < KB; ++j) {
                            const int kb = j + kbo < KB ? j + kbo : j + kbo - KB;
                            if (FUSED && l == 0 && c == 0 && (j % ACT_KPA) == 0) {
                                mbar_wait(obsa_b + 8u * (j / ACT_KPA), static_cast<uint32_t>(it) & 1u);
                                tc_fence_after();
                            }
#ifdef POD_EXP_GTIME
                            // fused rollout, CTA 0: [step][obs atom 0 landed, head accumulator ready, ...]
                            if (FUSED && l == 0 && j == 0 && blockIdx.x == 0 && it < 1024) g_ftime[it][0] = gtimer();
#endif
                            if (l > 0 && c == 0 && (j % ACT_KPA) == 0) {
                                // h_l atom by atom: own atoms as the epilogue finishes them, then the
                                // peer's atoms as its bulk copies land
                                const int ja = j / ACT_KPA;
                                if (ja < na) {
                                    mbar_wait(ownrdy_b + 8u * ja, par);
                                } else {
                                    mbar_arrive_expect_tx(peerrdy_b + 8u * (ja - na), 16384u);
                                    mbar_wait(peerrdy_b + 8u * (ja - na), par);
                                }
                                tc_fence_after();
                            }
                            mbar_wait(full_b + 8u * stage, phase);
                            tc_fence_after();
                            if (tr && it == 0 && l == 0 && c * KB + j < 16) tr[32 + c * KB + j] = clock64();
                            // descriptors: precomputed bases + the start-address field (16-B units)
                            const uint64_t ad =
                                adesc0 + (((kb / ACT_KPA) * 16384u + (kb % ACT_KPA) * (ACT_BK * 2u)) >> 4);
                            const uint64_t bd = bdesc0 + ((stage * stage_bytes) >> 4);
                            const uint32_t dt = tmem + (static_cast<uint32_t>(g) & 1u) * tbuf + static_cast<uint32_t>(c * bn);
    #pragma unroll
                            for (int h = 0; h < ACT_BK / 16; ++h)
                                mma_bf16(dt, ad + 2 * h, bd + 2 * h, idesc, (j != 0 || h > 0) ? 1u : 0u);
                            if (a.mc) mma_commit_mc(empty_b + 8u * stage, share_mask);   // free it in both CTAs
                            else mma_commit(empty_b + 8u * stage);
                            if (++stage == ACT_STAGES) {
                                stage = 0;
                                phase ^= 1u;
                            }
                        }
                    }
                    if (tr && it == 0) tr[3 + 4 * l] = clock64();
                    mma_commit(accl_b);                  // this CTA's accumulator is complete
                    mma_commit_mc(accum_b, pair_mask);   // ... and the pair has read h_l
                }
                mma_commit(actfree_b);   // the next tile's obs may overwrite act_s once these MMAs are done
            }
        }
        __syncwarp();
    } else {
        // ===================== epilogue (warps 2..9) =====================
        const int ew = warp - 2;                   // 0..7
        const int etid = ew * 32 + lane;           // 0..255
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int hh = ew >> 2;                    // which half of this CTA's columns
        const int r = quad * 32 + lane;            // row of the tile == TMEM lane
        const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
        const int hq = head_half / 2;              // head tickers of this thread
        int staged_agent = -1;
        Tile tl;
        if constexpr (FUSED) {
            if (fe->persist && fe->T > 0 && tile_of(0, tl)) {
                // this CTA's two env tiles: their state from HBM into the persistent shared-memory copies, and the
                // first step's market rows
                const int grp = ew >> 2, gtid = etid & 127;
                const int etile = (tl.env0 >> 5) + 2 * static_cast<int>(rank) + grp;
                uint8_t* pst = env_pst + grp * fe->persist;
                const EnvArgs& ea = fe->env;
                if (gtid < 32) {
                    double* pl = reinterpret_cast<double*>(pst + ENVP_LEDGER);
                    const int64_t ee = static_cast<int64_t>(etile) * 32 + gtid;
                    pl[gtid] = ea.cash[ee];
                    pl[32 + gtid] = ea.asset[ee];
                    pl[64 + gtid] = ea.disc[ee];
                }
                if (gtid == 0) {
                    const int64_t s0 = ea.tile_start[etile];
                    const int k0 = ea.tile_k[etile];
                    *reinterpret_cast<int64_t*>(pst + ENVP_HDR) = s0;
                    *reinterpret_cast<int32_t*>(pst + ENVP_HDR + 8) = k0;
                    *reinterpret_cast<double*>(pst + ENVP_HDR + 16) = ea.tile_gpow[etile];
                    env_mkt_issue(ea, pst, s0, k0, envmkt_b + 8u * grp);
                }
            }
        }
        for (int it = 0; tile_of(it, tl); ++it) {
            const int e = tl.env0 + r;
            const bool valid = r < tl.rows_valid && e < a.N;
            if (tl.agent != staged_agent) {
                // stage this CTA's halves of the agent's biases and log-std in smem
                if (staged_agent >= 0) named_bar_sync(1, 256);   // every thread is done with the previous agent's
                const char* slab = a.params + tl.agent * a.param_bytes;
                int off = 0;
                for (int l = 0; l < a.n_layers; ++l) {
                    const int half = actor_layer_out(l, a.n_layers, a.hidden, a.n_out_pad) / 2;
                    const float* b = reinterpret_cast<const float*>(slab + a.b_off[l]) + rank * half;
                    for (int j = etid; j < half; j += 256) bias_s[off + j] = b[j];
                    off += half;
                }
                const float* ls = reinterpret_cast<const float*>(slab + a.log_std_off) + rank * head_half;
                for (int j = etid; j < head_half; j += 256) {
                    bias_s[off + j] = ls[j];
                    bias_s[off + head_half + j] = expf(ls[j]);   // sigma
                }
                staged_agent = tl.agent;
            }
            // this iteration's outputs (FUSED: the slices of step it; iteration T is the value-only pass)
            const bool vo = a.value_only || (FUSED && it == fe->T);
            const bool det = a.deterministic || vo;
            const int64_t so = FUSED ? it : 0;
            const int64_t Nn = static_cast<int64_t>(a.N) * a.n;
            float* const act_out = vo ? nullptr : a.act_out + so * Nn;
            float* const mu_out = (vo || !a.mu_out) ? nullptr : a.mu_out + so * Nn;
            int16_t* const dbg_aint = (vo || !a.dbg_aint) ? nullptr : a.dbg_aint + so * Nn;
            float* const logp_out = (vo || !a.logp_out) ? nullptr : a.logp_out + so * a.N;
            float* const val_out = a.val_out ? a.val_out + so * a.N : nullptr;
            // FUSED: both CTAs' env steps of the previous step are done (the noise of this step is written)
            if (FUSED && it > 0) mbar_wait_cluster(envdone_b, static_cast<uint32_t>(it - 1) & 1u);
            // prefetch this thread's head noise z (written by the previous env step; L2 loads: the peer CTA
            // writes half of it inside the fused kernel):
            // one round of independent loads, long before the head needs them
            float zr[ACT_MAX_HQ];
#pragma unroll
            for (int q = 0; q < ACT_MAX_HQ; ++q) {
                const int i = static_cast<int>(rank) * head_half + hh * hq + q;
                const float* zp = a.znoise + static_cast<int64_t>(i) * a.N + e;
                zr[q] = (q < hq && valid && i < a.n && !det) ? (FUSED ? __ldcg(zp) : *zp) : 0.0f;
            }
            named_bar_sync(1, 256);
            int boff = 0;
            for (int l = 0; l < a.n_layers - 1; ++l) {
                const int g = it * a.n_layers + l;
                const uint32_t hpar = static_cast<uint32_t>(it * (a.n_layers - 1) + l) & 1u;
                // this CTA's MMAs of layer l are done (its accumulator is final and its act_s is free for
                // its own atoms); the peer's, before shipping atoms into its act_s (below)
                mbar_wait(accl_b, static_cast<uint32_t>(g) & 1u);
                tc_fence_after();
                if (tr && it == 0 && etid == 0) tr[4 + 4 * l] = clock64();
                // h_{l+1} atom by atom (64 columns = 8 warps x 32 columns x 128 rows), so the next
                // layer's MMAs and the DSMEM copy of each atom start as soon as it is written
                const int na = hid_half / 64;
                for (int j = 0; j < na; ++j) {
                    const int tc = j * 64 + hh * 32;                      // TMEM column (local)
                    uint32_t v[32];
                    tmem_ld32(trow + (static_cast<uint32_t>(g) & 1u) * tbuf + static_cast<uint32_t>(tc), v);
                    tmem_ld_wait();
                    const float4* b4 = reinterpret_cast<const float4*>(bias_s + boff + tc);
                    uint32_t pk[16];
                    epi_pack(v, b4, a.act, pk);
                    const int atom_g = static_cast<int>(rank) * na + j;           // global atom of h_{l+1}
                    const uint32_t atom = act_s + static_cast<uint32_t>(atom_g) * 16384u;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        st_shared_v4(atom + sw128_offset(static_cast<uint32_t>(r), static_cast<uint32_t>(hh * 4 + q)),
                                     pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                    fence_proxy_async_smem();
                    tc_fence_before();
                    mbar_arrive(ownrdy_b + 8u * j);
                    if (etid == 0) {
                        // the whole atom is written: ship it to the same offset in the peer, once the
                        // peer's MMAs are done reading its h_l
                        if (j == 0) mbar_wait(accum_b, static_cast<uint32_t>(g) & 1u);
                        mbar_wait(ownrdy_b + 8u * j, hpar);
                        bulk_s2peer(mapa_shared(atom, peer), atom, 16384u, mapa_shared(peerrdy_b + 8u * j, peer));
                    }
                }
                boff += hid_half;
                if (tr && it == 0 && etid == 0) tr[5 + 4 * l] = clock64();
            }
            // ----- head: this CTA's tickers [rank*head_half, ...), this warp's quarter of them
            const int L = a.n_layers - 1;
            const int gL = it * a.n_layers + L;
            mbar_wait(accl_b, static_cast<uint32_t>(gL) & 1u);
            tc_fence_after();
#ifdef POD_EXP_GTIME
            if (FUSED && blockIdx.x == 0 && etid == 0 && it < 1024) g_ftime[it][1] = gtimer();
#endif
            if (tr && it == 0 && etid == 0) tr[24] = clock64();
            // the head: sampling, the action map and the log-prob partials
            // FUSED: this thread's row is env lane `lane` of env tile `quad` of the M-tile (it lives in CTA quad >> 1, env
            // group quad & 1).  The head stages that tile's actions of this CTA's tickers ([head_half][32] int16) and its
            // two log-prob partials ([2][32] float) in this CTA's activation buffer past the env tiles' areas, and the
            // quad's two warps ship them with two bulk DSMEM copies into the tile's aint_s / stg, counted on its envin_b
            int16_t* aint_stage = nullptr;
            float* logp_stage = nullptr;
            if constexpr (FUSED) {
                uint8_t* qs = base + 2 * fe->env_stride + quad * FUSED_QUAD_STAGE;
                aint_stage = reinterpret_cast<int16_t*>(qs);
                logp_stage = reinterpret_cast<float*>(qs + ACT_MAX_HQ * 2 * 64);
            }
            auto head = [&] {
            const float* bias = bias_s + boff;
            const float* log_std = bias_s + boff + head_half;
            const float* sigma = bias_s + boff + 2 * head_half;
            float logp = 0.0f;
            // non-finite mean detector: 0 * mu is 0 for finite mu and NaN for inf / NaN, so the sum turns NaN iff
            // some (unmasked) mean is not finite — one predicated FMA per ticker
            float nanacc = 0.0f;
            const float half_ln_2pi = 0.918938533204672742f;
            const bool fast_map = FUSED && a.h_max <= 128;
            const float hmax_f = static_cast<float>(a.h_max);
            const bool vec = (a.n % 4) == 0;
            const int i00 = static_cast<int>(rank) * head_half;
    #pragma unroll
            // the next chunk's 8 accumulator columns are loaded while this chunk is processed (hn)
            const uint32_t hbase = trow + (static_cast<uint32_t>(gL) & 1u) * tbuf + static_cast<uint32_t>(hh * hq);
            uint32_t hn[8];
            __syncwarp();
            tmem_ld8(hbase, hn);
            tmem_ld_wait();
            for (int cc = 0; cc < ACT_MAX_HQ / 8; ++cc) {
                if (cc >= hq / 8) break;
                const int tc = hh * hq + cc * 8;                         // TMEM column (local)
                const int i0 = i00 + tc;                                 // global ticker
                uint32_t hv[8];
    #pragma unroll
                for (int jj = 0; jj < 8; ++jj) hv[jj] = hn[jj];
                __syncwarp();
                if (cc + 1 < hq / 8) tmem_ld8(hbase + static_cast<uint32_t>(8 * (cc + 1)), hn);
                if (valid && i0 <= a.n && val_out && a.n < i0 + 8) {
                    // critic: head row n over the same trunk (R#22)
                    float vh = 0.0f;
    #pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if (i0 + jj == a.n) vh = __uint_as_float(hv[jj]);
                    val_out[e] = vh + bias[tc + (a.n - i0)];
                }
                if (valid && i0 < a.n && !vo) {
                    float raw[8], mu[8];
                    int16_t ai8[8];
                    // the chunk's 8 staged biases, log-stds and sigmas as 16-byte loads (8-column aligned)
                    float bz[8], lsz[8], sgz[8];
                    {
                        const float4* b4 = reinterpret_cast<const float4*>(bias + tc);
                        const float4* l4 = reinterpret_cast<const float4*>(log_std + tc);
                        const float4* s4 = reinterpret_cast<const float4*>(sigma + tc);
    #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const float4 x = b4[h], y = l4[h], w = s4[h];
                            bz[4 * h] = x.x; bz[4 * h + 1] = x.y; bz[4 * h + 2] = x.z; bz[4 * h + 3] = x.w;
                            lsz[4 * h] = y.x; lsz[4 * h + 1] = y.y; lsz[4 * h + 2] = y.z; lsz[4 * h + 3] = y.w;
                            sgz[4 * h] = w.x; sgz[4 * h + 1] = w.y; sgz[4 * h + 2] = w.z; sgz[4 * h + 3] = w.w;
                        }
                    }
    #pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        mu[jj] = __uint_as_float(hv[jj]) + bz[jj];
                        raw[jj] = mu[jj];
                    }
                    // per ticker: noise z ~ N(0,1) for (env, step, ticker) generated by the previous env step,
                    // raw = mu + sigma z, log-prob term, tanh on the SFU, integer map in float64.  One straight-line
                    // body for all 8 columns of the chunk, the tickers past n masked (their stores and log-prob
                    // terms predicated off): half the code of a separate guarded copy for the last chunk
                    // FUSED: the map's floor(|u| h_max + 1/2) is decided in float32 when that is provably the float64 result
                    // (h_max <= 128: |fl32(fl32(|u| h) + 1/2) - (|u| h + 1/2)| <= 2^-16, so a fractional part d in
                    // [2^-15, 1 - 2^-15] has the exact floor); a chunk in which any lane lands closer to a half-integer
                    // redoes its map in float64, the oracle's precision (R#6)
                    bool unsure = !fast_map;
    #pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const bool ok = i0 + jj < a.n;
                        const float z = zr[cc * 8 + jj];
                        const float ls = lsz[jj];
                        if (ok) nanacc = fmaf(mu[jj], 0.0f, nanacc);
                        raw[jj] = fmaf(sgz[jj], z, mu[jj]);
                        if (ok) logp += (-0.5f * z * z - ls) - half_ln_2pi;
                        const float u = tanh_sfu(raw[jj]);
                        if constexpr (FUSED) {
                            const float r = fmaf(fabsf(u), hmax_f, 0.5f);
                            const float fl = floorf(r);
                            const float d = r - fl;
                            unsure |= d < 3.0517578125e-05f || d > 0.999969482421875f;
                            const int m = static_cast<int>(fl);
                            ai8[jj] = static_cast<int16_t>(u < 0.0f ? -m : m);
                        } else {
                            const double m = floor(static_cast<double>(fabsf(u)) * static_cast<double>(a.h_max) + 0.5);
                            ai8[jj] = static_cast<int16_t>(u < 0.0f ? -static_cast<int>(m) : static_cast<int>(m));
                            if (ok) a.aint[static_cast<int64_t>(i0 + jj) * a.N + e] = ai8[jj];
                        }
                    }
                    if (FUSED && __any_sync(0xffffffffu, unsure)) {
    #pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const float u = tanh_sfu(raw[jj]);
                            const double m = floor(static_cast<double>(fabsf(u)) * static_cast<double>(a.h_max) + 0.5);
                            ai8[jj] = static_cast<int16_t>(u < 0.0f ? -static_cast<int>(m) : static_cast<int>(m));
                        }
                    }
                    if constexpr (FUSED) {
    #pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            if (i0 + jj < a.n) aint_stage[(i0 + jj - i00) * 32 + lane] = ai8[jj];
                    }
                    if (dbg_aint) {
                        for (int jj = 0; jj < 8 && i0 + jj < a.n; ++jj)
                            dbg_aint[static_cast<int64_t>(e) * a.n + i0 + jj] = ai8[jj];
                    }
                    float* arow = act_out + static_cast<int64_t>(e) * a.n + i0;
                    float* mrow = mu_out ? mu_out + static_cast<int64_t>(e) * a.n + i0 : nullptr;
                    if (vec && i0 + 8 <= a.n) {
                        reinterpret_cast<float4*>(arow)[0] = make_float4(raw[0], raw[1], raw[2], raw[3]);
                        reinterpret_cast<float4*>(arow)[1] = make_float4(raw[4], raw[5], raw[6], raw[7]);
                        if (mrow) {
                            reinterpret_cast<float4*>(mrow)[0] = make_float4(mu[0], mu[1], mu[2], mu[3]);
                            reinterpret_cast<float4*>(mrow)[1] = make_float4(mu[4], mu[5], mu[6], mu[7]);
                        }
                    } else {
    #pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            if (i0 + jj < a.n) {
                                arow[jj] = raw[jj];
                                if (mrow) mrow[jj] = mu[jj];
                            }
                        }
                    }
                }
                tmem_ld_wait();   // the next chunk's columns (hn)
            }
            if (nanacc != nanacc && valid) atomicOr(a.err, 1u);
            if (tr && it == 0 && etid == 0) tr[25] = clock64();
            // log-prob partial of (rank, hh) for row r -> the [4][N] scratch (FUSED: the env tile's stg); the env step
            // that follows combines the four partials ((p0 + p1) + p2) + p3, so the kernel's tail needs no exchange
            if constexpr (FUSED) {
                if (!vo) logp_stage[hh * 32 + lane] = logp;
            } else {
                if (valid && logp_out) a.logp_parts[static_cast<int64_t>(rank * 2 + hh) * a.N + e] = logp;
            }
            };
            if constexpr (FUSED) {
                if (!vo) {
                    // ----- the env step of step it on this CTA's two env tiles of the M-tile (epilogue warps
                    // 2-5: tile 2 rank, warps 6-9: tile 2 rank + 1); the tiles wait for both CTAs' heads' bulk copies
                    // deliveries on their envin_b, no fence or cluster barrier in between
                    const int grp = ew >> 2;
                    if ((etid & 127) == 0) {
                        // this CTA's env tile: its holdings TMA (the activation buffer is free once this CTA's head
                        // MMAs are done), and the bytes its envin_b awaits from both CTAs' heads
                        const int etile = (tl.env0 >> 5) + 2 * static_cast<int>(rank) + grp;
                        mbar_arrive_expect_tx(envbar_b + 64u * grp, static_cast<uint32_t>(a.n) * 128u);
                        tma_load_2d(base_u32 + static_cast<uint32_t>(grp * fe->env_stride), &emaps->hold, etile * 32, 0,
                                    envbar_b + 64u * grp);
                        mbar_arrive_expect_tx(envin_b + 8u * grp, static_cast<uint32_t>(a.n) * 64u + 512u);
                    }
                    head();
                    // ship this quad's staged actions and log-prob partials to its env tile (this CTA or the peer;
                    // the copies land in the tile's area of the activation buffer: the pair's head MMAs must be done)
                    fence_proxy_async_smem();
                    named_bar_sync(5 + static_cast<uint32_t>(quad), 64);
                    if (hh == 0 && lane == 0) {
                        const EnvSmemLayout ESL = env_smem_layout(a.n, a.k_pad);
                        const uint32_t dst = static_cast<uint32_t>(quad >> 1);
                        const uint32_t tb = base_u32 + static_cast<uint32_t>((quad & 1) * fe->env_stride);
                        const uint32_t inb = mapa_shared(envin_b + 8u * static_cast<uint32_t>(quad & 1), dst);
                        const int i00 = static_cast<int>(rank) * head_half;
                        const int rows = (a.n < i00 + head_half ? a.n : i00 + head_half) - i00;
                        mbar_wait(accum_b, static_cast<uint32_t>(gL) & 1u);
                        if (rows > 0)
                            bulk_s2peer(mapa_shared(tb + static_cast<uint32_t>(ESL.aint + i00 * 64), dst), smem_u32(aint_stage),
                                        static_cast<uint32_t>(rows * 64), inb);
                        bulk_s2peer(mapa_shared(tb + static_cast<uint32_t>(ESL.stg + rank * 256), dst), smem_u32(logp_stage),
                                    256u, inb);
                    }
#ifdef POD_EXP_GTIME
                    if (blockIdx.x == 0 && etid == 0 && it < 1024) g_ftime[it][2] = gtimer();
                    if (blockIdx.x == 0 && etid == 0 && it < 1024) g_ftime[it][3] = gtimer();
#endif
                    const EnvArgs& ea = fe->env;
                    EnvStep st;
                    st.rew = ea.rew + so * a.N;
                    st.done = ea.done + so * a.N;
                    st.obs_out = ea.obs_out + so * a.N * fe->k_pad;
                    st.dbg_hold = ea.dbg_hold ? ea.dbg_hold + so * Nn : nullptr;
                    st.dbg_cash = ea.dbg_cash ? ea.dbg_cash + so * a.N : nullptr;
                    st.equity = ea.equity ? ea.equity + so * a.N : nullptr;
                    st.logp_out = ea.logp_out ? ea.logp_out + so * a.N : nullptr;
                    st.gen_noise = (fe->sampling && it + 1 < fe->T) ? 1 : 0;
                    st.noise_t = it + 1;
                    env_step_tile<SELL_UNROLL, BUY_UNROLL>(*emaps, ea, st, (tl.env0 >> 5) + 2 * static_cast<int>(rank) + grp,
                                                           env_role_tid(warp, lane),
                                                           base + grp * fe->env_stride, envbar_b + 64u * grp,
                                                           static_cast<uint32_t>(it) & 1u, 3 + grp,
                                                           fe->persist ? env_pst + grp * fe->persist : nullptr,
                                                           envmkt_b + 8u * grp, it + 1 < fe->T, envin_b + 8u * grp);
#ifdef POD_EXP_GTIME
                    if (blockIdx.x == 0 && etid == 0 && it < 1024) g_ftime[it][4] = gtimer();
#endif
                    // s_{t+1} and the holdings (TMA reads of the next step), the noise (the peer's loads), and
                    // this tile's shared memory (the next obs tile lands there)
                    __threadfence();
                    fence_proxy_async_global();
                    fence_proxy_async_smem();
                    named_bar_sync(1, 256);
                    if (etid == 0) {
                        mbar_arrive(envdone_b);
                        mbar_arrive_remote(mapa_shared(envdone_b, peer));
#ifdef POD_EXP_GTIME
                        if (blockIdx.x == 0 && it < 1024) g_ftime[it][5] = gtimer();
#endif
                    }
                } else {
                    head();
                }
            } else {
                head();
            }
        }
    }

    tc_fence_before();
    cluster_sync_all();      // every cross-CTA arrival and DSMEM copy of the launch is complete
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, tcols);
    }
    if (tr && threadIdx.x == 0) tr[26] = clock64();
#ifdef POD_EXP_GTIME
    if (!FUSED && threadIdx.x == 0 && a.t < 1024) atomicMax(&g_gtime[a.t][1], gtimer());
#endif
}

__global__ void __launch_bounds__(ACT_THREADS, 1)
    actor_forward_kernel(const __grid_constant__ ActorMaps maps, const __grid_constant__ ActorArgs a) {
    actor_body<false, 1, 1>(maps, a, nullptr, nullptr);
}

// the fused rollout: grid = 2 x M-tiles (one wave), cluster 2; see FusedEnvArgs
template <int SELL_UNROLL, int BUY_UNROLL>
__global__ void __launch_bounds__(ACT_THREADS, 1)
    rollout_fused_kernel(const __grid_constant__ FusedMaps maps, const __grid_constant__ ActorArgs a,
                         const __grid_constant__ FusedEnvArgs fe) {
    actor_body<true, SELL_UNROLL, BUY_UNROLL>(maps.am, a, &maps.em, &fe);
}

}  // namespace pod
