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
// B200 mapping: one warp per env tile (32 envs that share an episode start
// row, hence the same market rows); lane = env.  The ledger is float64 and
// evaluated per lane in exactly the order written above (explicit __dmul_rn /
// __dadd_rn / __ddiv_rn, no FMA contraction), so cash, account value, reward
// and the integer holdings are bit-identical to a sequential float64
// implementation — a warp-parallel prefix over tickers would reassociate the
// cash sums and could flip a floor() at a near tie.  State is ticker-major
// (hold[i][env], a[i][env]) so every per-ticker access of the warp is one
// coalesced 128-B (64-B for int16) transaction.  The tile's market rows
// (p_t, p_{t+1}, p_0, feat_{t+1}) are staged once per warp in shared memory;
// the per-tile part of s_{t+1} (price ratios, indicators, zero pad) is built
// once per warp and each env row of s_{t+1} is then written by the whole warp
// with coalesced 16-byte stores (512 contiguous bytes per instruction).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace pod {

constexpr int ENV_WARPS = 4;          // tiles per block
constexpr int ENV_MAX_STOCKS = 128;
constexpr int ENV_MAX_KPAD = 512;

struct EnvArgs {
    int32_t N;
    int32_t n;
    int32_t f;
    int32_t k_pad;
    int32_t obs_dim;
    int32_t horizon;
    int32_t n_tiles;
    int32_t mode;             // 0 = step, 1 = write obs of the current state, 2 = reset + obs
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
    uint32_t* err;
};

struct EnvSmem {
    float p_t[ENV_MAX_STOCKS];
    float p_1[ENV_MAX_STOCKS];
    float p_0[ENV_MAX_STOCKS];
    __align__(16) uint16_t tmpl[ENV_MAX_KPAD];                 // per-tile part of the obs row
    __align__(16) uint16_t stg[32][((1 + ENV_MAX_STOCKS) + 7) / 8 * 8];  // per-env part
};

__device__ __forceinline__ uint16_t f2bf(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

__global__ void __launch_bounds__(32 * ENV_WARPS) env_step_kernel(const EnvArgs a) {
    __shared__ EnvSmem sm_all[ENV_WARPS];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tile = blockIdx.x * ENV_WARPS + warp;
    if (tile >= a.n_tiles) return;   // warp-uniform
    EnvSmem& sm = sm_all[warp];
    const int n = a.n;
    const int e = tile * 32 + lane;
    const bool active = e < a.N;
    const int64_t N = a.N;

    const int64_t s = a.tile_start[tile];
    const int k = a.mode == 2 ? 0 : a.tile_k[tile];
    const double gpow = a.mode == 2 ? 1.0 : a.tile_gpow[tile];
    const int64_t t = s + k;
    const bool stepping = a.mode == 0;
    const bool done = stepping && ((k + 1 == a.horizon) || (t + 1 == a.T_data - 1));
    // market row the next observation is taken at
    const int64_t t_obs = stepping ? (done ? s : t + 1) : t;

    // ---- stage the tile's market rows (all lanes, coalesced)
    for (int i = lane; i < n; i += 32) {
        sm.p_t[i] = a.close[t * n + i];
        sm.p_1[i] = stepping ? a.close[(t + 1) * n + i] : a.close[t * n + i];
        sm.p_0[i] = a.close[s * n + i];
    }
    __syncwarp();
    // ---- per-tile part of the observation: p/p0 at t_obs, indicators, zero pad
    {
        const int e_cols = 1 + n;
        for (int c = lane; c < a.k_pad; c += 32) {
            float v = 0.0f;
            if (c >= e_cols && c < e_cols + n) {
                const int i = c - e_cols;
                const float p = t_obs == s ? sm.p_0[i] : (t_obs == t ? sm.p_t[i] : sm.p_1[i]);
                v = p / sm.p_0[i];
            } else if (c >= e_cols + n && c < a.obs_dim) {
                const int j = c - e_cols - n;   // channel-major: j = ch * n + i
                v = a.feat[t_obs * a.f * n + j];
            }
            sm.tmpl[c] = f2bf(v);
        }
    }
    __syncwarp();

    if (active) {
        double cash, v;
        if (a.mode == 2) {
            cash = a.C0;
            for (int i = 0; i < n; ++i) a.hold[i * N + e] = 0;
            a.cash[e] = a.C0;
            a.asset[e] = a.C0;
            a.disc[e] = 0.0;
            a.ep_ret[e] = 0.0;
        } else {
            cash = a.cash[e];
        }
        if (stepping) {
            v = a.asset[e];
            const double omc = __dadd_rn(1.0, -a.cost);
            const double opc = __dadd_rn(1.0, a.cost);
            // selling set (Eq. 3 "+ (p^S)^T k^S")
            for (int i = 0; i < n; ++i) {
                const int ai = a.aint[i * N + e];
                if (ai < 0) {
                    const int h = a.hold[i * N + e];
                    const int q = min(h, -ai);
                    cash = __dadd_rn(cash, __dmul_rn(__dmul_rn(static_cast<double>(sm.p_t[i]), static_cast<double>(q)), omc));
                }
            }
            // buying set (Eq. 3 "- (p^B)^T k^B"), then revalue at p_{t+1} (Eq. 2)
            double ph = 0.0;
            const float inv_c0 = static_cast<float>(1.0 / a.C0);
            for (int i = 0; i < n; ++i) {
                const int ai = a.aint[i * N + e];
                int h = a.hold[i * N + e];
                if (ai < 0) h -= min(h, -ai);
                if (ai > 0) {
                    const double unit = __dmul_rn(static_cast<double>(sm.p_t[i]), opc);
                    double qmax = floor(__ddiv_rn(cash, unit));
                    if (__dmul_rn(qmax, unit) > cash) qmax = __dadd_rn(qmax, -1.0);
                    double q = static_cast<double>(ai) < qmax ? static_cast<double>(ai) : qmax;
                    q = q < 0.0 ? 0.0 : q;
                    h += static_cast<int>(q);
                    cash = __dadd_rn(cash, -__dmul_rn(q, unit));
                }
                ph = __dadd_rn(ph, __dmul_rn(static_cast<double>(sm.p_1[i]), static_cast<double>(h)));
                a.hold[i * N + e] = done ? 0 : h;
                if (a.dbg_hold) a.dbg_hold[static_cast<int64_t>(e) * n + i] = h;
                sm.stg[lane][1 + i] = done ? f2bf(0.0f) : f2bf(static_cast<float>(h) * sm.p_1[i] * inv_c0);
            }
            const double v1 = __dadd_rn(cash, ph);
            const double r = __dmul_rn(a.scale, __dadd_rn(v1, -v));
            double disc = __dadd_rn(a.disc[e], __dmul_rn(gpow, r));
            a.rew[e] = static_cast<float>(r);
            a.done[e] = done ? 1 : 0;
            if (a.dbg_cash) a.dbg_cash[e] = cash;
            if (!isfinite(v1)) atomicOr(a.err, 2u);
            if (done) {
                a.ep_ret[e] = disc;
                cash = a.C0;
                v = a.C0;
                disc = 0.0;
            } else {
                v = v1;
            }
            a.cash[e] = cash;
            a.asset[e] = v;
            a.disc[e] = disc;
        } else {
            const float inv_c0 = static_cast<float>(1.0 / a.C0);
            for (int i = 0; i < n; ++i) {
                const int h = a.mode == 2 ? 0 : a.hold[i * N + e];
                sm.stg[lane][1 + i] = f2bf(static_cast<float>(h) * sm.p_t[i] * inv_c0);
            }
        }
        sm.stg[lane][0] = f2bf(static_cast<float>(cash / a.C0));
    }
    const int e_pad = (1 + n + 7) / 8 * 8;   // per-env staging width, 16-B multiple
    if (active) {
        for (int c = 1 + n; c < e_pad; ++c) sm.stg[lane][c] = sm.tmpl[c];
    }
    if (lane == 0 && stepping) {
        a.tile_k[tile] = done ? 0 : k + 1;
        a.tile_gpow[tile] = done ? 1.0 : __dmul_rn(gpow, a.gamma);
    }
    if (lane == 0 && a.mode == 2) {
        a.tile_k[tile] = 0;
        a.tile_gpow[tile] = 1.0;
    }
    __syncwarp();
    // ---- write s_{t+1}: each env row by the whole warp, 16-B chunks
    if (a.obs_out) {
        const int chunks = a.k_pad / 8;
        const int rows = min(32, a.N - tile * 32);
        for (int row = 0; row < rows; ++row) {
            uint4* dst = reinterpret_cast<uint4*>(a.obs_out + (static_cast<int64_t>(tile) * 32 + row) * a.k_pad);
            for (int c = lane; c < chunks; c += 32) {
                const uint4 val = c * 8 < e_pad ? *reinterpret_cast<const uint4*>(&sm.stg[row][c * 8])
                                                : *reinterpret_cast<const uint4*>(&sm.tmpl[c * 8]);
                dst[c] = val;
            }
        }
    }
}

// injected actions: a[i][e] = sgn(u) floor(|u| h_max + 1/2)  (R#6)
__global__ void inject_map_kernel(const float* __restrict__ u, int N, int n, int h_max, int16_t* __restrict__ aint,
                                  int16_t* __restrict__ dbg_aint) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(N) * n) return;
    const int e = static_cast<int>(idx / n);
    const int i = static_cast<int>(idx % n);
    const float x = u[idx];
    const double m = floor(static_cast<double>(fabsf(x)) * static_cast<double>(h_max) + 0.5);
    const int ai = x < 0.0f ? -static_cast<int>(m) : static_cast<int>(m);
    aint[static_cast<int64_t>(i) * N + e] = static_cast<int16_t>(ai);
    if (dbg_aint) dbg_aint[idx] = static_cast<int16_t>(ai);
}

// J_a = (sum over agent a's envs of ep_ret) / per_agent, one block per agent
__global__ void fitness_kernel(const double* __restrict__ ep_ret, int per_agent, double* __restrict__ out) {
    __shared__ double red[256];
    const int agent = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < per_agent; i += blockDim.x) acc += ep_ret[static_cast<int64_t>(agent) * per_agent + i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[agent] = red[0] / static_cast<double>(per_agent);
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
