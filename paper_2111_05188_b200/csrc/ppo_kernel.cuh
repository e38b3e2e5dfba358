// ppo_kernel.cuh — learner kernels of the PPO clipped-surrogate update.
//
// Method ("Proximal Policy Optimization (PPO)"; Table 3 hyper-parameters; S:L284–292;
// reading R#26).  Per sample of a minibatch of B rows (mean over the minibatch):
//   z_i = (raw_i - mu_i) / sigma_i,  logp = sum_i (-z_i^2/2 - log sigma_i - ln(2 pi)/2)
//   rho = exp(logp - logp_old),  s1 = rho A,  s2 = clip(rho, 1 - eps, 1 + eps) A
//   L = -mean(min(s1, s2)) - c_ent sum_i (log sigma_i + (1 + ln 2 pi)/2) + c_v mean((V - R)^2)
// Gradients at the head (the min's derivative is that of s1 when s1 <= s2 — inside the clip range
// both coincide — and 0 otherwise):
//   dL/dmu_i      = -(1/B) [s1 <= s2] A rho z_i / sigma_i
//   dL/dlog sig_i = -(1/B) sum_b [s1 <= s2] A rho (z_i^2 - 1) - c_ent
//   dL/dV         = (2 c_v / B) (V - R)
// The layer contractions are gemm_kernel.cuh's (tcgen05 bf16, or the float32 reference core); these
// kernels are the gather (row-major + transposed minibatch observations), the head loss (delta of the head
// layer, row-major + transposed, per-block partial sums of the head bias and log-std gradients), the
// fixed-order reduction of all bias partials, the transposed weights W_l^T for the input-gradient products,
// and the Adam step on the float32 master (skipped when the minibatch's loss was not finite).
// T = the operand type (bf16 for the tensor-core learner, float for the reference mode).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

#include "fuse_kernel.cuh"
#include "gemm_kernel.cuh"

namespace pod {

// per-call values in device memory (written by ppo_set_step_kernel before the captured minibatch loop), so
// one graph serves every call of a schedule: the Adam step base and the hyper-parameters; `err` is set by
// the head kernel when a sample's objective or value loss is not finite (divergence)
struct PpoDev {
    int64_t step_base;
    float ratio_clip, entropy_coef, value_coef, lr, b1, b2, eps;
    uint32_t err;
};

constexpr int PPO_HEAD_WARPS = 32;                                // one sample per warp: the head's latency is
constexpr int PPO_HEAD_SPW = 1;                                   // one sample's (samples per warp)
constexpr int PPO_HEAD_ROWS = PPO_HEAD_WARPS * PPO_HEAD_SPW;      // samples per block (32: one partial per 32 rows)

template <class T>
struct PpoHead {
    int32_t B, B_pad, n, n_out_pad, kp64;
    PpoDev* hpd;
    const float* act;        // [B_pad][n] raw actions of the minibatch
    const float* logp_old;   // [B_pad]
    const float* adv;        // [B_pad]
    const float* ret;        // [B_pad]
    const float* zh;         // [B_pad][n_out_pad] head output (mu in 0..n-1, V in n)
    const float* log_std;    // [n_out_pad] (master)
    T* delta;                // [B_pad][kp64] dL/d head output (pad columns 0)
    T* delta_t;              // [n_out_pad][B_pad]
    float* bpart;            // [B_pad / 32][n_out_pad] head-bias gradient partials of each block
    float* lspart;           // [B_pad / 32][n_out_pad] log-std gradient partials of each block
    double* losses;          // [4]
};

// gather the minibatch rows perm[0..B) of the flattened buffer into X0 [B_pad][k_pad] and X0^T
// [k_pad][B_pad] (padded rows zero) plus the per-row scalars; block = 32 rows x (k_pad) columns
template <class T>
__global__ void __launch_bounds__(256) ppo_gather_kernel(const uint16_t* __restrict__ obs, const float* __restrict__ act,
                                                         const float* __restrict__ lpo, const float* __restrict__ adv,
                                                         const float* __restrict__ ret, const int32_t* __restrict__ perm,
                                                         int B, int B_pad, int k_pad, int n, T* __restrict__ x0,
                                                         T* __restrict__ x0t, float* __restrict__ act_b,
                                                         float* __restrict__ lpo_b, float* __restrict__ adv_b,
                                                         float* __restrict__ ret_b) {
    __shared__ float tile[32][65];
    const int r0 = blockIdx.x * 32;
    const int c0 = blockIdx.y * 64;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;   // 64 columns x 4 row lanes
    int64_t src[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {   // the 8 rows of this thread: index loads first, then the row loads
        const int r = r0 + ty + 4 * q;
        src[q] = r < B ? static_cast<int64_t>(perm[r]) : -1;
    }
    uint16_t raw[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) raw[q] = src[q] >= 0 ? obs[src[q] * k_pad + c0 + tx] : static_cast<uint16_t>(0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int rr = ty + 4 * q;
        const float v = __uint_as_float(static_cast<uint32_t>(raw[q]) << 16);
        tile[rr][tx] = v;
        x0[static_cast<int64_t>(r0 + rr) * k_pad + c0 + tx] = from_f32<T>(v);
    }
    __syncthreads();
    // transposed: 64 columns x 32 rows, rows consecutive per warp
    for (int idx = threadIdx.x; idx < 64 * 32; idx += 256) {
        const int c = idx >> 5, rr = idx & 31;
        x0t[static_cast<int64_t>(c0 + c) * B_pad + r0 + rr] = from_f32<T>(tile[rr][c]);
    }
    if (blockIdx.y == 0) {
        for (int rr = ty; rr < 32; rr += 4) {
            const int r = r0 + rr;
            const int64_t src = r < B ? perm[r] : 0;
            for (int c = tx; c < n; c += 64) act_b[static_cast<int64_t>(r) * n + c] = r < B ? act[src * n + c] : 0.0f;
            if (tx == 0) {
                lpo_b[r] = r < B ? lpo[src] : 0.0f;
                adv_b[r] = r < B ? adv[src] : 0.0f;
                ret_b[r] = r < B ? ret[src] : 0.0f;
            }
        }
    }
}

// one warp per sample (lanes over tickers): head loss and dL/d(head output) -> delta (row-major, padded
// columns 0) and delta^T; the block's partial sums of the head-bias and log-std gradients go to
// [blockIdx][...] (reduced in a fixed order by ppo_bias_reduce_kernel); loss sums by one atomic per block.
// Rows b >= B (padding) write zeros.  A non-finite objective or value loss sets hpd->err.
template <class T>
__global__ void __launch_bounds__(32 * PPO_HEAD_WARPS) ppo_head_kernel(const PpoHead<T> h) {
    __shared__ float g_ls[PPO_HEAD_WARPS][128];
    __shared__ float g_b[PPO_HEAD_WARPS][128];
    __shared__ double red[3][PPO_HEAD_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float h_eps = h.hpd->ratio_clip, h_c_v = h.hpd->value_coef;
    const float inv_b = 1.0f / static_cast<float>(h.B);
    const float half_ln_2pi = 0.918938533204672742f;
    for (int i = lane; i < 128; i += 32) {
        g_b[warp][i] = 0.0f;
        g_ls[warp][i] = 0.0f;
    }
    __syncwarp();
    double obj = 0.0, vl = 0.0, cnt = 0.0;
    bool bad = false;
    for (int q = 0; q < PPO_HEAD_SPW; ++q) {   // this warp's samples, in order
        const int b = blockIdx.x * PPO_HEAD_ROWS + warp * PPO_HEAD_SPW + q;
        T* drow = h.delta + static_cast<int64_t>(b) * h.kp64;
        if (b < h.B) {
            const float* mu = h.zh + static_cast<int64_t>(b) * h.n_out_pad;
            const float* raw = h.act + static_cast<int64_t>(b) * h.n;
            float logp = 0.0f;
            for (int i = lane; i < h.n; i += 32) {
                const float z = (raw[i] - mu[i]) * expf(-h.log_std[i]);
                logp += -0.5f * z * z - h.log_std[i] - half_ln_2pi;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) logp += __shfl_xor_sync(0xffffffffu, logp, o);
            const float A = h.adv[b];
            const float rho = expf(logp - h.logp_old[b]);
            const float s1 = rho * A;
            const float s2 = fminf(fmaxf(rho, 1.0f - h_eps), 1.0f + h_eps) * A;
            const bool active = s1 <= s2;
            const double ob = static_cast<double>(active ? s1 : s2);
            const float coef = active ? -A * rho * inv_b : 0.0f;   // dL/dlogp of this sample
            const float V = mu[h.n];
            const float R = h.ret[b];
            const double vb = static_cast<double>(V - R) * static_cast<double>(V - R);
            bad |= !isfinite(ob) || !isfinite(vb);
            obj += ob;
            vl += vb;
            cnt += 1.0;
            for (int i = lane; i < h.kp64; i += 32) {
                float di = 0.0f, gl = 0.0f;
                if (i < h.n) {
                    const float isig = expf(-h.log_std[i]);
                    const float z = (raw[i] - mu[i]) * isig;
                    di = coef * z * isig;   // dlogp/dmu_i = z_i / sigma_i
                    gl = coef * (z * z - 1.0f);
                } else if (i == h.n) {
                    di = 2.0f * h_c_v * (V - R) * inv_b;
                }
                if (i < h.n_out_pad) {
                    g_b[warp][i] += di;
                    g_ls[warp][i] += gl;
                    h.delta_t[static_cast<int64_t>(i) * h.B_pad + b] = from_f32<T>(di);
                }
                drow[i] = from_f32<T>(di);
            }
        } else {
            for (int i = lane; i < h.kp64; i += 32) {
                if (i < h.n_out_pad) h.delta_t[static_cast<int64_t>(i) * h.B_pad + b] = from_f32<T>(0.0f);
                drow[i] = from_f32<T>(0.0f);
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&h.hpd->err, 1u);
    if (lane == 0) {
        red[0][warp] = obj;
        red[1][warp] = vl;
        red[2][warp] = cnt;
    }
    __syncthreads();
    // the block's partial gradients, warps summed in order
    for (int i = threadIdx.x; i < h.n_out_pad; i += blockDim.x) {
        float sb = 0.0f, sl = 0.0f;
#pragma unroll
        for (int w = 0; w < PPO_HEAD_WARPS; ++w) {
            sb += g_b[w][i];
            sl += g_ls[w][i];
        }
        h.bpart[static_cast<int64_t>(blockIdx.x) * h.n_out_pad + i] = sb;
        h.lspart[static_cast<int64_t>(blockIdx.x) * h.n_out_pad + i] = sl;
    }
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1v = 0.0, s2 = 0.0;
        for (int k = 0; k < PPO_HEAD_WARPS; ++k) {
            s0 += red[0][k];
            s1v += red[1][k];
            s2 += red[2][k];
        }
        atomicAdd(&h.losses[0], s0);
        atomicAdd(&h.losses[1], s1v);
        atomicAdd(&h.losses[3], s2);
        if (blockIdx.x == 0) {   // entropy of the state-independent Gaussian: sum_i (log sigma_i + (1 + ln 2 pi)/2)
            double ent = 0.0;
            for (int i = 0; i < h.n; ++i) ent += static_cast<double>(h.log_std[i]) + 1.4189385332046727418;
            atomicAdd(&h.losses[2], ent);
        }
    }
}

// the bias and log-std gradients are reduced from their partials (one per 32 rows) inside the Adam kernel,
// in a fixed order (deterministic)
struct PpoBiasReduce {
    int32_t n_layers, n, n_out_pad;
    int32_t nparts[POD_MAX_HIDDEN_LAYERS + 1];     // partials of layer l (B_pad / 128; the head: B_pad / 32)
    int32_t rows[POD_MAX_HIDDEN_LAYERS + 1];       // bias length of layer l
    const float* part[POD_MAX_HIDDEN_LAYERS + 1];  // [nparts][rows]
    const float* lspart;                           // [nparts][n_out_pad]
};

// W_l^T [in][ld] (T) from the float32 master W_l [out][in]; columns out..ld zero.  32 x 32 tiles;
// blockIdx.z = the layer (all layers l >= 1 in one launch)
template <class T>
struct PpoWt {
    int32_t n;                                       // layers in the launch
    const float* w[POD_MAX_HIDDEN_LAYERS + 1];
    T* wt[POD_MAX_HIDDEN_LAYERS + 1];
    int32_t out[POD_MAX_HIDDEN_LAYERS + 1], in[POD_MAX_HIDDEN_LAYERS + 1], ld[POD_MAX_HIDDEN_LAYERS + 1];
};
template <class T>
__global__ void ppo_wt_kernel(const PpoWt<T> a) {
    __shared__ float tile[32][33];
    const int z = blockIdx.z;
    const int out = a.out[z], in = a.in[z], ld = a.ld[z];
    const int o0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
    if (o0 >= ld || i0 >= in) return;
    const float* w = a.w[z];
    T* wt = a.wt[z];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int o = o0 + k, i = i0 + tx;
        tile[k][tx] = (o < out && i < in) ? w[static_cast<int64_t>(o) * in + i] : 0.0f;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int i = i0 + k, o = o0 + tx;
        if (i < in && o < ld) wt[static_cast<int64_t>(i) * ld + o] = from_f32<T>(o < out ? tile[tx][k] : 0.0f);
    }
}

__global__ void ppo_set_step_kernel(PpoDev* __restrict__ d, int64_t adam_t, float ratio_clip, float entropy_coef,
                                    float value_coef, float lr, float b1, float b2, float eps) {
    d->step_base = adam_t;
    d->ratio_clip = ratio_clip;
    d->entropy_coef = entropy_coef;
    d->value_coef = value_coef;
    d->lr = lr;
    d->b1 = b1;
    d->b2 = b2;
    d->eps = eps;
    d->err = 0u;
}

// Adam step on the float32 master (fa.work) fused with the narrowing of the result into the rollout slab
// (bf16 RNE weights, f32 biases / log-std: the fusion's segment table with K = 1); 8 consecutive elements
// per thread (segments are multiples of 8).  A minibatch whose loss was not finite (hpd->err) leaves the
// master, the moments and the slab untouched: the caller learns of it from pod_ppo_check / the next call.
__global__ void ppo_adam_narrow_kernel(const __grid_constant__ FuseArgs fa, const __grid_constant__ PpoBiasReduce br,
                                       float* __restrict__ m, float* __restrict__ v, float* __restrict__ g,
                                       const PpoDev* __restrict__ d, int j) {
    if (d->err) return;
    const float lr = d->lr, b1 = d->b1, b2 = d->b2, eps = d->eps;
    __shared__ float c12[2];   // the bias corrections 1 - beta^t, once per block (float64 pow)
    if (threadIdx.x == 0) {
        const double step = static_cast<double>(d->step_base + j + 1);
        c12[0] = static_cast<float>(1.0 - pow(static_cast<double>(b1), step));
        c12[1] = static_cast<float>(1.0 - pow(static_cast<double>(b2), step));
    }
    __syncthreads();
    const float c1 = c12[0], c2 = c12[1];
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n8 = fa.n_elems / 8;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n8; q += stride) {
        int64_t o;
        const int si = fuse_find(fa, 8 * q, &o);
        const FuseSeg& sg = fa.seg[si];
        float th[8], mi[8], vi[8], gi[8];
        float4* t4 = reinterpret_cast<float4*>(fa.work + 8 * q);
        float4* m4 = reinterpret_cast<float4*>(m + 8 * q);
        float4* v4 = reinterpret_cast<float4*>(v + 8 * q);
        float4* g4 = reinterpret_cast<float4*>(g + 8 * q);
        if (si >= br.n_layers) {
            // a bias (segment n_layers + l) or the log-std (2 n_layers): the sum of the partials, in order
            const int l = si - br.n_layers;
            const bool ls = l >= br.n_layers;
            const float* src = ls ? br.lspart : br.part[l];
            const int rows = ls ? br.n_out_pad : br.rows[l];
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            const int np = br.nparts[ls ? br.n_layers - 1 : l];
            for (int p = 0; p < np; ++p) {
                const float4* r4 = reinterpret_cast<const float4*>(src + static_cast<int64_t>(p) * rows + o);
                const float4 a0 = r4[0], a1 = r4[1];
                acc[0] += a0.x; acc[1] += a0.y; acc[2] += a0.z; acc[3] += a0.w;
                acc[4] += a1.x; acc[5] += a1.y; acc[6] += a1.z; acc[7] += a1.w;
            }
            if (ls)   // the entropy term: d(-c_ent H)/dlog sigma_i = -c_ent for the n real tickers
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] = o + k < br.n ? acc[k] - d->entropy_coef : 0.0f;
            g4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);   // (grad_out diagnostics read it)
            g4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 a = t4[h], b = m4[h], c = v4[h], e = g4[h];
            th[4 * h] = a.x; th[4 * h + 1] = a.y; th[4 * h + 2] = a.z; th[4 * h + 3] = a.w;
            mi[4 * h] = b.x; mi[4 * h + 1] = b.y; mi[4 * h + 2] = b.z; mi[4 * h + 3] = b.w;
            vi[4 * h] = c.x; vi[4 * h + 1] = c.y; vi[4 * h + 2] = c.z; vi[4 * h + 3] = c.w;
            gi[4 * h] = e.x; gi[4 * h + 1] = e.y; gi[4 * h + 2] = e.z; gi[4 * h + 3] = e.w;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            mi[k] = b1 * mi[k] + (1.0f - b1) * gi[k];
            vi[k] = b2 * vi[k] + (1.0f - b2) * gi[k] * gi[k];
            th[k] -= lr * (mi[k] / c1) / (sqrtf(vi[k] / c2) + eps);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            t4[h] = make_float4(th[4 * h], th[4 * h + 1], th[4 * h + 2], th[4 * h + 3]);
            m4[h] = make_float4(mi[4 * h], mi[4 * h + 1], mi[4 * h + 2], mi[4 * h + 3]);
            v4[h] = make_float4(vi[4 * h], vi[4 * h + 1], vi[4 * h + 2], vi[4 * h + 3]);
        }
        fuse_store8(fa.params, sg, o, th);
    }
}

}  // namespace pod
