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
// The layer GEMMs (forward X W^T, backward delta^T X and delta W) are bf16 x bf16 -> float32 tensor-core
// GEMMs (cuBLAS, as the rollout's actor: bf16 weights = the rollout slab, bf16 activations); these
// kernels are the gather, bias + activation, head loss, activation derivative (each writing the float32
// value and its bf16 copy for the next GEMM), bias reduction and the Adam step on the float32 master.
// Activations are kept post-nonlinearity: ReLU' = [h > 0], tanh' = 1 - h^2.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

#include "fuse_kernel.cuh"

namespace pod {

// per-call values in device memory (written by ppo_set_step_kernel before the captured minibatch loop), so
// one graph serves every call of a schedule: the Adam step base and the hyper-parameters
struct PpoDev {
    int64_t step_base;
    float ratio_clip, entropy_coef, value_coef, lr, b1, b2, eps, pad;
};

struct PpoHead {
    int32_t B, n, n_out_pad;
    const PpoDev* hpd;       // ratio clip, entropy and value coefficients
    const float* act;        // [B][n] raw actions of the minibatch
    const float* logp_old;   // [B]
    const float* adv;        // [B]
    const float* ret;        // [B]
    const float* zh;         // [B][n_out_pad] head output (mu in 0..n-1, V in n)
    const float* log_std;    // [n] (master)
    __nv_bfloat16* delta_bf; // [B][n_out_pad] dL/d head output, bf16 (the backward GEMMs' operand)
    float* g_bias;           // [n_out_pad] head bias gradient = column sums of the float32 delta (atomic)
    float* g_log_std;        // [n] accumulated (atomic)
    double* losses;          // [4]
};

// gather the minibatch rows perm[0..B) of the flattened buffer (obs rows stay bf16: the first GEMM's operand)
__global__ void ppo_gather_kernel(const uint16_t* __restrict__ obs, const float* __restrict__ act,
                                  const float* __restrict__ lpo, const float* __restrict__ adv,
                                  const float* __restrict__ ret, const int32_t* __restrict__ perm, int B, int k_pad,
                                  int n, uint16_t* __restrict__ x0, float* __restrict__ act_b, float* __restrict__ lpo_b,
                                  float* __restrict__ adv_b, float* __restrict__ ret_b) {
    const int r = blockIdx.x;
    const int64_t src = perm[r];
    const uint4* s4 = reinterpret_cast<const uint4*>(obs + src * k_pad);
    uint4* d4 = reinterpret_cast<uint4*>(x0 + static_cast<int64_t>(r) * k_pad);
    for (int c = threadIdx.x; c < k_pad / 8; c += blockDim.x) d4[c] = s4[c];   // bf16 rows, 16 B at a time
    for (int c = threadIdx.x; c < n; c += blockDim.x) act_b[static_cast<int64_t>(r) * n + c] = act[src * n + c];
    if (threadIdx.x == 0) {
        lpo_b[r] = lpo[src];
        adv_b[r] = adv[src];
        ret_b[r] = ret[src];
    }
}

// Z[B][N] (from the GEMM) + b, then the activation (act 0 ReLU, 1 tanh, -1 none): into z in place
// (head) or, when h is given, as the bf16 activation of the next layer.  Block = one row (grid-strided
// over rows), thread = 4 consecutive columns (N is a multiple of 32).
__global__ void ppo_bias_act_kernel(float* __restrict__ z, const float* __restrict__ b, int64_t B, int N, int act,
                                    __nv_bfloat16* __restrict__ h) {
    const int c = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (c >= N) return;
    for (int64_t r = blockIdx.y; r < B; r += gridDim.y) {
    const int64_t i = r * N + c;
    float4 v = *reinterpret_cast<const float4*>(z + i);
    const float4 bc = *reinterpret_cast<const float4*>(b + c);
    v.x += bc.x;
    v.y += bc.y;
    v.z += bc.z;
    v.w += bc.w;
    if (act == 0) {
        v.x = fmaxf(v.x, 0.0f);
        v.y = fmaxf(v.y, 0.0f);
        v.z = fmaxf(v.z, 0.0f);
        v.w = fmaxf(v.w, 0.0f);
    } else if (act == 1) {
        v.x = tanhf(v.x);
        v.y = tanhf(v.y);
        v.z = tanhf(v.z);
        v.w = tanhf(v.w);
    }
    if (h) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(h + i) = pk;
    } else {
        *reinterpret_cast<float4*>(z + i) = v;
    }
    }
}

// one warp per sample (lanes over tickers): head loss and dL/d(head output); the log-std gradient and the
// loss sums are reduced per block in shared memory, then one atomic each
// (n_out_pad <= 128, checked at layout time).  Block 0 also adds the entropy term of the log-std gradient,
// -c_ent, and the entropy value sum_i (log sigma_i + (1 + ln 2 pi) / 2).
constexpr int PPO_HEAD_WARPS = 8;
__global__ void __launch_bounds__(32 * PPO_HEAD_WARPS) ppo_head_kernel(const PpoHead h) {
    __shared__ float g_ls[128];
    __shared__ float g_b[128];
    __shared__ double red[4][PPO_HEAD_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        g_ls[i] = 0.0f;
        g_b[i] = 0.0f;
    }
    __syncthreads();
    const int b = blockIdx.x * PPO_HEAD_WARPS + warp;
    const float h_eps = h.hpd->ratio_clip, h_c_ent = h.hpd->entropy_coef, h_c_v = h.hpd->value_coef;
    const float inv_b = 1.0f / static_cast<float>(h.B);
    const float half_ln_2pi = 0.918938533204672742f;
    double obj = 0.0, vl = 0.0;
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
        obj = static_cast<double>(active ? s1 : s2);
        const float coef = active ? -A * rho * inv_b : 0.0f;   // dL/dlogp of this sample
        __nv_bfloat16* dbf = h.delta_bf + static_cast<int64_t>(b) * h.n_out_pad;
        const float V = mu[h.n];
        const float R = h.ret[b];
        for (int i = lane; i < h.n_out_pad; i += 32) {
            float di = 0.0f;
            if (i < h.n) {
                const float isig = expf(-h.log_std[i]);
                const float z = (raw[i] - mu[i]) * isig;
                di = coef * z * isig;                          // dlogp/dmu_i = z_i / sigma_i
                if (coef != 0.0f) atomicAdd(&g_ls[i], coef * (z * z - 1.0f));
            } else if (i == h.n) {
                di = 2.0f * h_c_v * (V - R) * inv_b;
            }
            if (di != 0.0f) atomicAdd(&g_b[i], di);
            dbf[i] = __float2bfloat16_rn(di);
        }
        vl = static_cast<double>(V - R) * static_cast<double>(V - R);
    }
    double ent = 0.0;
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < h.n; i += blockDim.x) {
            atomicAdd(&g_ls[i], -h_c_ent);
            ent += static_cast<double>(h.log_std[i]) + 1.4189385332046727418;   // (1 + ln 2 pi) / 2
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ent += __shfl_xor_sync(0xffffffffu, ent, o);
    if (lane == 0) {
        red[0][warp] = obj;
        red[1][warp] = vl;
        red[2][warp] = b < h.B ? 1.0 : 0.0;
        red[3][warp] = ent;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1v = 0.0, s2 = 0.0, s3 = 0.0;
        for (int k = 0; k < PPO_HEAD_WARPS; ++k) {
            s0 += red[0][k];
            s1v += red[1][k];
            s2 += red[2][k];
            s3 += red[3][k];
        }
        atomicAdd(&h.losses[0], s0);
        atomicAdd(&h.losses[1], s1v);
        atomicAdd(&h.losses[3], s2);
        if (blockIdx.x == 0) atomicAdd(&h.losses[2], s3);
    }
    for (int i = threadIdx.x; i < h.n; i += blockDim.x) atomicAdd(&h.g_log_std[i], g_ls[i]);
    for (int i = threadIdx.x; i < h.n_out_pad; i += blockDim.x)
        if (g_b[i] != 0.0f) atomicAdd(&h.g_bias[i], g_b[i]);
}

// delta = dX * act'(H) (dX the float32 GEMM output, H the layer's bf16 post-activation output), written as
// the bf16 operand of the next GEMMs, with the layer's bias gradient db[c] += sum over the block's rows of
// delta[r][c] fused in (one atomic per column per block).  Block = 128 threads x 2 columns, PPO_AG_ROWS
// rows; N is a multiple of 32.
constexpr int PPO_AG_ROWS = 16;
__global__ void ppo_act_grad_kernel(const float* __restrict__ dx, const __nv_bfloat16* __restrict__ hact, int B, int N,
                                    int act, __nv_bfloat16* __restrict__ dbf, float* __restrict__ db) {
    const int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (c >= N) return;
    const int r0 = blockIdx.y * PPO_AG_ROWS;
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll 8
    for (int k = 0; k < PPO_AG_ROWS; ++k) {
        const int r = r0 + k;
        if (r < B) {
            const int64_t i = static_cast<int64_t>(r) * N + c;
            const float2 g = *reinterpret_cast<const float2*>(dx + i);
            const float2 hv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(hact + i));
            const float d0 = g.x * (act == 0 ? (hv.x > 0.0f ? 1.0f : 0.0f) : (1.0f - hv.x * hv.x));
            const float d1 = g.y * (act == 0 ? (hv.y > 0.0f ? 1.0f : 0.0f) : (1.0f - hv.y * hv.y));
            *reinterpret_cast<__nv_bfloat162*>(dbf + i) = __floats2bfloat162_rn(d0, d1);
            s0 += d0;
            s1 += d1;
        }
    }
    if (s0 != 0.0f) atomicAdd(&db[c], s0);
    if (s1 != 0.0f) atomicAdd(&db[c + 1], s1);
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
}

// Adam step on the float32 master (fa.work) fused with the narrowing of the result into the rollout slab
// (bf16 RNE weights, f32 biases / log-std: the fusion's segment table with K = 1) and the clearing of the
// gradient for the next minibatch; 8 consecutive elements per thread (segments are multiples of 8).
__global__ void ppo_adam_narrow_kernel(const __grid_constant__ FuseArgs fa, float* __restrict__ m,
                                       float* __restrict__ v, float* __restrict__ g, const PpoDev* __restrict__ d,
                                       int j) {
    const float lr = d->lr, b1 = d->b1, b2 = d->b2, eps = d->eps;
    const double step = static_cast<double>(d->step_base + j + 1);
    const float c1 = static_cast<float>(1.0 - pow(static_cast<double>(b1), step));
    const float c2 = static_cast<float>(1.0 - pow(static_cast<double>(b2), step));
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n8 = fa.n_elems / 8;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n8; q += stride) {
        int64_t o;
        const FuseSeg& sg = fa.seg[fuse_find(fa, 8 * q, &o)];
        float th[8], mi[8], vi[8], gi[8];
        float4* t4 = reinterpret_cast<float4*>(fa.work + 8 * q);
        float4* m4 = reinterpret_cast<float4*>(m + 8 * q);
        float4* v4 = reinterpret_cast<float4*>(v + 8 * q);
        float4* g4 = reinterpret_cast<float4*>(g + 8 * q);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 a = t4[h], b = m4[h], c = v4[h], d = g4[h];
            th[4 * h] = a.x; th[4 * h + 1] = a.y; th[4 * h + 2] = a.z; th[4 * h + 3] = a.w;
            mi[4 * h] = b.x; mi[4 * h + 1] = b.y; mi[4 * h + 2] = b.z; mi[4 * h + 3] = b.w;
            vi[4 * h] = c.x; vi[4 * h + 1] = c.y; vi[4 * h + 2] = c.z; vi[4 * h + 3] = c.w;
            gi[4 * h] = d.x; gi[4 * h + 1] = d.y; gi[4 * h + 2] = d.z; gi[4 * h + 3] = d.w;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            mi[k] = b1 * mi[k] + (1.0f - b1) * gi[k];
            vi[k] = b2 * vi[k] + (1.0f - b2) * gi[k] * gi[k];
            th[k] -= lr * (mi[k] / c1) / (sqrtf(vi[k] / c2) + eps);
        }
        const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            t4[h] = make_float4(th[4 * h], th[4 * h + 1], th[4 * h + 2], th[4 * h + 3]);
            m4[h] = make_float4(mi[4 * h], mi[4 * h + 1], mi[4 * h + 2], mi[4 * h + 3]);
            v4[h] = make_float4(vi[4 * h], vi[4 * h + 1], vi[4 * h + 2], vi[4 * h + 3]);
            g4[h] = zero;
        }
        fuse_store8(fa.params, sg, o, th);
    }
}

}  // namespace pod
