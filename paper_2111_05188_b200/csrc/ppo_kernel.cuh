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

namespace pod {

struct PpoHead {
    int32_t B, n, n_out_pad;
    float eps, c_ent, c_v;
    const float* act;        // [B][n] raw actions of the minibatch
    const float* logp_old;   // [B]
    const float* adv;        // [B]
    const float* ret;        // [B]
    const float* zh;         // [B][n_out_pad] head output (mu in 0..n-1, V in n)
    const float* log_std;    // [n] (master)
    float* delta;            // [B][n_out_pad] dL/d head output
    __nv_bfloat16* delta_bf; // [B][n_out_pad] its bf16 copy (GEMM operand)
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
// (head) or, when h is given, as the bf16 activation of the next layer
__global__ void ppo_bias_act_kernel(float* __restrict__ z, const float* __restrict__ b, int64_t B, int N, int act,
                                    __nv_bfloat16* __restrict__ h) {
    const int64_t total = B * N;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        float v = z[i] + b[i % N];
        if (act == 0) v = fmaxf(v, 0.0f);
        else if (act == 1) v = tanhf(v);
        if (h) h[i] = __float2bfloat16_rn(v);
        else z[i] = v;
    }
}

// one thread per sample: head loss and dL/d(head output); log-std gradient and loss sums reduced per block
__global__ void __launch_bounds__(128) ppo_head_kernel(const PpoHead h) {
    __shared__ float g_ls[128];
    __shared__ double red[3][128];
    for (int i = threadIdx.x; i < h.n && i < 128; i += blockDim.x) g_ls[i] = 0.0f;
    __syncthreads();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const float inv_b = 1.0f / static_cast<float>(h.B);
    const float half_ln_2pi = 0.918938533204672742f;
    double obj = 0.0, vl = 0.0;
    if (b < h.B) {
        const float* mu = h.zh + static_cast<int64_t>(b) * h.n_out_pad;
        const float* raw = h.act + static_cast<int64_t>(b) * h.n;
        float logp = 0.0f;
        for (int i = 0; i < h.n; ++i) {
            const float z = (raw[i] - mu[i]) * expf(-h.log_std[i]);
            logp += -0.5f * z * z - h.log_std[i] - half_ln_2pi;
        }
        const float A = h.adv[b];
        const float rho = expf(logp - h.logp_old[b]);
        const float s1 = rho * A;
        const float s2 = fminf(fmaxf(rho, 1.0f - h.eps), 1.0f + h.eps) * A;
        const bool active = s1 <= s2;
        obj = static_cast<double>(active ? s1 : s2);
        const float coef = active ? -A * rho * inv_b : 0.0f;   // dL/dlogp of this sample
        float* d = h.delta + static_cast<int64_t>(b) * h.n_out_pad;
        for (int i = 0; i < h.n; ++i) {
            const float isig = expf(-h.log_std[i]);
            const float z = (raw[i] - mu[i]) * isig;
            d[i] = coef * z * isig;                            // dlogp/dmu_i = z_i / sigma_i
            h.delta_bf[static_cast<int64_t>(b) * h.n_out_pad + i] = __float2bfloat16_rn(d[i]);
            if (coef != 0.0f) atomicAdd(&g_ls[i], coef * (z * z - 1.0f));
        }
        const float V = mu[h.n];
        const float R = h.ret[b];
        d[h.n] = 2.0f * h.c_v * (V - R) * inv_b;
        h.delta_bf[static_cast<int64_t>(b) * h.n_out_pad + h.n] = __float2bfloat16_rn(d[h.n]);
        for (int i = h.n + 1; i < h.n_out_pad; ++i) {
            d[i] = 0.0f;
            h.delta_bf[static_cast<int64_t>(b) * h.n_out_pad + i] = __float2bfloat16_rn(0.0f);
        }
        vl = static_cast<double>(V - R) * static_cast<double>(V - R);
    }
    red[0][threadIdx.x] = obj;
    red[1][threadIdx.x] = vl;
    red[2][threadIdx.x] = b < h.B ? 1.0 : 0.0;
    __syncthreads();
    for (int o = 64; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        atomicAdd(&h.losses[0], red[0][0]);
        atomicAdd(&h.losses[1], red[1][0]);
        atomicAdd(&h.losses[3], red[2][0]);
    }
    for (int i = threadIdx.x; i < h.n && i < 128; i += blockDim.x) atomicAdd(&h.g_log_std[i], g_ls[i]);
}

// entropy term of the log-std gradient (once per minibatch) and the entropy value
__global__ void ppo_entropy_kernel(const float* __restrict__ log_std, int n, float c_ent, float* __restrict__ g_log_std,
                                   double* __restrict__ losses) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        g_log_std[i] += -c_ent;
        s += static_cast<double>(log_std[i]) + 1.4189385332046727418;   // (1 + ln 2 pi) / 2
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&losses[2], s);
}

// delta = dX * act'(H) in place on dX (H the layer's bf16 post-activation output), plus its bf16 copy
__global__ void ppo_act_grad_kernel(float* __restrict__ dx, const __nv_bfloat16* __restrict__ hact, int64_t total,
                                    int act, __nv_bfloat16* __restrict__ dbf) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const float h = __bfloat162float(hact[i]);
        const float d = dx[i] * (act == 0 ? (h > 0.0f ? 1.0f : 0.0f) : (1.0f - h * h));
        dx[i] = d;
        dbf[i] = __float2bfloat16_rn(d);
    }
}

// db[N] = sum over the B rows of delta[B][N] (thread per column, coalesced rows)
__global__ void ppo_colsum_kernel(const float* __restrict__ delta, int B, int N, float* __restrict__ db) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    float s = 0.0f;
    for (int r = 0; r < B; ++r) s += delta[static_cast<int64_t>(r) * N + c];
    db[c] = s;
}

// Adam (bias-corrected) over the flat parameter vector
__global__ void ppo_adam_kernel(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ v,
                                const float* __restrict__ g, int64_t count, float lr, float b1, float b2, float eps,
                                float c1, float c2) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float gi = g[i];
        const float mi = b1 * m[i] + (1.0f - b1) * gi;
        const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        theta[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    }
}

}  // namespace pod
