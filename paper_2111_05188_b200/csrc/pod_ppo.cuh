// pod_ppo.cuh — host side of pod_ppo_update (included by pod_api.cu; kernels in ppo_kernel.cuh).
// Forward/backward GEMMs are bf16 x bf16 -> float32 library GEMMs (cuBLAS tensor cores, column-major view
// of the row-major [rows][cols] matrices); every other step runs in this library's kernels.  The whole
// minibatch loop (19 launches per minibatch) is captured once into a CUDA graph per buffer set and
// replayed; the Adam step counter and the hyper-parameters (schedules: learning rate, clip, entropy
// coefficient) are written to device memory by one small kernel per call and read from there.
#pragma once
#include <cublas_v2.h>

#include "ppo_kernel.cuh"

namespace pod {

constexpr size_t kPpoCublasWs = 32u << 20;
constexpr size_t kPpoGraphCache = 16;   // captured minibatch loops kept per thread (e.g. one per pod learner)

struct PpoWs {
    size_t x0, h, zf, zh, d0, b0, b1, act, lpo, adv, ret, grad, step, cublas, total;
};

inline PpoWs ppo_ws_layout(const pod_actor_layout& L, int n_hidden, int hidden, int B, int n) {
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    PpoWs w{};
    size_t o = 0;
    const size_t dmax = static_cast<size_t>(B) * (hidden > L.n_out_pad ? hidden : L.n_out_pad);
    w.x0 = o;  o += up(2 * static_cast<size_t>(B) * L.k_pad);                       // bf16 minibatch obs
    w.h = o;   o += up(2 * static_cast<size_t>(B) * hidden * n_hidden);             // bf16 activations
    w.zf = o;  o += up(sizeof(float) * static_cast<size_t>(B) * hidden);            // f32 GEMM output
    w.zh = o;  o += up(sizeof(float) * static_cast<size_t>(B) * L.n_out_pad);       // f32 head output
    w.d0 = o;  o += up(sizeof(float) * dmax);                                       // f32 dX GEMM output
    w.b0 = o;  o += up(2 * dmax);                                                   // their bf16 copies
    w.b1 = o;  o += up(2 * dmax);
    w.act = o; o += up(sizeof(float) * static_cast<size_t>(B) * n);
    w.lpo = o; o += up(sizeof(float) * B);
    w.adv = o; o += up(sizeof(float) * B);
    w.ret = o; o += up(sizeof(float) * B);
    w.grad = o; o += up(sizeof(float) * L.n_elems);
    w.step = o; o += 256;                                                            // int64 Adam step base
    w.cublas = o; o += kPpoCublasWs;                     // this call's cuBLAS workspace (concurrent learners)
    w.total = o;
    return w;
}

// one cuBLAS handle per thread and device; each call points it at the workspace inside its own `ws`
// (no allocation under graph capture, and learners replayed concurrently on different streams do not
// share cuBLAS scratch)
inline cublasHandle_t ppo_cublas() {
    static thread_local cublasHandle_t h = nullptr;
    static thread_local int dev = -1;
    int d = 0;
    cudaGetDevice(&d);
    if (!h || d != dev) {
        if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
        dev = d;
    }
    return h;
}

// captured minibatch loops, keyed on every pointer and size (not adam_t, the hyper-parameters or the stream)
struct PpoGraphKey {
    const void* p[16];
    int64_t M, k_pad, n_elems;
    int32_t cfg_n, n_hidden, hidden, act, batch, n_mb, dev;
    size_t param_bytes, ws_bytes;
    bool operator==(const PpoGraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};
struct PpoGraph {
    PpoGraphKey key;
    cudaGraphExec_t exec;
    uint64_t used;
};
inline std::vector<PpoGraph>& ppo_graphs() {
    static thread_local std::vector<PpoGraph> g;
    return g;
}
inline cudaStream_t ppo_cap_stream() {
    static thread_local cudaStream_t cs = nullptr;
    static thread_local int dev = -1;
    int d = 0;
    cudaGetDevice(&d);
    if (!cs || d != dev) {
        if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        dev = d;
    }
    return cs;
}

}  // namespace pod

extern "C" pod_status pod_ppo_workspace_size(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                                             int32_t batch, size_t* bytes) {
    if (!bytes) return pod_fail(POD_ERR_ARG, "bytes is NULL");
    if (batch < 1) return pod_fail(POD_ERR_ARG, "batch must be >= 1");
    pod_actor_layout L;
    pod_status st = pod_actor_layout_get(cfg, n_hidden, hidden, &L);
    if (st) return st;
    *bytes = pod::ppo_ws_layout(L, n_hidden, hidden, batch, cfg->n_stocks).total;
    return POD_OK;
}

#define POD_CUBLAS(call)                                                                      \
    do {                                                                                      \
        cublasStatus_t _s = (call);                                                           \
        if (_s != CUBLAS_STATUS_SUCCESS) return pod_fail(POD_ERR_CUDA, "%s: cuBLAS status %d", #call, static_cast<int>(_s)); \
    } while (0)

extern "C" pod_status pod_ppo_update(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden, int32_t act,
                                     const pod_ppo_hparams* hp, float* master, float* adam_m, float* adam_v,
                                     int64_t adam_t, void* params, size_t param_bytes, const uint16_t* obs,
                                     const float* act_raw, const float* logp_old, const float* adv, const float* ret,
                                     int64_t M, const int32_t* perm, int32_t batch, int32_t n_minibatches,
                                     double* losses, float* grad_out, void* ws, size_t ws_bytes, void* stream) {
    using namespace pod;
    if (!hp || !master || !adam_m || !adam_v || !params || !obs || !act_raw || !logp_old || !adv || !ret ||
        (!perm && n_minibatches > 0) || !losses || !ws)
        return pod_fail(POD_ERR_ARG, "NULL argument");
    if (act != 0 && act != 1) return pod_fail(POD_ERR_ARG, "act must be 0 (ReLU) or 1 (tanh)");
    if (batch < 1 || n_minibatches < 0 || M < 1 || adam_t < 0) return pod_fail(POD_ERR_ARG, "bad batch / M / adam_t");
    if (!(hp->ratio_clip > 0.0f && hp->ratio_clip < 1.0f) || !(hp->learning_rate > 0.0f) || hp->entropy_coef < 0.0f ||
        hp->value_coef < 0.0f || !(hp->adam_beta1 >= 0.0f && hp->adam_beta1 < 1.0f) ||
        !(hp->adam_beta2 >= 0.0f && hp->adam_beta2 < 1.0f) || !(hp->adam_eps > 0.0f))
        return pod_fail(POD_ERR_ARG, "hyper-parameters out of range (0 < ratio_clip < 1, lr > 0, betas in [0,1))");
    pod_actor_layout L;
    pod_status st = pod_actor_layout_get(cfg, n_hidden, hidden, &L);
    if (st) return st;
    if (param_bytes < L.param_bytes || param_bytes % 16 != 0)
        return pod_fail(POD_ERR_SHAPE, "param_bytes %zu must be >= %zu and a multiple of 16", param_bytes, L.param_bytes);
    const int n = cfg->n_stocks;
    const PpoWs W = ppo_ws_layout(L, n_hidden, hidden, batch, n);
    if (ws_bytes < W.total) return pod_fail(POD_ERR_ARG, "workspace needs %zu bytes", W.total);
    if (reinterpret_cast<uintptr_t>(ws) % 256 != 0 || reinterpret_cast<uintptr_t>(master) % 16 != 0 ||
        reinterpret_cast<uintptr_t>(adam_m) % 16 != 0 || reinterpret_cast<uintptr_t>(adam_v) % 16 != 0 ||
        reinterpret_cast<uintptr_t>(params) % 16 != 0)
        return pod_fail(POD_ERR_ARG, "ws must be 256-byte aligned, master, adam_m, adam_v and params 16-byte aligned");
    st = pod_require_sm100();
    if (st) return st;
    cudaStream_t user_s = static_cast<cudaStream_t>(stream);
    cublasHandle_t cb = ppo_cublas();
    if (!cb) return pod_fail(POD_ERR_CUDA, "cublasCreate failed");
    char* w = static_cast<char*>(ws);
    PpoDev* hpd = reinterpret_cast<PpoDev*>(w + W.step);   // step base + hyper-parameters of this call
    __nv_bfloat16* x0 = reinterpret_cast<__nv_bfloat16*>(w + W.x0);
    __nv_bfloat16* hbuf = reinterpret_cast<__nv_bfloat16*>(w + W.h);
    float* zf = reinterpret_cast<float*>(w + W.zf);
    float* zh = reinterpret_cast<float*>(w + W.zh);
    float* d0 = reinterpret_cast<float*>(w + W.d0);
    __nv_bfloat16* b0 = reinterpret_cast<__nv_bfloat16*>(w + W.b0);
    __nv_bfloat16* b1 = reinterpret_cast<__nv_bfloat16*>(w + W.b1);
    float* act_b = reinterpret_cast<float*>(w + W.act);
    float* lpo_b = reinterpret_cast<float*>(w + W.lpo);
    float* adv_b = reinterpret_cast<float*>(w + W.adv);
    float* ret_b = reinterpret_cast<float*>(w + W.ret);
    float* grad = reinterpret_cast<float*>(w + W.grad);
    const __nv_bfloat16* wslab[POD_MAX_HIDDEN_LAYERS + 1];
    for (int l = 0; l < L.n_layers; ++l)
        wslab[l] = reinterpret_cast<const __nv_bfloat16*>(static_cast<const char*>(params) + L.w_offset[l]);
    // flat offsets (elements) of W_l, b_l, log_std: pod_fuse_pods order
    int64_t woff[POD_MAX_HIDDEN_LAYERS + 1], boff[POD_MAX_HIDDEN_LAYERS + 1];
    int64_t f = 0;
    for (int l = 0; l < L.n_layers; ++l) {
        woff[l] = f;
        f += static_cast<int64_t>(L.w_rows[l]) * L.w_cols[l];
    }
    for (int l = 0; l < L.n_layers; ++l) {
        boff[l] = f;
        f += L.w_rows[l];
    }
    const int64_t lsoff = f;
    // slab refresh from the master copy after every Adam step (the GEMMs read the bf16 slab): the fusion
    // narrowing with K = 1, tau = 1
    FuseArgs fa{};
    {
        uint64_t fl = 0;
        int ns = 0;
        for (int l = 0; l < L.n_layers; ++l) {
            fa.seg[ns++] = FuseSeg{L.w_offset[l], fl, static_cast<uint32_t>(L.w_rows[l]) * L.w_cols[l], 1u};
            fl += static_cast<uint64_t>(L.w_rows[l]) * L.w_cols[l];
        }
        for (int l = 0; l < L.n_layers; ++l) {
            fa.seg[ns++] = FuseSeg{L.b_offset[l], fl, static_cast<uint32_t>(L.w_rows[l]), 0u};
            fl += static_cast<uint64_t>(L.w_rows[l]);
        }
        fa.seg[ns++] = FuseSeg{L.log_std_offset, fl, static_cast<uint32_t>(L.n_out_pad), 0u};
        fl += static_cast<uint64_t>(L.n_out_pad);
        fa.n_seg = ns;
        fa.K_local = 1;
        fa.n_elems = static_cast<int64_t>(fl);
        fa.param_bytes = param_bytes;
        fa.params = static_cast<char*>(params);
        fa.work = master;
        fa.prev = nullptr;
        fa.scale = 1.0f;
        fa.tau = 1.0f;
    }
    const int64_t g8 = fa.n_elems / 8;
    const dim3 ngrid(static_cast<unsigned>(std::min<int64_t>((g8 + 255) / 256, 8 * 148)), 1);
    const float one = 1.0f, zero = 0.0f;
    const int B = batch;
    const unsigned ag_rows = static_cast<unsigned>((B + PPO_AG_ROWS - 1) / PPO_AG_ROWS);   // <= 2^31 / 16
    // the minibatch loop, enqueued on stream s (captured below, or eager with POD_PPO_GRAPH=0)
    auto enqueue = [&](cudaStream_t s) -> pod_status {
    POD_CUBLAS(cublasSetStream(cb, s));
    POD_CUBLAS(cublasSetWorkspace(cb, w + W.cublas, kPpoCublasWs));
    // the gradient vector is cleared once here, then by each minibatch's Adam step for the next
    POD_CUDA(cudaMemsetAsync(grad, 0, sizeof(float) * L.n_elems, s));
    for (int j = 0; j < n_minibatches; ++j) {
        ppo_gather_kernel<<<B, 128, 0, s>>>(obs, act_raw, logp_old, adv, ret, perm + static_cast<int64_t>(j) * B, B,
                                            L.k_pad, n, reinterpret_cast<uint16_t*>(x0), act_b, lpo_b, adv_b, ret_b);
        // forward: X_{l+1} = act(X_l W_l^T + b_l) (bf16 x bf16 -> f32 GEMM, bias + activation -> bf16)
        const __nv_bfloat16* xin = x0;
        for (int l = 0; l < L.n_layers; ++l) {
            const int rows = L.w_rows[l], cols = L.w_cols[l];
            const bool head = l == L.n_layers - 1;
            float* out = head ? zh : zf;
            POD_CUBLAS(cublasGemmEx(cb, CUBLAS_OP_T, CUBLAS_OP_N, rows, B, cols, &one, wslab[l], CUDA_R_16BF, cols, xin,
                                    CUDA_R_16BF, cols, &zero, out, CUDA_R_32F, rows, CUBLAS_COMPUTE_32F,
                                    CUBLAS_GEMM_DEFAULT));
            __nv_bfloat16* hout = head ? nullptr : hbuf + static_cast<int64_t>(l) * B * hidden;
            ppo_bias_act_kernel<<<dim3((rows / 4 + 127) / 128, std::min(B, 65535)), 128, 0, s>>>(out, master + boff[l], B, rows,
                                                                                head ? -1 : act, hout);
            xin = hout;
        }
        // head loss and dL/d(head output) -> b0 [B][n_out_pad] (bf16) and the head bias gradient; gradient
        // vector cleared first
        PpoHead hh{B, n, L.n_out_pad, hpd, act_b, lpo_b, adv_b, ret_b,
                   zh, master + lsoff, b0, grad + boff[L.n_layers - 1], grad + lsoff, losses};
        ppo_head_kernel<<<(B + PPO_HEAD_WARPS - 1) / PPO_HEAD_WARPS, 32 * PPO_HEAD_WARPS, 0, s>>>(hh);
        // backward: dW_l = delta_l^T X_l, delta_{l-1} = (delta_l W_l) * act'(X_l) with db_{l-1} = colsum
        // (delta_{l-1}) fused into the activation-derivative kernel
        __nv_bfloat16* bcur = b0;
        __nv_bfloat16* bnext = b1;
        for (int l = L.n_layers - 1; l >= 0; --l) {
            const int rows = L.w_rows[l], cols = L.w_cols[l];
            const __nv_bfloat16* xl = l == 0 ? x0 : hbuf + static_cast<int64_t>(l - 1) * B * hidden;
            POD_CUBLAS(cublasGemmEx(cb, CUBLAS_OP_N, CUBLAS_OP_T, cols, rows, B, &one, xl, CUDA_R_16BF, cols, bcur,
                                    CUDA_R_16BF, rows, &zero, grad + woff[l], CUDA_R_32F, cols, CUBLAS_COMPUTE_32F,
                                    CUBLAS_GEMM_DEFAULT));
            if (l > 0) {
                POD_CUBLAS(cublasGemmEx(cb, CUBLAS_OP_N, CUBLAS_OP_N, cols, B, rows, &one, wslab[l], CUDA_R_16BF, cols,
                                        bcur, CUDA_R_16BF, rows, &zero, d0, CUDA_R_32F, cols, CUBLAS_COMPUTE_32F,
                                        CUBLAS_GEMM_DEFAULT));
                ppo_act_grad_kernel<<<dim3((cols / 2 + 127) / 128, ag_rows), 128, 0, s>>>(
                    d0, xl, B, cols, act, bnext, grad + boff[l - 1]);
                __nv_bfloat16* tb = bcur;
                bcur = bnext;
                bnext = tb;
            }
        }
        if (grad_out && j == n_minibatches - 1)
            POD_CUDA(cudaMemcpyAsync(grad_out, grad, sizeof(float) * L.n_elems, cudaMemcpyDeviceToDevice, s));
        // Adam on the master, narrowed into the slab, gradient cleared for the next minibatch
        ppo_adam_narrow_kernel<<<ngrid, 256, 0, s>>>(fa, adam_m, adam_v, grad, hpd, j);
        POD_CUDA(cudaGetLastError());
    }
    if (n_minibatches == 0) {
        fuse_blend_kernel<<<ngrid, 256, 0, s>>>(fa);
        POD_CUDA(cudaGetLastError());
    }
    return POD_OK;
    };
    ppo_set_step_kernel<<<1, 1, 0, user_s>>>(hpd, adam_t, hp->ratio_clip, hp->entropy_coef, hp->value_coef,
                                             hp->learning_rate, hp->adam_beta1, hp->adam_beta2, hp->adam_eps);
    POD_CUDA(cudaGetLastError());
    static const bool use_graph = [] {
        const char* e = std::getenv("POD_PPO_GRAPH");
        return !(e && e[0] == '0');
    }();
    if (!use_graph) return enqueue(user_s);
    PpoGraphKey key;
    std::memset(&key, 0, sizeof(key));
    const void* kp[16] = {master, adam_m, adam_v, params, obs, act_raw, logp_old, adv, ret, perm, losses, grad_out, ws,
                          nullptr, nullptr, nullptr};
    std::memcpy(key.p, kp, sizeof(kp));
    key.M = M;
    key.k_pad = L.k_pad;
    key.n_elems = static_cast<int64_t>(L.n_elems);
    key.cfg_n = n;
    key.n_hidden = n_hidden;
    key.hidden = hidden;
    key.act = act;
    key.batch = batch;
    key.n_mb = n_minibatches;
    cudaGetDevice(&key.dev);
    key.param_bytes = param_bytes;
    key.ws_bytes = ws_bytes;
    static thread_local uint64_t ppo_clock = 0;
    auto& cache = ppo_graphs();
    PpoGraph* hit = nullptr;
    for (auto& g : cache)
        if (g.key == key) hit = &g;
    if (!hit) {
        cudaStream_t cs = ppo_cap_stream();
        if (!cs) return pod_fail(POD_ERR_CUDA, "capture stream creation failed");
        cudaGraph_t graph;
        POD_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        pod_status est = enqueue(cs);
        cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        if (est) {
            if (ce == cudaSuccess) cudaGraphDestroy(graph);
            return est;
        }
        if (ce != cudaSuccess) return pod_fail(POD_ERR_CUDA, "PPO graph capture: %s", cudaGetErrorString(ce));
        cudaGraphExec_t exec;
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return pod_fail(POD_ERR_CUDA, "PPO graph instantiate: %s", cudaGetErrorString(ce));
        if (cache.size() >= kPpoGraphCache) {   // evict the least recently used
            size_t victim = 0;
            for (size_t i = 1; i < cache.size(); ++i)
                if (cache[i].used < cache[victim].used) victim = i;
            cudaGraphExecDestroy(cache[victim].exec);
            cache.erase(cache.begin() + static_cast<long>(victim));
        }
        cache.push_back(PpoGraph{key, exec, 0});
        hit = &cache.back();
    }
    hit->used = ++ppo_clock;
    POD_CUDA(cudaGraphLaunch(hit->exec, user_s));
    return POD_OK;
}
