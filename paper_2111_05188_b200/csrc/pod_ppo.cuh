// pod_ppo.cuh — host side of pod_ppo_update (included by pod_api.cu; kernels in ppo_kernel.cuh and
// gemm_kernel.cuh).  Per minibatch of B rows (B_pad = B rounded up to the 128-row tile; padded rows are
// zeros and contribute nothing):
//   gather (X0, X0^T) -> forward products l = 0..L (epilogues: bias + activation into X_{l+1}, X_{l+1}^T;
//   the head's f32 output) -> head loss (delta_L, delta_L^T, bias / log-std partials) -> for l = L..0 the
//   weight-gradient product into the flat gradient and, for l > 0, the input-gradient product (epilogue:
//   activation derivative, delta_{l-1}, delta_{l-1}^T, bias partials) -> fixed-order bias reduction ->
//   Adam on the float32 master, narrowed into the rollout slab -> W_l^T for the next minibatch.
// The products run on this library's tcgen05 kernel (bf16 operands: the rollout slab's weights and bf16
// activations / deltas, f32 accumulate) or, with hp->fp32_operands, on its float32 reference core (the
// master weights and float32 activations / deltas) — same launches, layouts and epilogues.  The whole
// minibatch loop (14 launches per minibatch; the weight-gradient products on a parallel branch) is captured once into a CUDA graph per buffer set and
// replayed; the Adam step counter and the hyper-parameters (schedules: learning rate, clip, entropy
// coefficient) are written to device memory by one small kernel per call and read from there.
#pragma once
#include "ppo_kernel.cuh"

namespace pod {

constexpr size_t kPpoGraphCache = 16;   // captured minibatch loops kept per thread (e.g. one per pod learner)
constexpr int PPO_BN = 32;              // output columns per GEMM tile (more CTAs for these small products)

struct PpoWs {
    int B_pad, kp64, dmax;
    size_t x0, x0t, h[POD_MAX_HIDDEN_LAYERS + 1], ht[POD_MAX_HIDDEN_LAYERS + 1], zh, d[3], dt[3],
        wt[POD_MAX_HIDDEN_LAYERS + 1], bpart[POD_MAX_HIDDEN_LAYERS + 1], lspart, act, lpo, adv, ret, grad, hpd, total;
};

inline PpoWs ppo_ws_layout(const pod_actor_layout& L, int n_hidden, int hidden, int B, int n) {
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    PpoWs w{};
    w.B_pad = (B + 127) / 128 * 128;
    w.kp64 = (L.n_out_pad + 63) / 64 * 64;
    w.dmax = hidden > w.kp64 ? hidden : w.kp64;
    const size_t Bp = static_cast<size_t>(w.B_pad), E = 4;   // element bytes: float32 covers both modes
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t r = o;
        o += up(bytes);
        return r;
    };
    w.x0 = take(E * Bp * L.k_pad);
    w.x0t = take(E * Bp * L.k_pad);
    for (int l = 1; l <= n_hidden; ++l) {
        w.h[l] = take(E * Bp * hidden);
        w.ht[l] = take(E * Bp * hidden);
    }
    w.zh = take(sizeof(float) * Bp * L.n_out_pad);
    for (int k = 0; k < 3; ++k) {   // delta ring (pod_ppo.cuh backward)
        w.d[k] = take(E * Bp * w.dmax);
        w.dt[k] = take(E * Bp * w.dmax);
    }
    for (int l = 1; l <= n_hidden; ++l)   // W_l^T [in_l][out_l (head: padded to 64)]
        w.wt[l] = take(E * static_cast<size_t>(hidden) * (l == n_hidden ? w.kp64 : hidden));
    for (int l = 0; l < n_hidden; ++l) w.bpart[l] = take(sizeof(float) * (Bp / 128) * hidden);
    w.bpart[n_hidden] = take(sizeof(float) * (Bp / PPO_HEAD_ROWS) * L.n_out_pad);
    w.lspart = take(sizeof(float) * (Bp / PPO_HEAD_ROWS) * L.n_out_pad);
    w.act = take(sizeof(float) * Bp * n);
    w.lpo = take(sizeof(float) * Bp);
    w.adv = take(sizeof(float) * Bp);
    w.ret = take(sizeof(float) * Bp);
    w.grad = take(sizeof(float) * L.n_elems);
    w.hpd = take(256);
    w.total = o;
    return w;
}

// captured minibatch loops, keyed on every pointer and size (not adam_t, the hyper-parameters or the stream)
struct PpoGraphKey {
    const void* p[16];
    int64_t M, k_pad, n_elems;
    int32_t cfg_n, n_hidden, hidden, act, batch, n_mb, dev, fp32;
    size_t param_bytes, ws_bytes;
    bool operator==(const PpoGraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};
struct PpoGraph {
    PpoGraphKey key;
    cudaGraphExec_t exec;
    uint64_t used;
    unsigned long long kernels;   // kernel nodes of the graph
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

// the side branch of the backward pass (weight-gradient products) and its fork / join events, per thread
// and device
inline cudaStream_t ppo_side_stream() {
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
inline cudaEvent_t* ppo_events() {
    static thread_local cudaEvent_t ev[12] = {};
    static thread_local int dev = -1;
    int d = 0;
    cudaGetDevice(&d);
    if (!ev[0] || d != dev) {
        for (auto& e : ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        dev = d;
    }
    return ev;
}

// host mirror of the learner's error word, per workspace (the next call on the same workspace refuses to
// run after a non-finite loss; pod_ppo_check synchronises and clears)
struct PpoErrMirror {
    const void* ws;
    uint32_t* h;
};
inline std::vector<PpoErrMirror>& ppo_err_mirrors() {
    static std::vector<PpoErrMirror> v;
    return v;
}
inline uint32_t* ppo_err_host(const void* ws) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& m : ppo_err_mirrors())
        if (m.ws == ws) return m.h;
    uint32_t* h = nullptr;
    if (cudaMallocHost(reinterpret_cast<void**>(&h), sizeof(uint32_t)) != cudaSuccess) return nullptr;
    *h = 0;
    ppo_err_mirrors().push_back(PpoErrMirror{ws, h});
    return h;
}

// plain stream-ordered launch (programmatic dependent launch was measured: no gain for these kernels, in a
// graph or eagerly — tools/gemm_probe.cu)
template <typename... KArgs, typename... Args>
pod_status launch_k(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = g;
    lc.blockDim = b;
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    POD_CUDA(cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...));
    pod_note_launch(s);
    return POD_OK;
}

// one product C = A B^T into the epilogue, on the tensor cores (bf16) or the float32 reference core
template <class T>
struct PpoGemm;

template <>
struct PpoGemm<__nv_bfloat16> {
    static pod_status run(const void* A, int lda, int rowsA, const void* B, int ldb, int rowsB, int K, int grid_rows,
                          const GemmEpi<__nv_bfloat16>& ep, cudaStream_t s) {
        CUtensorMap ma, mb;
        const uint64_t da[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(rowsA)};
        const uint64_t sa[1] = {static_cast<uint64_t>(lda) * 2};
        const uint32_t ba[2] = {GEMM_BK, GEMM_BM};
        pod_status st = encode_bf16(&ma, A, 2, da, sa, ba);
        if (st) return st;
        const uint64_t db[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(rowsB)};
        const uint64_t sb[1] = {static_cast<uint64_t>(ldb) * 2};
        const uint32_t bb[2] = {GEMM_BK, PPO_BN};
        st = encode_bf16(&mb, B, 2, db, sb, bb);
        if (st) return st;
        const dim3 grid(static_cast<unsigned>((grid_rows + GEMM_BM - 1) / GEMM_BM),
                        static_cast<unsigned>((ep.N + PPO_BN - 1) / PPO_BN));
        return launch_k(tc_gemm_kernel<PPO_BN>, grid, dim3(128), gemm_smem_bytes(PPO_BN), s, ma, mb, ep, K);
    }
};

template <>
struct PpoGemm<float> {
    static pod_status run(const void* A, int lda, int rowsA, const void* B, int ldb, int rowsB, int K, int grid_rows,
                          const GemmEpi<float>& ep, cudaStream_t s) {
        const dim3 grid(static_cast<unsigned>((grid_rows + GEMM_BM - 1) / GEMM_BM),
                        static_cast<unsigned>((ep.N + PPO_BN - 1) / PPO_BN));
        return launch_k(simt_gemm_f32_kernel<PPO_BN>, grid, dim3(128), 0, s, static_cast<const float*>(A), lda, rowsA,
                          static_cast<const float*>(B), ldb, rowsB, K, ep);
    }
};

struct PpoPlan {
    const pod_actor_layout* L;
    int n_hidden, hidden, act, n, B, n_mb;
    const PpoWs* W;
    char* ws;
    const void* params;   // the rollout slab (bf16 weights: the bf16 forward's B operands)
    float* master;
    float* adam_m;
    float* adam_v;
    const uint16_t* obs;
    const float *act_raw, *logp_old, *adv, *ret;
    const int32_t* perm;
    double* losses;
    float* grad_out;
    const FuseArgs* fa;
    int64_t woff[POD_MAX_HIDDEN_LAYERS + 1], boff[POD_MAX_HIDDEN_LAYERS + 1], lsoff;
};

// the minibatch loop on stream s, operands of type T
template <class T>
pod_status ppo_enqueue(const PpoPlan& p, cudaStream_t s, cudaStream_t s2) {
    const pod_actor_layout& L = *p.L;
    const PpoWs& W = *p.W;
    char* w = p.ws;
    const int Bp = W.B_pad, H = p.hidden, NL = L.n_layers;
    PpoDev* hpd = reinterpret_cast<PpoDev*>(w + W.hpd);
    T* x0 = reinterpret_cast<T*>(w + W.x0);
    T* x0t = reinterpret_cast<T*>(w + W.x0t);
    auto X = [&](int l) { return l == 0 ? x0 : reinterpret_cast<T*>(w + W.h[l]); };
    auto XT = [&](int l) { return l == 0 ? x0t : reinterpret_cast<T*>(w + W.ht[l]); };
    auto in_of = [&](int l) { return L.w_cols[l]; };
    auto kout_of = [&](int l) { return l == NL - 1 ? W.kp64 : H; };   // padded K of the input-gradient product
    float* zh = reinterpret_cast<float*>(w + W.zh);
    float* grad = reinterpret_cast<float*>(w + W.grad);
    const bool f32 = sizeof(T) == 4;
    // forward B operands: the slab (bf16) or the master (float32), both [out][in] K-contiguous
    auto wfwd = [&](int l) -> const void* {
        return f32 ? static_cast<const void*>(p.master + p.woff[l])
                   : static_cast<const void*>(static_cast<const char*>(p.params) + L.w_offset[l]);
    };
    PpoWt<T> wta{};
    int wt_gx = 1, wt_gy = 1;
    for (int l = 1; l < NL; ++l) {
        const int z = wta.n++;
        wta.w[z] = p.master + p.woff[l];
        wta.wt[z] = reinterpret_cast<T*>(w + W.wt[l]);
        wta.out[z] = L.w_rows[l];
        wta.in[z] = in_of(l);
        wta.ld[z] = kout_of(l);
        wt_gx = std::max(wt_gx, (in_of(l) + 31) / 32);
        wt_gy = std::max(wt_gy, (kout_of(l) + 31) / 32);
    }
    auto refresh_wt = [&](cudaStream_t st_) -> pod_status {
        if (wta.n == 0) return POD_OK;
        const dim3 g(static_cast<unsigned>(wt_gx), static_cast<unsigned>(wt_gy), static_cast<unsigned>(wta.n));
        return launch_k(ppo_wt_kernel<T>, g, dim3(256), 0, st_, wta);
    };
    auto gather = [&](int j, cudaStream_t st_) -> pod_status {
        const dim3 g(static_cast<unsigned>(Bp / 32), static_cast<unsigned>(L.k_pad / 64));
        return launch_k(ppo_gather_kernel<T>, g, dim3(256), 0, st_, p.obs, p.act_raw, p.logp_old, p.adv, p.ret,
                          p.perm + static_cast<int64_t>(j) * p.B, p.B, Bp, static_cast<int>(L.k_pad), p.n, x0, x0t,
                          reinterpret_cast<float*>(w + W.act), reinterpret_cast<float*>(w + W.lpo),
                          reinterpret_cast<float*>(w + W.adv), reinterpret_cast<float*>(w + W.ret));
    };
    PpoBiasReduce br{};
    br.n_layers = NL;
    br.n = p.n;
    br.n_out_pad = L.n_out_pad;
    for (int l = 0; l < NL; ++l) {
        br.nparts[l] = l == NL - 1 ? Bp / PPO_HEAD_ROWS : Bp / GEMM_BM;
        br.rows[l] = L.w_rows[l];
        br.part[l] = reinterpret_cast<const float*>(w + W.bpart[l]);
    }
    br.lspart = reinterpret_cast<const float*>(w + W.lspart);
    const int64_t g8 = p.fa->n_elems / 8;
    const dim3 ngrid(static_cast<unsigned>(std::min<int64_t>((g8 + 255) / 256, 8 * 148)), 1);
    cudaEvent_t* ev = ppo_events();
    if (!ev) return pod_fail(POD_ERR_CUDA, "PPO event creation failed");
    // events: 0 fork of the backward branch, 1..3 delta_l ready, 4..6 dW_l done, 7 branch joined,
    // 8 next minibatch gathered (side), 9 W^T refreshed (side), 10 Adam done
    // Pipeline across minibatches: the next minibatch's gather and W^T refresh run on the side branch while
    // this one's Adam step runs on the main chain.
    pod_status st = POD_OK;
    if (p.n_mb > 0) {
        st = gather(0, s);
        if (st) return st;
        st = refresh_wt(s);
        if (st) return st;
    }
    for (int j = 0; j < p.n_mb; ++j) {
        if (j > 0) POD_CUDA(cudaStreamWaitEvent(s, ev[8], 0));   // X0 of this minibatch
        // forward: X_{l+1} = act(X_l W_l^T + b_l); the head's output Z = X_L W_L^T + b_L (f32)
        for (int l = 0; l < NL; ++l) {
            const bool head = l == NL - 1;
            GemmEpi<T> ep{};
            ep.mode = head ? EPI_FWD_HEAD : EPI_FWD_HIDDEN;
            ep.M = p.B;
            ep.N = L.w_rows[l];
            ep.act = p.act;
            ep.bias = p.master + p.boff[l];
            if (head) {
                ep.outf = zh;
                ep.ld_outf = L.n_out_pad;
            } else {
                ep.out = X(l + 1);
                ep.ld_out = H;
                ep.out_t = XT(l + 1);
                ep.ld_out_t = Bp;
            }
            st = PpoGemm<T>::run(X(l), in_of(l), Bp, wfwd(l), in_of(l), L.w_rows[l], in_of(l), Bp, ep, s);
            if (st) return st;
        }
        PpoHead<T> hh{p.B, Bp, p.n, L.n_out_pad, W.kp64, hpd,
                      reinterpret_cast<const float*>(w + W.act), reinterpret_cast<const float*>(w + W.lpo),
                      reinterpret_cast<const float*>(w + W.adv), reinterpret_cast<const float*>(w + W.ret),
                      zh, p.master + p.lsoff, reinterpret_cast<T*>(w + W.d[0]), reinterpret_cast<T*>(w + W.dt[0]),
                      reinterpret_cast<float*>(w + W.bpart[NL - 1]), reinterpret_cast<float*>(w + W.lspart),
                      p.losses};
        st = launch_k(ppo_head_kernel<T>, dim3(Bp / PPO_HEAD_ROWS), dim3(32 * PPO_HEAD_WARPS), 0, s, hh);
        if (st) return st;
        // backward: dW_l = delta_l^T X_l on the side branch (stream s2), delta_{l-1} = (delta_l W_l) * act'(X_l)
        // on the main chain: the weight-gradient products overlap the input-gradient chain.  delta_l lives
        // in ring buffer (L - l) % 3; dX_l writes delta_{l-1} into the buffer of delta_{l+2}, so it waits for
        // dW_{l+2} (long finished in practice).
        POD_CUDA(cudaEventRecord(ev[0], s));
        POD_CUDA(cudaStreamWaitEvent(s2, ev[0], 0));
        if (j > 0) POD_CUDA(cudaStreamWaitEvent(s, ev[9], 0));   // W^T of the updated master
        for (int l = NL - 1; l >= 0; --l) {
            const int cur = (NL - 1 - l) % 3, nxt = (NL - l) % 3;
            const T* dl = reinterpret_cast<const T*>(w + W.d[cur]);
            const T* dlt = reinterpret_cast<const T*>(w + W.dt[cur]);
            if (l < NL - 1) {   // dW_l reads delta_l, written by the chain's dX_{l+1}
                POD_CUDA(cudaEventRecord(ev[1 + (l % 3)], s));
                POD_CUDA(cudaStreamWaitEvent(s2, ev[1 + (l % 3)], 0));
            }
            {
                GemmEpi<T> ep{};
                ep.mode = EPI_DW;
                ep.M = L.w_rows[l];
                ep.N = in_of(l);
                ep.outf = grad + p.woff[l];
                ep.ld_outf = in_of(l);
                st = PpoGemm<T>::run(dlt, Bp, L.w_rows[l], XT(l), Bp, in_of(l), Bp, L.w_rows[l], ep, s2);
                if (st) return st;
                POD_CUDA(cudaEventRecord(ev[4 + (l % 3)], s2));   // dW_l done (its delta buffer is free)
            }
            if (l > 0) {
                // the buffer this product writes, (NL - l) % 3, is the one dW_{l+2} reads
                if (l + 2 <= NL - 1) POD_CUDA(cudaStreamWaitEvent(s, ev[4 + ((l + 2) % 3)], 0));
                GemmEpi<T> ep{};
                ep.mode = EPI_DX;
                ep.M = p.B;
                ep.N = in_of(l);
                ep.act = p.act;
                ep.out = reinterpret_cast<T*>(w + W.d[nxt]);
                ep.ld_out = H;
                ep.out_t = reinterpret_cast<T*>(w + W.dt[nxt]);
                ep.ld_out_t = Bp;
                ep.xl = X(l);
                ep.ld_xl = H;
                ep.bpart = reinterpret_cast<float*>(w + W.bpart[l - 1]);
                const int ko = kout_of(l);
                st = PpoGemm<T>::run(dl, ko, Bp, w + W.wt[l], ko, in_of(l), ko, Bp, ep, s);
                if (st) return st;
            }
        }
        POD_CUDA(cudaEventRecord(ev[7], s2));
        POD_CUDA(cudaStreamWaitEvent(s, ev[7], 0));   // every weight gradient is in `grad`
        if (j + 1 < p.n_mb) {
            // the side branch (already past this minibatch's dW_0, the last reader of X0) gathers the next one
            st = gather(j + 1, s2);
            if (st) return st;
            POD_CUDA(cudaEventRecord(ev[8], s2));
        }
        // Adam on the master (bias / log-std gradients reduced from their partials), narrowed into the slab
        st = launch_k(ppo_adam_narrow_kernel, ngrid, dim3(256), 0, s, *p.fa, br, p.adam_m, p.adam_v, grad,
                        static_cast<const PpoDev*>(hpd), j);
        if (st) return st;
        if (p.grad_out && j == p.n_mb - 1)
            POD_CUDA(cudaMemcpyAsync(p.grad_out, grad, sizeof(float) * L.n_elems, cudaMemcpyDeviceToDevice, s));
        if (j + 1 < p.n_mb) {   // W^T of the updated master, on the side branch, for the next backward pass
            POD_CUDA(cudaEventRecord(ev[10], s));
            POD_CUDA(cudaStreamWaitEvent(s2, ev[10], 0));
            st = refresh_wt(s2);
            if (st) return st;
            POD_CUDA(cudaEventRecord(ev[9], s2));
        }
    }
    // (the last minibatch's join above leaves nothing on the side branch: the capture is closed on s)
    if (p.n_mb == 0) {
        fuse_blend_kernel<<<ngrid, 256, 0, s>>>(*p.fa);
        pod_note_launch(s);
        POD_CUDA(cudaGetLastError());
    }
    return POD_OK;
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

extern "C" pod_status pod_ppo_check(void* ws, void* stream) {
    if (!ws) return pod_fail(POD_ERR_ARG, "ws is NULL");
    uint32_t* h = pod::ppo_err_host(ws);
    if (!h) return pod_fail(POD_ERR_CUDA, "pinned error mirror allocation failed");
    POD_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    const uint32_t e = *static_cast<volatile uint32_t*>(h);
    *static_cast<volatile uint32_t*>(h) = 0;
    if (e) return pod_fail(POD_ERR_NONFINITE, "a PPO minibatch loss was not finite (the update was skipped)");
    return POD_OK;
}

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
    if (hp->fp32_operands != 0 && hp->fp32_operands != 1) return pod_fail(POD_ERR_ARG, "fp32_operands must be 0 or 1");
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
        reinterpret_cast<uintptr_t>(params) % 16 != 0 || reinterpret_cast<uintptr_t>(obs) % 16 != 0)
        return pod_fail(POD_ERR_ARG, "ws must be 256-byte aligned, master, adam_m, adam_v, params and obs 16-byte aligned");
    st = pod_require_sm100();
    if (st) return st;
    uint32_t* herr = ppo_err_host(ws);
    if (!herr) return pod_fail(POD_ERR_CUDA, "pinned error mirror allocation failed");
    if (*static_cast<volatile uint32_t*>(herr))
        return pod_fail(POD_ERR_NONFINITE,
                        "an earlier update on this workspace had a non-finite loss (S:L288: divergence); "
                        "pod_ppo_check clears it");
    cudaStream_t user_s = static_cast<cudaStream_t>(stream);
    {
        // per-device opt-in of the GEMM kernel's shared memory
        static std::mutex mu;
        static bool done[64] = {};
        int dev = 0;
        POD_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 0 && dev < 64 && !done[dev]) {
            POD_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<PPO_BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          gemm_smem_bytes(PPO_BN)));
            done[dev] = true;
        }
    }
    char* w = static_cast<char*>(ws);
    PpoDev* hpd = reinterpret_cast<PpoDev*>(w + W.hpd);
    PpoPlan p{};
    p.L = &L;
    p.n_hidden = n_hidden;
    p.hidden = hidden;
    p.act = act;
    p.n = n;
    p.B = batch;
    p.n_mb = n_minibatches;
    p.W = &W;
    p.ws = w;
    p.params = params;
    p.master = master;
    p.adam_m = adam_m;
    p.adam_v = adam_v;
    p.obs = obs;
    p.act_raw = act_raw;
    p.logp_old = logp_old;
    p.adv = adv;
    p.ret = ret;
    p.perm = perm;
    p.losses = losses;
    p.grad_out = grad_out;
    // flat offsets (elements) of W_l, b_l, log_std: pod_fuse_pods order
    int64_t f = 0;
    for (int l = 0; l < L.n_layers; ++l) {
        p.woff[l] = f;
        f += static_cast<int64_t>(L.w_rows[l]) * L.w_cols[l];
    }
    for (int l = 0; l < L.n_layers; ++l) {
        p.boff[l] = f;
        f += L.w_rows[l];
    }
    p.lsoff = f;
    // slab refresh from the master copy after every Adam step (the bf16 forward reads the slab): the fusion
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
    p.fa = &fa;
    const bool f32 = hp->fp32_operands == 1;
    cudaStream_t side = ppo_side_stream();
    if (!side) return pod_fail(POD_ERR_CUDA, "PPO side stream creation failed");
    auto enqueue = [&](cudaStream_t s) -> pod_status {
        return f32 ? ppo_enqueue<float>(p, s, side) : ppo_enqueue<__nv_bfloat16>(p, s, side);
    };
    ppo_set_step_kernel<<<1, 1, 0, user_s>>>(hpd, adam_t, hp->ratio_clip, hp->entropy_coef, hp->value_coef,
                                             hp->learning_rate, hp->adam_beta1, hp->adam_beta2, hp->adam_eps);
    pod_note_launch(user_s);
    POD_CUDA(cudaGetLastError());
    static const bool use_graph = [] {
        const char* e = std::getenv("POD_PPO_GRAPH");
        return !(e && e[0] == '0');
    }();
    if (!use_graph) {
        st = enqueue(user_s);
        if (st) return st;
    } else {
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
        key.fp32 = f32 ? 1 : 0;
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
            const unsigned long long kn = pod_graph_kernel_nodes(graph);
            cudaGraphDestroy(graph);
            if (ce != cudaSuccess) return pod_fail(POD_ERR_CUDA, "PPO graph instantiate: %s", cudaGetErrorString(ce));
            if (cache.size() >= kPpoGraphCache) {   // evict the least recently used
                size_t victim = 0;
                for (size_t i = 1; i < cache.size(); ++i)
                    if (cache[i].used < cache[victim].used) victim = i;
                cudaGraphExecDestroy(cache[victim].exec);
                cache.erase(cache.begin() + static_cast<long>(victim));
            }
            cache.push_back(PpoGraph{key, exec, 0, kn});
            hit = &cache.back();
        }
        hit->used = ++ppo_clock;
        POD_CUDA(cudaGraphLaunch(hit->exec, user_s));
        pod_note_graph_launch(hit->kernels);
    }
    // publish the error word to the host mirror of this workspace (read by the next call / pod_ppo_check)
    POD_CUDA(cudaMemcpyAsync(herr, &hpd->err, sizeof(uint32_t), cudaMemcpyDeviceToHost, user_s));
    return POD_OK;
}
