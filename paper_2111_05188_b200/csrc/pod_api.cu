// pod_api.cu — host side of libpod.so: the C ABI declared in include/pod.h.
// Validation, workspace carving, TMA descriptor encoding (cuTensorMapEncodeTiled
// through cudaGetDriverEntryPoint, so the library links no libcuda), the
// rollout driver (T x {actor, env-step} captured once into a CUDA graph and
// replayed), GAE and fitness launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <memory>
#include <mutex>
#include <vector>

#include "actor_kernel.cuh"
#include "env_kernel.cuh"
#include "fuse_kernel.cuh"
#include "metrics_kernel.cuh"
#include "gae_kernel.cuh"
#include "pod.h"
#include "pod_internal.h"

using namespace pod;

// ------------------------------------------------------------ error helpers
static thread_local char g_last_error[512] = "";

pod_status pod_fail(pod_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
    return s;
}

#define POD_CUDA(call)                                                                                \
    do {                                                                                              \
        cudaError_t _e = (call);                                                                      \
        if (_e != cudaSuccess) return pod_fail(POD_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
    } while (0)

extern "C" const char* pod_status_string(pod_status s) {
    switch (s) {
        case POD_OK: return "POD_OK";
        case POD_ERR_ARG: return "POD_ERR_ARG";
        case POD_ERR_SHAPE: return "POD_ERR_SHAPE";
        case POD_ERR_RANGE: return "POD_ERR_RANGE";
        case POD_ERR_WORKSPACE: return "POD_ERR_WORKSPACE";
        case POD_ERR_CUDA: return "POD_ERR_CUDA";
        case POD_ERR_NCCL: return "POD_ERR_NCCL";
        case POD_ERR_NONFINITE: return "POD_ERR_NONFINITE";
        case POD_ERR_UNSUPPORTED: return "POD_ERR_UNSUPPORTED";
    }
    return "POD_ERR_UNKNOWN";
}
extern "C" const char* pod_last_error(void) { return g_last_error; }
extern "C" int pod_abi_version(void) { return POD_ABI_VERSION; }

static inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------ device check
pod_status pod_require_sm100() {
    static thread_local int ok_dev = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return pod_fail(POD_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    if (dev == ok_dev) return POD_OK;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return pod_fail(POD_ERR_UNSUPPORTED, "device %d is sm_%d%d; libpod is built for sm_100a only", dev, major, minor);
    ok_dev = dev;
    return POD_OK;
}

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// bf16 tensor, rank 2 or 3, 128B swizzle (box inner 64 elements) or 64B swizzle (32 elements)
static pod_status encode_bf16(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                              const uint64_t* strides_bytes, const uint32_t* box,
                              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return pod_fail(POD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t d[4], s[3];
    cuuint32_t b[4], es[4] = {1, 1, 1, 1};
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
    }
    for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<cuuint32_t>(rank), const_cast<void*>(base), d, s, b,
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return pod_fail(POD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return POD_OK;
}

// 2-D, no swizzle (state tiles for the env-step kernel)
static pod_status encode_plain(CUtensorMap* m, const void* base, CUtensorMapDataType dt, const uint64_t* dims,
                               const uint64_t* strides_bytes, const uint32_t* box) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return pod_fail(POD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t d[2] = {dims[0], dims[1]}, s[1] = {strides_bytes[0]};
    cuuint32_t b[2] = {box[0], box[1]}, es[2] = {1, 1};
    CUresult r = enc(m, dt, 2, const_cast<void*>(base), d, s, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return pod_fail(POD_ERR_CUDA, "cuTensorMapEncodeTiled (state) failed (%d)", static_cast<int>(r));
    return POD_OK;
}

// ------------------------------------------------------------ layout
static pod_status dims_of(const pod_env_config* c, int* obs_dim, int* k_pad, int* n_out_pad) {
    if (!c) return pod_fail(POD_ERR_ARG, "config is NULL");
    if (c->n_stocks < 1 || c->n_feat < 0) return pod_fail(POD_ERR_ARG, "n_stocks >= 1 and n_feat >= 0 required");
    *obs_dim = 1 + 2 * c->n_stocks + c->n_stocks * c->n_feat;
    *k_pad = static_cast<int>(round_up(static_cast<size_t>(*obs_dim), 64));
    // head rows: the n action means, then the critic V in row n (R#22), padded to the 32-row MMA granule
    *n_out_pad = static_cast<int>(round_up(static_cast<size_t>(c->n_stocks) + 1, 32));
    if (*k_pad > ENV_MAX_KPAD || c->n_stocks > ENV_MAX_STOCKS)
        return pod_fail(POD_ERR_UNSUPPORTED, "obs_dim %d exceeds the kernel limit (k_pad <= %d, n <= %d)", *obs_dim,
                        ENV_MAX_KPAD, ENV_MAX_STOCKS);
    return POD_OK;
}

extern "C" pod_status pod_actor_layout_get(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                                           pod_actor_layout* out) {
    if (!out) return pod_fail(POD_ERR_ARG, "out is NULL");
    int od = 0, kp = 0, nop = 0;
    pod_status st = dims_of(cfg, &od, &kp, &nop);
    if (st) return st;
    if (n_hidden < 1 || n_hidden > POD_MAX_HIDDEN_LAYERS)
        return pod_fail(POD_ERR_UNSUPPORTED, "n_hidden must be in [1, %d]", POD_MAX_HIDDEN_LAYERS);
    if (!(hidden == 128 || hidden == 256 || hidden == 512))
        return pod_fail(POD_ERR_UNSUPPORTED, "hidden must be one of 128, 256, 512");
    if (nop > 128) return pod_fail(POD_ERR_UNSUPPORTED, "n_stocks + 1 > 128");
    memset(out, 0, sizeof(*out));
    out->obs_dim = od;
    out->k_pad = kp;
    out->n_out_pad = nop;
    out->n_layers = n_hidden + 1;
    size_t off = 0;
    for (int l = 0; l <= n_hidden; ++l) {
        out->w_rows[l] = l == n_hidden ? nop : hidden;
        out->w_cols[l] = l == 0 ? kp : hidden;
        out->w_offset[l] = off;
        off += static_cast<size_t>(out->w_rows[l]) * out->w_cols[l] * 2;
        off = round_up(off, 128);
    }
    for (int l = 0; l <= n_hidden; ++l) {
        out->b_offset[l] = off;
        off += static_cast<size_t>(out->w_rows[l]) * 4;
        off = round_up(off, 128);
    }
    out->log_std_offset = off;
    off += static_cast<size_t>(nop) * 4;
    out->param_bytes = round_up(off, 1024);
    size_t ne = static_cast<size_t>(nop);
    for (int l = 0; l <= n_hidden; ++l) ne += static_cast<size_t>(out->w_rows[l]) * (out->w_cols[l] + 1);
    out->n_elems = ne;
    return POD_OK;
}

// ------------------------------------------------------------ env handle
#define POD_MAX_GROUPS 4

struct GraphKey {
    int32_t T, deterministic, n_hidden, hidden, act, profile;
    const void* ptrs[14];
    size_t param_bytes;
};

// CUDA events recorded around the actor / env-step launches of every stride-th
// step of one rollout (profiling mode): ev[4 (m G + g) + 0..1] bracket group g's
// actor at marked step m, ev[4 (m G + g) + 2..3] its env step.
struct ProfEvents {
    std::vector<cudaEvent_t> ev;
    std::vector<double> frac;   // envs of group g / N
    int T = 0;
    int stride = 1;
    int n_marked = 0;
    int groups = 1;
    bool injected = false;
    pod_status create(int T_, int stride_, bool inj, int G, const std::vector<double>& fr) {
        T = T_;
        stride = stride_ < 1 ? 1 : stride_;
        n_marked = (T_ + stride - 1) / stride;
        injected = inj;
        groups = G;
        frac = fr;
        ev.resize(static_cast<size_t>(4) * n_marked * G);
        for (auto& x : ev)
            if (cudaEventCreate(&x) != cudaSuccess) return pod_fail(POD_ERR_CUDA, "cudaEventCreate failed");
        return POD_OK;
    }
    void destroy() {
        for (auto& x : ev)
            if (x) cudaEventDestroy(x);
        ev.clear();
    }
};

static std::atomic<unsigned long long> g_kernel_launches{0};
void pod_note_launch(cudaStream_t s, unsigned long long n) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) cs = cudaStreamCaptureStatusNone;
    if (cs == cudaStreamCaptureStatusNone) g_kernel_launches.fetch_add(n, std::memory_order_relaxed);
}
unsigned long long pod_graph_kernel_nodes(cudaGraph_t g) {
    size_t n = 0;
    if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess || n == 0) return 0;
    std::vector<cudaGraphNode_t> nodes(n);
    if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
    unsigned long long k = 0;
    for (size_t i = 0; i < n; ++i) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
}
void pod_note_graph_launch(unsigned long long kernel_nodes) {
    g_kernel_launches.fetch_add(kernel_nodes, std::memory_order_relaxed);
}
extern "C" unsigned long long pod_kernel_launches(void) { return g_kernel_launches.load(std::memory_order_relaxed); }

struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t last_use;
    ProfEvents* prof;
    unsigned long long kernels;   // kernel nodes of the graph
};

struct pod_env {
    pod_env_config cfg;
    pod_market market;
    int obs_dim, k_pad, n_out_pad, n_tiles, per_agent, env_tma_ok, mc_ok;
    // env groups: independent slices of the envs whose actor / env-step chains run on
    // separate graph branches, so one group's env step overlaps another's actor
    int groups;
    int g_m0[POD_MAX_GROUPS + 1];          // M-tile boundaries (128 envs)
    cudaStream_t gstream[POD_MAX_GROUPS];
    cudaEvent_t fork_ev, join_ev[POD_MAX_GROUPS];
    EnvMaps env_maps;
    // workspace carve
    int32_t* hold;
    int16_t* aint;
    float* logp_parts;          // [4][N] K1's log-prob partials, combined by K2
    float* znoise;
    double *cash, *asset, *disc, *ep_ret, *tile_gpow;
    int32_t *tile_start, *tile_k;
    uint64_t* step;
    uint32_t* err;
    uint32_t* h_err;     // pinned host mirror of *err, refreshed by a D2H copy at the end of every rollout
    int32_t* h_starts;   // pinned staging for reset
    cudaStream_t cap_stream;
    std::vector<GraphEntry> graphs;
    uint64_t use_clock;
    bool use_graphs;
    int persist;                // persistent actor clusters (POD_PERSIST=0 turns it off)
    int pdl;                    // env step as a programmatic dependent of the actor (POD_PDL=0 turns it off)
    int fused;                  // the fused rollout kernel where eligible (POD_FUSED=0 turns it off)
    int wt_on;                  // weights re-tiled per rollout and streamed by 1-D bulk copies (POD_WT=0: tensor maps)
    char* wt;                   // the re-tiled weights (cudaMalloc'd on first use, grown as needed)
    size_t wt_bytes;
    int sm_count;
    int profile;                // 0 = off, k = bracket every k-th step
    unsigned long long* trace;  // diagnostics: actor clock64 stamps of the last launch
    unsigned long long* env_trace;
    ProfEvents* last_prof;      // events of the most recent profiled rollout
    ProfEvents direct_prof;     // events for non-graph profiled rollouts
};

struct WsLayout {
    size_t hold, aint, znoise, logp_parts, cash, asset, disc, ep_ret, tile_start, tile_k, tile_gpow, step, err, total;
};

static WsLayout ws_layout(const pod_env_config* c) {
    WsLayout w{};
    const size_t N = static_cast<size_t>(c->n_envs), n = static_cast<size_t>(c->n_stocks);
    const size_t NT = (N + POD_ENV_TILE - 1) / POD_ENV_TILE;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = round_up(off + bytes, 256);
        return o;
    };
    w.hold = take(n * N * 4);
    w.aint = take(n * N * 2);
    w.znoise = take(n * N * 4);
    w.logp_parts = take(4 * N * 4);
    w.cash = take(N * 8);
    w.asset = take(N * 8);
    w.disc = take(N * 8);
    w.ep_ret = take(N * 8);
    w.tile_start = take(NT * 4);
    w.tile_k = take(NT * 4);
    w.tile_gpow = take(NT * 8);
    w.step = take(8);
    w.err = take(4);
    w.total = off;
    return w;
}

static pod_status check_config(const pod_env_config* c) {
    if (!c) return pod_fail(POD_ERR_ARG, "config is NULL");
    if (c->n_envs < 1) return pod_fail(POD_ERR_ARG, "n_envs must be >= 1");
    if (c->n_agents < 1 || c->n_envs % c->n_agents != 0)
        return pod_fail(POD_ERR_ARG, "n_agents must be >= 1 and divide n_envs");
    if (c->horizon < 1) return pod_fail(POD_ERR_ARG, "horizon must be >= 1");
    if (c->h_max < 1 || c->h_max > 32767) return pod_fail(POD_ERR_ARG, "h_max must be in [1, 32767]");
    if (!(c->initial_capital > 0.0)) return pod_fail(POD_ERR_ARG, "initial_capital must be > 0");
    if (!(c->cost_rate >= 0.0 && c->cost_rate < 1.0)) return pod_fail(POD_ERR_ARG, "cost_rate must be in [0, 1)");
    if (!(c->gamma > 0.0 && c->gamma <= 1.0)) return pod_fail(POD_ERR_ARG, "gamma must be in (0, 1]");
    if (!(c->reward_scale == c->reward_scale)) return pod_fail(POD_ERR_ARG, "reward_scale is NaN");
    int od = 0, kp = 0, nop = 0;
    return dims_of(c, &od, &kp, &nop);
}

extern "C" pod_status pod_env_workspace_size(const pod_env_config* cfg, size_t* bytes) {
    pod_status st = check_config(cfg);
    if (st) return st;
    if (!bytes) return pod_fail(POD_ERR_ARG, "bytes is NULL");
    *bytes = ws_layout(cfg).total;
    return POD_OK;
}

extern "C" pod_status pod_env_create(const pod_env_config* cfg, const pod_market* market, void* ws, size_t ws_bytes,
                                     pod_env_t** out) {
    pod_status st = check_config(cfg);
    if (st) return st;
    if (!market || !market->close || (cfg->n_feat > 0 && !market->feat) || !out)
        return pod_fail(POD_ERR_ARG, "market tensors and out must be non-NULL");
    if (market->T_data < 2 || market->T_data >= (1ll << 31)) return pod_fail(POD_ERR_SHAPE, "T_data must be in [2, 2^31)");
    WsLayout w = ws_layout(cfg);
    if (!ws || ws_bytes < w.total) return pod_fail(POD_ERR_WORKSPACE, "workspace needs %zu bytes", w.total);
    if (reinterpret_cast<uintptr_t>(ws) % 256 != 0) return pod_fail(POD_ERR_WORKSPACE, "workspace must be 256-byte aligned");
    st = pod_require_sm100();
    if (st) return st;
    pod_env* e = new pod_env();
    e->cfg = *cfg;
    e->market = *market;
    dims_of(cfg, &e->obs_dim, &e->k_pad, &e->n_out_pad);
    e->n_tiles = (cfg->n_envs + POD_ENV_TILE - 1) / POD_ENV_TILE;
    e->per_agent = cfg->n_envs / cfg->n_agents;
    char* b = static_cast<char*>(ws);
    e->hold = reinterpret_cast<int32_t*>(b + w.hold);
    e->aint = reinterpret_cast<int16_t*>(b + w.aint);
    e->logp_parts = reinterpret_cast<float*>(b + w.logp_parts);
    e->znoise = reinterpret_cast<float*>(b + w.znoise);
    e->cash = reinterpret_cast<double*>(b + w.cash);
    e->asset = reinterpret_cast<double*>(b + w.asset);
    e->disc = reinterpret_cast<double*>(b + w.disc);
    e->ep_ret = reinterpret_cast<double*>(b + w.ep_ret);
    e->tile_start = reinterpret_cast<int32_t*>(b + w.tile_start);
    e->tile_k = reinterpret_cast<int32_t*>(b + w.tile_k);
    e->tile_gpow = reinterpret_cast<double*>(b + w.tile_gpow);
    e->step = reinterpret_cast<uint64_t*>(b + w.step);
    e->err = reinterpret_cast<uint32_t*>(b + w.err);
    e->use_clock = 0;
    {
        const int mt = (cfg->n_envs + 127) / 128;
        int G = 1;   // per-CTA latency bound at C3: branches run in lockstep, so 1 by default
        const char* gs = getenv("POD_GROUPS");
        if (gs && atoi(gs) >= 1) G = atoi(gs);
        if (G > POD_MAX_GROUPS) G = POD_MAX_GROUPS;
        if (G > mt) G = mt;
        if (e->per_agent % 128 != 0) G = 1;
        // weight-tile multicast across 2 M-tiles: measured no faster (the fills are limited by
        // shared-memory bandwidth under SS-mode MMAs, not by L2), so opt-in only
        const char* mcs = getenv("POD_MULTICAST");   // 1 or 2: pairs of M-tiles, 4: quads (8-CTA clusters)
        const int mcg = mcs ? (atoi(mcs) == 4 ? 4 : (atoi(mcs) >= 1 ? 2 : 0)) : 0;
        e->mc_ok = (mcg && e->per_agent % (128 * mcg) == 0) ? mcg : 0;
        // boundaries in units of M-tile pairs when agents fill pairs (the 2-SM actor needs them)
        const int unit = (e->per_agent % 256 == 0) ? 2 : 1;
        const int units = (mt + unit - 1) / unit;
        if (G > units) G = units;
        for (int g = 0; g <= G; ++g) {
            const int m = static_cast<int>(static_cast<int64_t>(g) * units / G) * unit;
            e->g_m0[g] = m < mt ? m : mt;
        }
        e->groups = G;
    }
    e->profile = 0;
    e->last_prof = nullptr;
    e->trace = nullptr;
    e->env_trace = nullptr;
    const char* ng = getenv("POD_NO_GRAPH");
    e->use_graphs = !(ng && ng[0] == '1');
    {
        const char* ps = getenv("POD_PERSIST");
        e->persist = !(ps && ps[0] == '0');
        const char* pd = getenv("POD_PDL");
        e->pdl = (pd && pd[0] == '0') ? 0 : ((pd && pd[0] == '2') ? 2 : 1);   // 2: every env step (experiments)
        const char* fu = getenv("POD_FUSED");
        e->fused = !(fu && fu[0] == '0');
        const char* wv = getenv("POD_WT");
        e->wt_on = !(wv && wv[0] == '0');
        e->wt = nullptr;
        e->wt_bytes = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (e->sm_count < 2) e->sm_count = 2;
    }
    cudaError_t ce = cudaMallocHost(reinterpret_cast<void**>(&e->h_starts), sizeof(int32_t) * e->n_tiles);
    if (ce == cudaSuccess) ce = cudaMallocHost(reinterpret_cast<void**>(&e->h_err), sizeof(uint32_t));
    if (ce == cudaSuccess) *e->h_err = 0;
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking);
    for (int g = 0; g < POD_MAX_GROUPS && ce == cudaSuccess; ++g) {
        ce = cudaStreamCreateWithFlags(&e->gstream[g], cudaStreamNonBlocking);
        if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->join_ev[g], cudaEventDisableTiming);
    }
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaMemset(e->err, 0, 4);
    if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(actor_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(rollout_fused_kernel<16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(rollout_fused_kernel<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(env_step_kernel<16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(env_step_kernel<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(gae_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(gae_smem_bytes()));
    if (ce != cudaSuccess) {
        delete e;
        return pod_fail(POD_ERR_CUDA, "pod_env_create: %s", cudaGetErrorString(ce));
    }
    {
        // the market must be usable by the float64 ledger: close prices finite and > 0, indicators finite
        const int64_t nc = static_cast<int64_t>(market->T_data) * cfg->n_stocks;
        const int64_t nf = static_cast<int64_t>(market->T_data) * cfg->n_feat * cfg->n_stocks;
        uint32_t flags = 0;
        market_check_kernel<<<296, 256>>>(market->close, nc, market->feat, nf, e->err);
        pod_note_launch(nullptr);
        ce = cudaGetLastError();
        if (ce == cudaSuccess) ce = cudaMemcpy(&flags, e->err, 4, cudaMemcpyDeviceToHost);
        if (ce == cudaSuccess) ce = cudaMemset(e->err, 0, 4);
        if (ce != cudaSuccess) {
            pod_env_destroy(e);
            return pod_fail(POD_ERR_CUDA, "pod_env_create (market check): %s", cudaGetErrorString(ce));
        }
        if (flags) {
            pod_env_destroy(e);
            return pod_fail(POD_ERR_NONFINITE, "market: %s%s", (flags & 1u) ? "close prices must be finite and > 0 " : "",
                            (flags & 2u) ? "indicators must be finite" : "");
        }
    }
    // 2-D tensor maps over the ticker-major state: one TMA box = one tile's [n][32]
    e->env_tma_ok = (cfg->n_envs % 8 == 0) ? 1 : 0;
    if (e->env_tma_ok) {
        const uint64_t N = static_cast<uint64_t>(cfg->n_envs), n = static_cast<uint64_t>(cfg->n_stocks);
        const uint64_t dh[2] = {N, n}, sh[1] = {N * 4};
        const uint64_t da[2] = {N, n}, sa[1] = {N * 2};
        const uint32_t box[2] = {32, static_cast<uint32_t>(n)};
        st = encode_plain(&e->env_maps.hold, e->hold, CU_TENSOR_MAP_DATA_TYPE_INT32, dh, sh, box);
        if (!st) st = encode_plain(&e->env_maps.aint, e->aint, CU_TENSOR_MAP_DATA_TYPE_UINT16, da, sa, box);
        if (st) {
            delete e;
            return st;
        }
    } else {
        memset(&e->env_maps, 0, sizeof(e->env_maps));
    }
    *out = e;
    return POD_OK;
}

extern "C" pod_status pod_env_destroy(pod_env_t* e) {
    if (!e) return POD_OK;
    if (e->wt) cudaFree(e->wt);
    for (auto& g : e->graphs) {
        cudaGraphExecDestroy(g.exec);
        if (g.prof) {
            g.prof->destroy();
            delete g.prof;
        }
    }
    e->direct_prof.destroy();
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
    for (int g = 0; g < POD_MAX_GROUPS; ++g) {
        if (e->gstream[g]) cudaStreamDestroy(e->gstream[g]);
        if (e->join_ev[g]) cudaEventDestroy(e->join_ev[g]);
    }
    if (e->fork_ev) cudaEventDestroy(e->fork_ev);
    if (e->h_starts) cudaFreeHost(e->h_starts);
    if (e->h_err) cudaFreeHost(e->h_err);
    delete e;
    return POD_OK;
}

static EnvArgs env_args(const pod_env* e, int mode) {
    EnvArgs a{};
    a.N = e->cfg.n_envs;
    a.n = e->cfg.n_stocks;
    a.f = e->cfg.n_feat;
    a.k_pad = e->k_pad;
    a.obs_dim = e->obs_dim;
    a.horizon = e->cfg.horizon;
    a.n_tiles = e->n_tiles;
    a.mode = mode;
    a.T_data = e->market.T_data;
    a.C0 = e->cfg.initial_capital;
    a.cost = e->cfg.cost_rate;
    a.scale = e->cfg.reward_scale;
    a.gamma = e->cfg.gamma;
    a.close = e->market.close;
    a.feat = e->market.feat;
    a.hold = e->hold;
    a.aint = e->aint;
    a.cash = e->cash;
    a.asset = e->asset;
    a.disc = e->disc;
    a.ep_ret = e->ep_ret;
    a.tile_start = e->tile_start;
    a.tile_k = e->tile_k;
    a.tile_gpow = e->tile_gpow;
    a.err = e->err;
    a.tma_ok = e->env_tma_ok;
    a.seed = e->cfg.seed;
    a.env_offset = e->cfg.env_offset;
    a.step_base = e->step;
    a.znoise = e->znoise;
    a.trace = e->env_trace;
    return a;
}

static inline int env_blocks(const pod_env* e) { return e->n_tiles; }
// the env-step instantiation for this handle's ticker count (ledger loop unroll depths)
using EnvStepFn = void (*)(EnvMaps, EnvArgs);
static inline EnvStepFn env_step_fn(const pod_env* e) {
    return e->cfg.n_stocks >= 64 ? env_step_kernel<16, 8> : env_step_kernel<8, 4>;
}

static inline size_t env_smem(const pod_env* e) {
    static const size_t over = [] {   // experiments: POD_ENV_SMEM=<bytes> raises the request (fewer tiles per SM)
        const char* v = getenv("POD_ENV_SMEM");
        return v ? static_cast<size_t>(atol(v)) : 0;
    }();
    return std::max(static_cast<size_t>(env_smem_bytes(e->cfg.n_stocks, e->k_pad)), over);
}

static uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

extern "C" pod_status pod_env_reset(pod_env_t* e, const int64_t* starts, uint16_t* obs0, void* stream) {
    if (!e) return pod_fail(POD_ERR_ARG, "env is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t max_start = e->market.T_data - 1 - e->cfg.horizon;
    if (max_start < 0) return pod_fail(POD_ERR_RANGE, "horizon %d does not fit in T_data %lld", e->cfg.horizon,
                                       static_cast<long long>(e->market.T_data));
    uint64_t rs = e->cfg.seed ^ 0x5EED5EED5EEDull;
    for (int i = 0; i < e->n_tiles; ++i) {
        int64_t v = starts ? starts[i] : static_cast<int64_t>(splitmix64(rs) % static_cast<uint64_t>(max_start + 1));
        if (v < 0 || v > max_start)
            return pod_fail(POD_ERR_RANGE, "tile %d start row %lld outside [0, %lld] (start + H <= T_data - 1)", i,
                            static_cast<long long>(v), static_cast<long long>(max_start));
        e->h_starts[i] = static_cast<int32_t>(v);
    }
    POD_CUDA(cudaMemcpyAsync(e->tile_start, e->h_starts, sizeof(int32_t) * e->n_tiles, cudaMemcpyHostToDevice, s));
    POD_CUDA(cudaMemsetAsync(e->step, 0, 8, s));
    POD_CUDA(cudaMemsetAsync(e->err, 0, 4, s));   // a fresh state carries no earlier fault
    EnvArgs a = env_args(e, 2);
    a.obs_out = obs0;
    env_step_fn(e)<<<env_blocks(e), ENV_THREADS, env_smem(e), s>>>(e->env_maps, a);
    pod_note_launch(s);
    POD_CUDA(cudaGetLastError());
    POD_CUDA(cudaStreamSynchronize(s));   // the pinned staging buffer is reused by the next reset
    *static_cast<volatile uint32_t*>(e->h_err) = 0;
    return POD_OK;
}

// ------------------------------------------------------------ rollout
struct RolloutPlan {
    bool injected;
    bool fused;          // one rollout_fused_kernel launch for the T steps (see fused_eligible)
    ActorMaps maps;
    ActorArgs aa;
    size_t actor_smem;
    RetileArgs ra;       // the weight re-tiling of this rollout (ra.wt null: none)
};

// The fused rollout needs every M-tile's cluster resident at once (one wave: the clusters are independent
// over the T steps, but a second wave would serialise T steps per tile), M-tiles aligned with the 32-env
// tiles and with agents, and both env tiles of a CTA inside its activation buffer.
static bool fused_eligible(const pod_env* e, const RolloutPlan& p) {
    // (env_tma_ok: the env tiles read the actions through the tensor map, i.e. from L2 — plain loads could hit
    // lines of the peer CTA's actions cached in this SM's L1 by an earlier step)
    if (!e->fused || p.injected || e->groups != 1 || e->mc_ok || !e->env_tma_ok) return false;
    if (e->per_agent % 128 != 0) return false;
    const int mtiles = e->cfg.n_agents * (e->per_agent / 128);
    if (2 * mtiles > e->sm_count) return false;
    return fused_env_fits(e->cfg.n_stocks, e->k_pad, p.aa.hidden);
}

// one group's chain: s_0, then T x {actor (or injected map), env step}
static void enqueue_group(pod_env* e, const RolloutPlan& p, int T, const pod_traj* tr, const float* inj, cudaStream_t s,
                          ProfEvents* prof, int g) {
    const int N = e->cfg.n_envs, n = e->cfg.n_stocks;
    const int m0 = e->g_m0[g], m1 = e->g_m0[g + 1];
    const int e0 = e->groups == 1 ? 0 : m0 * 128;
    const int e1 = e->groups == 1 ? N : (m1 * 128 < N ? m1 * 128 : N);
    const int t0 = e0 / POD_ENV_TILE, t1 = (e1 + POD_ENV_TILE - 1) / POD_ENV_TILE;
    auto mark = [&](int t, int k) {
        // external event-record node when captured into the graph (timing-capable);
        // only every `stride`-th step is bracketed, to keep the timing overhead small
        if (prof && t % prof->stride == 0)
            cudaEventRecordWithFlags(prof->ev[static_cast<size_t>(4 * ((t / prof->stride) * prof->groups + g) + k)], s,
                                     cudaEventRecordExternal);
    };
    const int sampling = (!p.injected && !p.aa.deterministic) ? 1 : 0;
    int actor_ctas = 0;   // CTAs of the last actor launch (SMs it occupies)
    auto launch_actor = [&](ActorArgs& aa) {
        // one 2-CTA cluster per 128-env tile (column split of every layer)
        cudaLaunchConfig_t lc{};
        const int mtiles = e->groups == 1 ? e->cfg.n_agents * aa.tiles_per_agent : (m1 - m0);
        // 4-CTA clusters (two M-tiles of one agent) share weight tiles by multicast when
        // every agent has an even number of full M-tiles and so does this launch
        aa.mc = (e->mc_ok && mtiles % e->mc_ok == 0 && m0 % e->mc_ok == 0) ? e->mc_ok : 0;
        aa.mtiles = mtiles;
        // persistent clusters (one per SM pair) loop over the M-tiles: the next tile's obs and first
        // weight stages load while the current tile's head runs (multi-wave batches)
        const int ncl = (!aa.mc && e->persist) ? std::min(mtiles, e->sm_count / 2) : mtiles;
        lc.gridDim = dim3(static_cast<unsigned>(2 * ncl));
        actor_ctas = static_cast<int>(lc.gridDim.x);
        lc.blockDim = dim3(ACT_THREADS);
        lc.dynamicSmemBytes = p.actor_smem;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = aa.mc ? 2 * aa.mc : 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, actor_forward_kernel, p.maps, aa);
        pod_note_launch(s);
    };
    EnvArgs a0 = env_args(e, 1);
    a0.tile0 = t0;
    a0.obs_out = tr->obs;
    a0.gen_noise = sampling;          // noise for the actor launch of step 0
    a0.noise_t = 0;
    env_step_fn(e)<<<t1 - t0, ENV_THREADS, env_smem(e), s>>>(e->env_maps, a0);
    pod_note_launch(s);
    if (p.fused && !prof) {
        // the T steps (and the critic bootstrap pass) in one launch: cluster c owns M-tile c for all steps
        FusedMaps fm;
        fm.am = p.maps;
        fm.em = e->env_maps;
        ActorArgs aa = p.aa;
        aa.t = 0;
        aa.obs_row0 = 0;
        aa.mtile0 = 0;
        aa.mc = 0;
        aa.mtiles = e->cfg.n_agents * (e->per_agent / 128);
        aa.act_out = tr->act;
        aa.logp_out = tr->logp;
        aa.logp_parts = e->logp_parts;
        aa.mu_out = tr->mu;
        aa.dbg_aint = tr->dbg_aint;
        aa.val_out = tr->val;
        FusedEnvArgs fe{};
        fe.env = env_args(e, 0);
        fe.env.rew = tr->rew;
        fe.env.done = tr->done;
        fe.env.obs_out = tr->obs + static_cast<int64_t>(N) * e->k_pad;
        fe.env.dbg_hold = tr->dbg_hold;
        fe.env.dbg_cash = tr->dbg_cash;
        fe.env.equity = tr->equity;
        fe.env.logp_parts = e->logp_parts;
        fe.env.logp_out = tr->logp;
        fe.env.trace = nullptr;
        fe.T = T;
        fe.sampling = sampling;
        fe.env_stride = (env_smem_bytes(n, e->k_pad) + 127) / 128 * 128;
        fe.k_pad = e->k_pad;
        // the env tiles' persistent state (header, ledger, the next step's market rows by bulk copy)
        fe.persist = p.actor_smem + 2 * static_cast<size_t>(env_persist_bytes(n, e->cfg.n_feat)) <= 232448
                         ? env_persist_bytes(n, e->cfg.n_feat) : 0;
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(static_cast<unsigned>(2 * aa.mtiles));
        lc.blockDim = dim3(ACT_THREADS);
        lc.dynamicSmemBytes = p.actor_smem + 2 * static_cast<size_t>(fe.persist);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        if (n >= 64) cudaLaunchKernelEx(&lc, rollout_fused_kernel<16, 8>, fm, aa, fe);
        else cudaLaunchKernelEx(&lc, rollout_fused_kernel<8, 4>, fm, aa, fe);
        pod_note_launch(s);
        return;
    }
    for (int t = 0; t < T; ++t) {
        mark(t, 0);
        if (p.injected) {
            const int64_t tot = static_cast<int64_t>(e1 - e0) * n;
            inject_map_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(
                inj + static_cast<int64_t>(t) * N * n, N, n, e->cfg.h_max, e->aint,
                tr->dbg_aint ? tr->dbg_aint + static_cast<int64_t>(t) * N * n : nullptr, e0, e1);
            pod_note_launch(s);
        } else {
            ActorArgs aa = p.aa;
            aa.t = t;
            aa.obs_row0 = t * N;
            aa.mtile0 = m0;
            aa.act_out = tr->act + static_cast<int64_t>(t) * N * n;
            aa.logp_out = tr->logp + static_cast<int64_t>(t) * N;
            aa.logp_parts = e->logp_parts;
            aa.mu_out = tr->mu ? tr->mu + static_cast<int64_t>(t) * N * n : nullptr;
            aa.dbg_aint = tr->dbg_aint ? tr->dbg_aint + static_cast<int64_t>(t) * N * n : nullptr;
            aa.val_out = tr->val ? tr->val + static_cast<int64_t>(t) * N : nullptr;
            launch_actor(aa);
        }
        mark(t, 1);
        mark(t, 2);
        EnvArgs a = env_args(e, 0);
        a.tile0 = t0;
        a.rew = tr->rew + static_cast<int64_t>(t) * N;
        a.done = tr->done + static_cast<int64_t>(t) * N;
        a.obs_out = tr->obs + static_cast<int64_t>(t + 1) * N * e->k_pad;
        a.dbg_hold = tr->dbg_hold ? tr->dbg_hold + static_cast<int64_t>(t) * N * n : nullptr;
        a.dbg_cash = tr->dbg_cash ? tr->dbg_cash + static_cast<int64_t>(t) * N : nullptr;
        a.equity = tr->equity ? tr->equity + static_cast<int64_t>(t) * N : nullptr;
        // the column-split actor leaves its log-prob partials to this step
        a.logp_parts = (!p.injected && tr->logp) ? e->logp_parts : nullptr;
        a.logp_out = a.logp_parts ? tr->logp + static_cast<int64_t>(t) * N : nullptr;
        a.gen_noise = (sampling && t + 1 < T) ? 1 : 0;   // noise for the actor launch of step t+1
        a.noise_t = t + 1;
        // Programmatic dependent of the actor launch just before (not across a profiling event node):
        // its blocks are scheduled as SMs free up, the first ones on the SMs the actor leaves idle.
        // Used when that helps: a dense launch (>= 7 tiles per SM: the launch latency is hidden as actor
        // CTAs exit) or a small one whose tiles fit two per idle SM (C2); not when a few idle SMs would
        // collect a dense, slow cluster of tiles ahead of the rest (C3: 20 idle SMs, 256 tiles).
        const int tiles = t1 - t0;
        const int idle_sms = std::max(0, e->sm_count - actor_ctas);
        const bool dense = tiles >= 7 * e->sm_count;
        const bool roomy = 2 * idle_sms >= tiles;
        const bool pdl = e->pdl && e->groups == 1 && !p.injected && (dense || roomy || e->pdl == 2) &&
                         !(prof && t % prof->stride == 0);
        if (pdl) {
            a.pdl = 1;
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(static_cast<unsigned>(t1 - t0));
            lc.blockDim = dim3(ENV_THREADS);
            lc.dynamicSmemBytes = static_cast<size_t>(env_smem(e));
            lc.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            cudaLaunchKernelEx(&lc, env_step_fn(e), e->env_maps, a);
            pod_note_launch(s);
        } else {
            env_step_fn(e)<<<t1 - t0, ENV_THREADS, env_smem(e), s>>>(e->env_maps, a);
            pod_note_launch(s);
        }
        mark(t, 3);
    }
    if (!p.injected && tr->val) {
        // critic bootstrap V(s_T): one value-only pass of the actor over obs[T] (no sampling, no action)
        ActorArgs aa = p.aa;
        aa.t = T;
        aa.obs_row0 = T * N;
        aa.mtile0 = m0;
        aa.value_only = 1;
        aa.deterministic = 1;
        aa.act_out = nullptr;
        aa.logp_out = nullptr;
        aa.mu_out = nullptr;
        aa.dbg_aint = nullptr;
        aa.val_out = tr->val + static_cast<int64_t>(T) * N;
        aa.logp_parts = e->logp_parts;   // written only with logp_out: untouched here
        launch_actor(aa);
    }
}

static pod_status enqueue_rollout(pod_env* e, const RolloutPlan& p, int T, const pod_traj* tr, const float* inj,
                                  double* fitness_out, cudaStream_t s, ProfEvents* prof) {
    if (p.ra.wt) {
        int maxc = 0;
        for (int l = 0; l < p.ra.n_layers; ++l) maxc = std::max(maxc, p.ra.rows[l] * (p.ra.cols[l] / 8));
        actor_retile_kernel<<<dim3(static_cast<unsigned>((maxc + 255) / 256), static_cast<unsigned>(p.ra.n_layers),
                               static_cast<unsigned>(e->cfg.n_agents)),
                              256, 0, s>>>(p.ra);
        pod_note_launch(s);
    }
    if (e->groups == 1) {
        enqueue_group(e, p, T, tr, inj, s, prof, 0);
    } else {
        // fork: each env group's chain on its own stream (graph branch), then join
        POD_CUDA(cudaEventRecord(e->fork_ev, s));
        for (int g = 0; g < e->groups; ++g) {
            POD_CUDA(cudaStreamWaitEvent(e->gstream[g], e->fork_ev, 0));
            enqueue_group(e, p, T, tr, inj, e->gstream[g], prof, g);
            POD_CUDA(cudaEventRecord(e->join_ev[g], e->gstream[g]));
            POD_CUDA(cudaStreamWaitEvent(s, e->join_ev[g], 0));
        }
    }
    if (!p.injected) bump_step_kernel<<<1, 1, 0, s>>>(e->step, static_cast<uint64_t>(T));
    if (!p.injected) pod_note_launch(s);
    if (fitness_out) fitness_kernel<<<e->cfg.n_agents, 1024, 0, s>>>(e->ep_ret, e->per_agent, fitness_out);
    if (fitness_out) pod_note_launch(s);
    POD_CUDA(cudaGetLastError());
    // publish the device error word to the pinned host mirror: the next pod_rollout refuses to run on a
    // state that an earlier rollout has already flagged (non-finite mean action or account value)
    POD_CUDA(cudaMemcpyAsync(e->h_err, e->err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    return POD_OK;
}

static std::vector<double> group_fracs(const pod_env* e) {
    std::vector<double> fr;
    const int N = e->cfg.n_envs;
    for (int g = 0; g < e->groups; ++g) {
        if (e->groups == 1) {
            fr.push_back(1.0);
        } else {
            const int e0 = e->g_m0[g] * 128;
            const int e1 = e->g_m0[g + 1] * 128 < N ? e->g_m0[g + 1] * 128 : N;
            fr.push_back(static_cast<double>(e1 - e0) / N);
        }
    }
    return fr;
}

extern "C" pod_status pod_rollout(pod_env_t* e, const pod_actor* actor, int32_t T, const pod_traj* tr,
                                  const float* injected_u, int32_t deterministic, double* fitness_out, void* stream) {
    if (!e || !tr) return pod_fail(POD_ERR_ARG, "env and traj must be non-NULL");
    if (T < 1) return pod_fail(POD_ERR_ARG, "T must be >= 1");
    if (!tr->obs || !tr->rew || !tr->done) return pod_fail(POD_ERR_ARG, "traj.obs, traj.rew and traj.done are required");
    if (reinterpret_cast<uintptr_t>(tr->obs) % 16 != 0) return pod_fail(POD_ERR_ARG, "traj.obs must be 16-byte aligned");
    const int N = e->cfg.n_envs;
    if (static_cast<int64_t>(T + 1) * N >= (1ll << 31)) return pod_fail(POD_ERR_SHAPE, "(T+1) * N must be < 2^31");
    {
        // an earlier rollout of this handle that has completed on the device flagged a non-finite actor
        // mean or account value (pod_env_check / pod_env_reset clear it)
        const uint32_t he = *static_cast<volatile uint32_t*>(e->h_err);
        if (he)
            return pod_fail(POD_ERR_NONFINITE,
                            "an earlier rollout set the device error word 0x%x (1 = non-finite actor mean, 2 = "
                            "non-finite account value); pod_env_check or pod_env_reset clears it", he);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    RolloutPlan p{};
    p.injected = injected_u != nullptr;
    if (!p.injected) {
        if (!actor || !actor->params) return pod_fail(POD_ERR_ARG, "actor (or injected_u) is required");
        if (!tr->act || !tr->logp) return pod_fail(POD_ERR_ARG, "traj.act and traj.logp are required when sampling");
        pod_actor_layout L;
        pod_status st = pod_actor_layout_get(&e->cfg, actor->n_hidden, actor->hidden, &L);
        if (st) return st;
        if (actor->act != 0 && actor->act != 1) return pod_fail(POD_ERR_ARG, "actor.act must be 0 (ReLU) or 1 (tanh)");
        if (actor->param_bytes < L.param_bytes || actor->param_bytes % 16 != 0)
            return pod_fail(POD_ERR_SHAPE, "param_bytes %zu must be >= %zu and a multiple of 16", actor->param_bytes,
                            L.param_bytes);
        if (reinterpret_cast<uintptr_t>(actor->params) % 16 != 0)
            return pod_fail(POD_ERR_ARG, "actor.params must be 16-byte aligned");
        // TMA descriptors: obs [(T+1) N][k_pad], weights [agents][out][in]
        {
            const uint64_t dims[2] = {static_cast<uint64_t>(e->k_pad), static_cast<uint64_t>(T + 1) * N};
            const uint64_t str[1] = {static_cast<uint64_t>(e->k_pad) * 2};
            const uint32_t box[2] = {64, 128};
            st = encode_bf16(&p.maps.obs, tr->obs, 2, dims, str, box);
            if (st) return st;
        }
        const char* kpe = getenv("POD_KPB");   // experiments: POD_KPB=0 keeps one box per stage
        const bool kpb_off = kpe && kpe[0] == '0';
        for (int l = 0; l < L.n_layers; ++l) {
            const int rows = L.w_rows[l];
            const int bn = actor_bn(rows / 2);   // this CTA's column half of the layer
            const int KB = L.w_cols[l] / ACT_BK;
            // narrow layers: several K blocks per ring stage (not with the multicast variant)
            const int kph = (bn < ACT_BN && !e->mc_ok && !kpb_off) ? actor_kpb(KB, bn, l > 0) : 1;
            p.aa.kpb_pack |= static_cast<uint32_t>(kph) << (5 * l);
            if (kph == 1) {
                const uint64_t dims[3] = {static_cast<uint64_t>(L.w_cols[l]), static_cast<uint64_t>(rows),
                                          static_cast<uint64_t>(e->cfg.n_agents)};
                const uint64_t str[2] = {static_cast<uint64_t>(L.w_cols[l]) * 2, actor->param_bytes};
                const uint32_t box[3] = {ACT_BK, static_cast<uint32_t>(bn), 1};
                st = encode_bf16(&p.maps.w[l], static_cast<const char*>(actor->params) + L.w_offset[l], 3, dims, str,
                                 box, ACT_BK == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : (ACT_BK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B));
            } else {
                // [agents][K block][out][32]: the K-block stride is 64 bytes inside each weight row
                const uint64_t dims[4] = {static_cast<uint64_t>(ACT_BK), static_cast<uint64_t>(rows),
                                          static_cast<uint64_t>(KB), static_cast<uint64_t>(e->cfg.n_agents)};
                const uint64_t str[3] = {static_cast<uint64_t>(L.w_cols[l]) * 2, ACT_BK * 2, actor->param_bytes};
                const uint32_t box[4] = {ACT_BK, static_cast<uint32_t>(bn), static_cast<uint32_t>(kph), 1};
                st = encode_bf16(&p.maps.w[l], static_cast<const char*>(actor->params) + L.w_offset[l], 4, dims, str,
                                 box, ACT_BK == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : (ACT_BK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B));
            }
            if (st) return st;
        }
        ActorArgs& aa = p.aa;
        aa.N = N;
        aa.per_agent = e->per_agent;
        aa.tiles_per_agent = (e->per_agent + 127) / 128;
        aa.n = e->cfg.n_stocks;
        aa.n_out_pad = L.n_out_pad;
        aa.k_pad = L.k_pad;
        aa.hidden = actor->hidden;
        aa.n_layers = L.n_layers;
        aa.act = actor->act;
        aa.h_max = e->cfg.h_max;
        aa.deterministic = deterministic ? 1 : 0;
        aa.seed = e->cfg.seed;
        aa.env_offset = e->cfg.env_offset;
        aa.step_base = e->step;
        aa.params = static_cast<const char*>(actor->params);
        aa.param_bytes = actor->param_bytes;
        for (int l = 0; l < L.n_layers; ++l) aa.b_off[l] = L.b_offset[l];
        aa.log_std_off = L.log_std_offset;
        aa.aint = e->aint;
        aa.znoise = e->znoise;
        aa.err = e->err;
        aa.trace = e->trace;
        p.actor_smem = actor_smem_bytes(L.k_pad, actor->hidden);
        if (p.actor_smem > 232448) return pod_fail(POD_ERR_UNSUPPORTED, "actor needs %zu B of shared memory", p.actor_smem);
        p.fused = fused_eligible(e, p);
        if (e->wt_on && !e->mc_ok) {
            // the weights re-tiled in ring-stage order once per rollout (they may change between rollouts)
            RetileArgs& ra = p.ra;
            ra.params = static_cast<const char*>(actor->params);
            ra.param_bytes = actor->param_bytes;
            ra.n_layers = L.n_layers;
            uint64_t off = 0;
            for (int l = 0; l < L.n_layers; ++l) {
                ra.w_off[l] = L.w_offset[l];
                ra.rows[l] = L.w_rows[l];
                ra.cols[l] = L.w_cols[l];
                ra.kp[l] = static_cast<int32_t>((p.aa.kpb_pack >> (5 * l)) & 31u);
                ra.layer_off[l] = off;
                p.aa.wt_layer_off[l] = off;
                off += static_cast<uint64_t>(L.w_rows[l]) * L.w_cols[l] * 2;
            }
            ra.agent_bytes = (off + 1023) / 1024 * 1024;
            const size_t need = ra.agent_bytes * static_cast<size_t>(e->cfg.n_agents);
            if (need > e->wt_bytes) {
                if (e->wt) cudaFree(e->wt);
                e->wt = nullptr;
                e->wt_bytes = 0;
                // a capture of the rollout graph may hold the old buffer: cached graphs are dropped with it
                for (auto& g : e->graphs) cudaGraphExecDestroy(g.exec);
                e->graphs.clear();
                POD_CUDA(cudaMalloc(reinterpret_cast<void**>(&e->wt), need));
                e->wt_bytes = need;
            }
            ra.wt = e->wt;
            p.aa.wt = e->wt;
            p.aa.wt_agent_bytes = ra.agent_bytes;
        }
    }
    if (!e->use_graphs) {
        ProfEvents* prof = nullptr;
        if (e->profile) {
            e->direct_prof.destroy();
            pod_status st = e->direct_prof.create(T, e->profile, p.injected, e->groups, group_fracs(e));
            if (st) return st;
            prof = &e->direct_prof;
        }
        e->last_prof = prof;
        return enqueue_rollout(e, p, T, tr, injected_u, fitness_out, s, prof);
    }

    GraphKey key;
    memset(&key, 0, sizeof(key));
    key.T = T;
    key.deterministic = deterministic ? 1 : 0;
    key.profile = e->profile;
    if (!p.injected) {
        key.n_hidden = actor->n_hidden;
        key.hidden = actor->hidden;
        key.act = actor->act;
        key.param_bytes = actor->param_bytes;
        key.ptrs[0] = actor->params;
    }
    const void* ptrs[] = {tr->obs, tr->act, tr->logp, tr->rew, tr->done, tr->mu, tr->dbg_aint,
                          tr->dbg_hold, tr->dbg_cash, injected_u, fitness_out, tr->val, tr->equity};
    for (int i = 0; i < 13; ++i) key.ptrs[1 + i] = ptrs[i];
    GraphEntry* hit = nullptr;
    for (auto& g : e->graphs)
        if (memcmp(&g.key, &key, sizeof(key)) == 0) hit = &g;
    if (!hit) {
        cudaGraph_t graph;
        ProfEvents* prof = nullptr;
        if (e->profile) {
            prof = new ProfEvents();
            pod_status pst = prof->create(T, e->profile, p.injected, e->groups, group_fracs(e));
            if (pst) {
                prof->destroy();
                delete prof;
                return pst;
            }
        }
        POD_CUDA(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
        pod_status st = enqueue_rollout(e, p, T, tr, injected_u, fitness_out, e->cap_stream, prof);
        cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &graph);
        if (st) return st;
        if (ce != cudaSuccess) return pod_fail(POD_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
        cudaGraphExec_t exec;
        ce = cudaGraphInstantiate(&exec, graph, 0);
        const unsigned long long kn = pod_graph_kernel_nodes(graph);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return pod_fail(POD_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
        if (e->graphs.size() >= 8) {
            size_t victim = 0;
            for (size_t i = 1; i < e->graphs.size(); ++i)
                if (e->graphs[i].last_use < e->graphs[victim].last_use) victim = i;
            cudaGraphExecDestroy(e->graphs[victim].exec);
            if (e->graphs[victim].prof) {
                e->graphs[victim].prof->destroy();
                delete e->graphs[victim].prof;
            }
            e->graphs.erase(e->graphs.begin() + static_cast<long>(victim));
        }
        e->graphs.push_back(GraphEntry{key, exec, 0, prof, kn});
        hit = &e->graphs.back();
    }
    hit->last_use = ++e->use_clock;
    e->last_prof = hit->prof;
    POD_CUDA(cudaGraphLaunch(hit->exec, s));
    pod_note_graph_launch(hit->kernels);
    return POD_OK;
}

extern "C" pod_status pod_debug_trace(pod_env_t* e, unsigned long long* actor_buf, unsigned long long* env_buf) {
    if (!e) return pod_fail(POD_ERR_ARG, "env is NULL");
    e->trace = actor_buf;
    e->env_trace = env_buf;
    for (auto& g : e->graphs) cudaGraphExecDestroy(g.exec);
    e->graphs.clear();
    return POD_OK;
}

extern "C" pod_status pod_env_profile(pod_env_t* e, int32_t enable) {
    if (!e) return pod_fail(POD_ERR_ARG, "env is NULL");
    if (enable < 0) return pod_fail(POD_ERR_ARG, "profile stride must be >= 0");
    e->profile = enable;
    e->last_prof = nullptr;
    return POD_OK;
}

extern "C" pod_status pod_env_profile_read(pod_env_t* e, double* actor_ms, double* actor_units, double* env_ms,
                                           double* env_units, void* stream) {
    if (!e || !actor_ms || !actor_units || !env_ms || !env_units) return pod_fail(POD_ERR_ARG, "NULL argument");
    *actor_ms = *env_ms = 0.0;
    *actor_units = *env_units = 0.0;
    ProfEvents* p = e->last_prof;
    if (!p) return POD_OK;
    POD_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    double a = 0.0, v = 0.0, u = 0.0;
    for (int m = 0; m < p->n_marked; ++m) {
        for (int g = 0; g < p->groups; ++g) {
            const size_t b = static_cast<size_t>(4 * (m * p->groups + g));
            float ms = 0.f;
            POD_CUDA(cudaEventElapsedTime(&ms, p->ev[b], p->ev[b + 1]));
            a += ms;
            POD_CUDA(cudaEventElapsedTime(&ms, p->ev[b + 2], p->ev[b + 3]));
            v += ms;
            u += p->frac[static_cast<size_t>(g)];
        }
    }
    *actor_ms = a;
    *env_ms = v;
    *actor_units = u;
    *env_units = u;
    e->last_prof = nullptr;
    return POD_OK;
}

extern "C" pod_status pod_env_fitness(pod_env_t* e, double* fitness_out, void* stream) {
    if (!e || !fitness_out) return pod_fail(POD_ERR_ARG, "env and fitness_out must be non-NULL");
    fitness_kernel<<<e->cfg.n_agents, 1024, 0, static_cast<cudaStream_t>(stream)>>>(e->ep_ret, e->per_agent, fitness_out);
    pod_note_launch(static_cast<cudaStream_t>(stream));
    POD_CUDA(cudaGetLastError());
    return POD_OK;
}

extern "C" pod_status pod_env_check(pod_env_t* e, void* stream) {
    if (!e) return pod_fail(POD_ERR_ARG, "env is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t h = 0;
    POD_CUDA(cudaStreamSynchronize(s));
    POD_CUDA(cudaMemcpy(&h, e->err, 4, cudaMemcpyDeviceToHost));
    *static_cast<volatile uint32_t*>(e->h_err) = 0;
    if (h) {
        POD_CUDA(cudaMemset(e->err, 0, 4));
        return pod_fail(POD_ERR_NONFINITE, "device error word 0x%x (1 = non-finite actor mean, 2 = non-finite account value)", h);
    }
    return POD_OK;
}

extern "C" pod_status pod_env_read_state(pod_env_t* e, int32_t* hold, double* cash, double* asset, double* ep_ret,
                                         void* stream) {
    if (!e) return pod_fail(POD_ERR_ARG, "env is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int N = e->cfg.n_envs, n = e->cfg.n_stocks;
    if (hold) {
        const int64_t tot = static_cast<int64_t>(N) * n;
        hold_transpose_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(e->hold, N, n, hold);
        pod_note_launch(s);
        POD_CUDA(cudaGetLastError());
    }
    if (cash) POD_CUDA(cudaMemcpyAsync(cash, e->cash, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    if (asset) POD_CUDA(cudaMemcpyAsync(asset, e->asset, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    if (ep_ret) POD_CUDA(cudaMemcpyAsync(ep_ret, e->ep_ret, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    return pod_env_check(e, stream);
}

// ------------------------------------------------------------ GAE
static pod_status gae_launch(const float* rew, const float* val, const uint8_t* done, const float* boot, int32_t T,
                             int32_t N, float gamma, float lambda, float* adv, float* ret, double* stats,
                             cudaStream_t stream, bool* normalized);

extern "C" pod_status pod_gae(const float* rew, const float* val, const uint8_t* done, const float* boot, int32_t T,
                              int32_t N, float gamma, float lambda, float* adv, float* ret, double* adv_stats,
                              void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (adv_stats && reinterpret_cast<uintptr_t>(adv_stats) % 8 != 0)
        return pod_fail(POD_ERR_ARG, "adv_stats must be 8-byte aligned");
    bool normalized = false;
    pod_status st = gae_launch(rew, val, done, boot, T, N, gamma, lambda, adv, ret, adv_stats, s, &normalized);
    if (st || !adv_stats || normalized) return st;
    const int64_t count = static_cast<int64_t>(T) * N;
    const int64_t want = (count / 4 + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < 148 * 16 ? (want > 0 ? want : 1) : 148 * 16);
    adv_normalize_kernel<<<blocks, 256, 0, s>>>(adv, count, adv_stats, reinterpret_cast<uintptr_t>(adv) % 16 == 0);
    pod_note_launch(s);
    POD_CUDA(cudaGetLastError());
    return POD_OK;
}

static pod_status gae_launch(const float* rew, const float* val, const uint8_t* done, const float* boot, int32_t T,
                             int32_t N, float gamma, float lambda, float* adv, float* ret, double* stats,
                             cudaStream_t stream, bool* normalized) {
    *normalized = false;
    if (!rew || !val || !done || !boot || !adv || !ret) return pod_fail(POD_ERR_ARG, "GAE pointers must be non-NULL");
    if (T < 1 || N < 1) return pod_fail(POD_ERR_ARG, "T and N must be >= 1");
    if (static_cast<int64_t>(T) * N >= (1ll << 40)) return pod_fail(POD_ERR_SHAPE, "T * N too large");
    pod_status st = pod_require_sm100();
    if (st) return st;
    auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
    // Tensor-map encoding costs several microseconds of host time per map; a rollout loop calls pod_gae on the
    // same trajectory buffers every iteration, so the last few encodings are cached by (pointers, T, N).
    struct GaeCacheEntry {
        const void *r, *v, *d;
        int32_t T, N, use_bulk;
        GaeMaps maps;
    };
    static std::mutex cache_mu;
    static GaeCacheEntry cache[4];
    static int cache_next = 0;
    GaeMaps maps;
    memset(&maps, 0, sizeof(maps));
    int use_bulk = (N % 16 == 0) && al(rew) && al(val) && al(done) ? 1 : 0;
    if (use_bulk) {
        std::lock_guard<std::mutex> lk(cache_mu);
        bool hit = false;
        for (const GaeCacheEntry& c : cache)
            if (c.r == rew && c.v == val && c.d == done && c.T == T && c.N == N) {
                maps = c.maps;
                use_bulk = c.use_bulk;
                hit = true;
                break;
            }
        if (!hit) {
            const uint64_t dims[2] = {static_cast<uint64_t>(N), static_cast<uint64_t>(T)};
            const uint64_t s4[1] = {static_cast<uint64_t>(N) * 4}, s1[1] = {static_cast<uint64_t>(N)};
            const uint32_t box[2] = {32, GAE_L};
            if (encode_plain(&maps.r, rew, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, dims, s4, box) ||
                encode_plain(&maps.v, val, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, dims, s4, box) ||
                encode_plain(&maps.d, done, CU_TENSOR_MAP_DATA_TYPE_UINT8, dims, s1, box))
                use_bulk = 0;
            cache[cache_next] = GaeCacheEntry{rew, val, done, T, N, use_bulk, maps};
            cache_next = (cache_next + 1) % 4;
        }
    }
    const int groups = (N + 31) / 32;
    // Few column groups (under four per SM): split time across the warps of a block (gae_seg_kernel), as long
    // as the [T x 32] slab fits in shared memory.  POD_GAE_PATH=seq|seg forces a path (tests compare both).
    const int nchunks = (T + GAE_L - 1) / GAE_L;
    bool seg_ok = use_bulk && nchunks <= 20;
    bool use_seg = seg_ok && groups < 4 * 148;
    if (const char* f = getenv("POD_GAE_PATH")) {
        if (!strcmp(f, "seq")) use_seg = false;
        if (!strcmp(f, "seg")) use_seg = seg_ok;
    }
    if (use_seg) {
        const int cpw = nchunks <= GAE_SEG_MAX ? 1 : GAE_CPW_MAX;
        const int seg = (nchunks + cpw - 1) / cpw;
        const int want = static_cast<int>(gae_seg_smem_bytes(seg, cpw));
        // the opt-in is a per-device function attribute: track what each device has been granted
        static std::mutex seg_mu;
        static int seg_attr[64] = {};   // dynamic shared memory granted so far, per device ordinal
        int cur_dev = 0;
        POD_CUDA(cudaGetDevice(&cur_dev));
        if (cur_dev < 0 || cur_dev >= 64) return pod_fail(POD_ERR_UNSUPPORTED, "device ordinal %d >= 64", cur_dev);
        {
            std::lock_guard<std::mutex> lk(seg_mu);
            if (seg_attr[cur_dev] < want) {
                cudaError_t ce = cudaFuncSetAttribute(gae_seg_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
                if (ce == cudaSuccess)
                    ce = cudaFuncSetAttribute(gae_seg_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
                if (ce != cudaSuccess) {
                    cudaFuncAttributes fa;
                    memset(&fa, 0, sizeof(fa));
                    cudaError_t ce2 = cudaFuncGetAttributes(&fa, gae_seg_kernel<false>);
                    int dev = 0, optin = 0;
                    cudaGetDevice(&dev);
                    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
                    return pod_fail(POD_ERR_CUDA,
                                    "gae_seg_kernel smem attribute %d B: %s (getattr %s: static %zu B, max dyn %d B, "
                                    "max threads %d, regs %d; device opt-in %d B)",
                                    want, cudaGetErrorString(ce), cudaGetErrorString(ce2), fa.sharedSizeBytes,
                                    fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock, fa.numRegs, optin);
                }
                seg_attr[cur_dev] = want;
            }
        }
        if (stats) {
            // normalisation fused in when every block fits on the device at once (cooperative launch)
            int per_sm = 0, sms = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_seg_kernel<true>, 32 * seg,
                                                          gae_seg_smem_bytes(seg, cpw));
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur_dev);
            static const bool fuse_off = [] {   // experiments: POD_GAE_FUSED_NORM=0 keeps the separate pass
                const char* v = getenv("POD_GAE_FUSED_NORM");
                return v && v[0] == '0';
            }();
            if (!fuse_off && per_sm * sms >= groups) {
                cudaLaunchConfig_t lc{};
                lc.gridDim = dim3(static_cast<unsigned>(groups));
                lc.blockDim = dim3(static_cast<unsigned>(32 * seg));
                lc.dynamicSmemBytes = gae_seg_smem_bytes(seg, cpw);
                lc.stream = stream;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                lc.attrs = at;
                lc.numAttrs = 1;
                POD_CUDA(cudaLaunchKernelEx(&lc, gae_seg_kernel<true>, maps, boot, T, N, gamma, lambda, adv, ret, cpw,
                                            stats));
                pod_note_launch(stream);
                *normalized = true;
                return POD_OK;
            }
            POD_CUDA(cudaMemsetAsync(stats, 0, 2 * sizeof(double), stream));
        }
        gae_seg_kernel<false><<<static_cast<unsigned>(groups), 32 * seg, gae_seg_smem_bytes(seg, cpw), stream>>>(
            maps, boot, T, N, gamma, lambda, adv, ret, cpw, stats);
        pod_note_launch(stream);
        POD_CUDA(cudaGetLastError());
        return POD_OK;
    }
    if (stats) POD_CUDA(cudaMemsetAsync(stats, 0, 2 * sizeof(double), stream));
    const unsigned blocks = static_cast<unsigned>((groups + GAE_WARPS - 1) / GAE_WARPS);
    {
        // per-device opt-in (pod_gae may run on any device without an env handle there)
        static std::mutex gae_mu;
        static bool gae_attr[64] = {};
        int cur_dev = 0;
        POD_CUDA(cudaGetDevice(&cur_dev));
        if (cur_dev < 0 || cur_dev >= 64) return pod_fail(POD_ERR_UNSUPPORTED, "device ordinal %d >= 64", cur_dev);
        std::lock_guard<std::mutex> lk(gae_mu);
        if (!gae_attr[cur_dev]) {
            POD_CUDA(cudaFuncSetAttribute(gae_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(gae_smem_bytes())));
            gae_attr[cur_dev] = true;
        }
    }
    gae_kernel<<<blocks, 32 * GAE_WARPS, gae_smem_bytes(), stream>>>(maps, rew, val, done, boot, T, N, gamma, lambda,
                                                                       adv, ret, use_bulk, stats);
    pod_note_launch(stream);
    POD_CUDA(cudaGetLastError());
    return POD_OK;
}

// ------------------------------------------------------------ K-pod ensemble fusion (R#24)
// the parts of fuse_x_kernel's arguments that depend only on the slab layout
static pod_status fuse_x_common(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden, size_t param_bytes,
                                int32_t P_local, int32_t K_local, float tau, int32_t R, FuseXArgs* a) {
    if (K_local < 1 || P_local < 1 || P_local % K_local != 0)
        return pod_fail(POD_ERR_ARG, "P_local (%d) must be a positive multiple of K_local (%d)", P_local, K_local);
    if (!(tau >= 0.0f && tau <= 1.0f)) return pod_fail(POD_ERR_ARG, "tau must be in [0, 1]");
    if (R < 1 || R > FUSE_MAX_RANKS) return pod_fail(POD_ERR_ARG, "ranks must be in [1, %d]", FUSE_MAX_RANKS);
    pod_actor_layout L;
    pod_status st = pod_actor_layout_get(cfg, n_hidden, hidden, &L);
    if (st) return st;
    if (param_bytes < L.param_bytes || param_bytes % 16 != 0)
        return pod_fail(POD_ERR_SHAPE, "param_bytes %zu must be >= %zu and a multiple of 16", param_bytes, L.param_bytes);
    memset(a, 0, sizeof(*a));
    uint64_t flat = 0;
    int ns = 0;
    for (int l = 0; l < L.n_layers; ++l) {
        a->seg[ns++] = FuseSeg{L.w_offset[l], flat, static_cast<uint32_t>(L.w_rows[l]) * L.w_cols[l], 1u};
        flat += static_cast<uint64_t>(L.w_rows[l]) * L.w_cols[l];
    }
    for (int l = 0; l < L.n_layers; ++l) {
        a->seg[ns++] = FuseSeg{L.b_offset[l], flat, static_cast<uint32_t>(L.w_rows[l]), 0u};
        flat += static_cast<uint64_t>(L.w_rows[l]);
    }
    a->seg[ns++] = FuseSeg{L.log_std_offset, flat, static_cast<uint32_t>(L.n_out_pad), 0u};
    flat += static_cast<uint64_t>(L.n_out_pad);
    a->n_seg = ns;
    a->K_local = K_local;
    a->n_elems = static_cast<int64_t>(flat);
    a->param_bytes = param_bytes;
    a->scale = 1.0f / static_cast<float>(K_local * R);
    a->tau = tau;
    a->R = R;
    a->A_local = P_local / K_local;
    a->nchunks = (a->n_elems + FUSE_CHUNK - 1) / FUSE_CHUNK;
    if (a->n_elems % 8 != 0) return pod_fail(POD_ERR_SHAPE, "flat parameter count must be a multiple of 8");
    return pod_require_sm100();
}

// resident blocks of fuse_x_kernel on this device (every block of an R-rank launch must be resident)
static int fuse_x_capacity() {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fuse_x_kernel, 256, 0);
    return sms * (per > 0 ? per : 1);
}

extern "C" pod_status pod_fuse_pods(pod_comm_t* comm, const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                                    void* params, size_t param_bytes, int32_t P_local, int32_t K_local, float tau,
                                    float* prev, float* work, void* stream) {
    (void)work;   // no float32 work vector: the exchange happens inside fuse_x_kernel
    if (!params) return pod_fail(POD_ERR_ARG, "params must be non-NULL");
    if (!prev && tau != 1.0f) return pod_fail(POD_ERR_ARG, "prev is required when tau < 1");
    if (reinterpret_cast<uintptr_t>(params) % 16 != 0 || (prev && reinterpret_cast<uintptr_t>(prev) % 16 != 0))
        return pod_fail(POD_ERR_ARG, "params and prev must be 16-byte aligned");
    const int nranks = comm ? pod_comm_size(comm) : 1;
    FuseXArgs a;
    pod_status st = fuse_x_common(cfg, n_hidden, hidden, param_bytes, P_local, K_local, tau, nranks, &a);
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int me = comm ? pod_comm_rank(comm) : 0;
    a.my_rank = me;
    a.params[me] = static_cast<char*>(params);
    a.prev[me] = prev;
    a.epoch = 1;
    if (nranks > 1) {
        float* stage[FUSE_MAX_RANKS];
        uint32_t *flag[FUSE_MAX_RANKS], *ack[FUSE_MAX_RANKS];
        const size_t nflags = static_cast<size_t>(a.A_local) * a.nchunks;
        st = pod_comm_fuse_buffers(comm, static_cast<size_t>(a.A_local) * a.n_elems, nflags, stage, flag, ack, &a.epoch, s);
        if (st) return st;
        for (int q = 0; q < nranks; ++q) {
            a.stage[q] = stage[q];
            a.flag[q] = flag[q];
            a.ack[q] = ack[q];
        }
    }
    const int64_t chunks = static_cast<int64_t>(a.A_local) * a.nchunks;
    const unsigned X = static_cast<unsigned>(std::min<int64_t>(chunks, fuse_x_capacity()));
    fuse_x_kernel<<<dim3(X, 1), 256, 0, s>>>(a);
    pod_note_launch(s);
    POD_CUDA(cudaGetLastError());
    return POD_OK;
}

extern "C" pod_status pod_fuse_workspace_size(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                                              int32_t P_local, int32_t K_local, int32_t R, size_t* bytes) {
    if (!bytes) return pod_fail(POD_ERR_ARG, "bytes is NULL");
    pod_actor_layout L;
    pod_status st = pod_actor_layout_get(cfg, n_hidden, hidden, &L);
    if (st) return st;
    if (K_local < 1 || P_local < 1 || P_local % K_local != 0 || R < 1 || R > FUSE_MAX_RANKS)
        return pod_fail(POD_ERR_ARG, "bad P_local / K_local / R");
    const size_t A = static_cast<size_t>(P_local / K_local), ne = L.n_elems;
    const size_t nch = (ne + FUSE_CHUNK - 1) / FUSE_CHUNK;
    *bytes = static_cast<size_t>(R) * (round_up(A * ne * 4, 256) + round_up(2 * A * nch * 4, 256));
    return POD_OK;
}

extern "C" pod_status pod_fuse_pods_local_ranks(const pod_env_config* cfg, int32_t n_hidden, int32_t hidden,
                                                void* const* params, size_t param_bytes, int32_t R, int32_t P_local,
                                                int32_t K_local, float tau, float* const* prev, void* ws,
                                                size_t ws_bytes, void* stream) {
    if (!params || !ws) return pod_fail(POD_ERR_ARG, "params and ws must be non-NULL");
    if (!prev && tau != 1.0f) return pod_fail(POD_ERR_ARG, "prev is required when tau < 1");
    FuseXArgs a;
    pod_status st = fuse_x_common(cfg, n_hidden, hidden, param_bytes, P_local, K_local, tau, R, &a);
    if (st) return st;
    size_t need = 0;
    st = pod_fuse_workspace_size(cfg, n_hidden, hidden, P_local, K_local, R, &need);
    if (st) return st;
    if (ws_bytes < need || reinterpret_cast<uintptr_t>(ws) % 256 != 0)
        return pod_fail(POD_ERR_WORKSPACE, "workspace needs %zu bytes, 256-byte aligned", need);
    const size_t A = static_cast<size_t>(a.A_local);
    const size_t sb = round_up(A * a.n_elems * 4, 256), fb = round_up(2 * A * a.nchunks * 4, 256);
    char* w = static_cast<char*>(ws);
    for (int q = 0; q < R; ++q) {
        if (!params[q] || reinterpret_cast<uintptr_t>(params[q]) % 16 != 0)
            return pod_fail(POD_ERR_ARG, "params[%d] must be non-NULL and 16-byte aligned", q);
        a.params[q] = static_cast<char*>(params[q]);
        a.prev[q] = prev ? prev[q] : nullptr;
        if (a.prev[q] && reinterpret_cast<uintptr_t>(a.prev[q]) % 16 != 0)
            return pod_fail(POD_ERR_ARG, "prev[%d] must be 16-byte aligned", q);
        char* b = w + static_cast<size_t>(q) * (sb + fb);
        a.stage[q] = reinterpret_cast<float*>(b);
        a.flag[q] = reinterpret_cast<uint32_t*>(b + sb);
        a.ack[q] = reinterpret_cast<uint32_t*>(b + sb) + A * a.nchunks;
    }
    a.my_rank = -1;   // block row y plays rank y
    a.epoch = 1;
    const int cap = fuse_x_capacity();
    if (cap < R) return pod_fail(POD_ERR_UNSUPPORTED, "%d ranks exceed the resident blocks of the device", R);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int q = 0; q < R; ++q) POD_CUDA(cudaMemsetAsync(a.flag[q], 0, fb, s));   // flags and acks: epoch 1 from zero
    const int64_t chunks = static_cast<int64_t>(A) * a.nchunks;
    const unsigned X = static_cast<unsigned>(std::min<int64_t>(chunks, cap / R));
    fuse_x_kernel<<<dim3(X, static_cast<unsigned>(R)), 256, 0, s>>>(a);
    pod_note_launch(s);
    POD_CUDA(cudaGetLastError());
    return POD_OK;
}

// ------------------------------------------------------------ evaluator (R#25)
extern "C" pod_status pod_backtest_metrics(const double* v0, const double* curve, int32_t T, int32_t N,
                                           double periods_per_year, double rf_per_period, double* out, void* stream) {
    if (!v0 || !curve || !out) return pod_fail(POD_ERR_ARG, "v0, curve and out must be non-NULL");
    if (T < 1 || N < 1) return pod_fail(POD_ERR_ARG, "T and N must be >= 1");
    if (!(periods_per_year > 0.0)) return pod_fail(POD_ERR_ARG, "periods_per_year must be > 0");
    pod_status st = pod_require_sm100();
    if (st) return st;
    backtest_metrics_kernel<<<static_cast<unsigned>((N + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        v0, curve, T, N, periods_per_year, rf_per_period, out);
    pod_note_launch(static_cast<cudaStream_t>(stream));
    POD_CUDA(cudaGetLastError());
    return POD_OK;
}

extern "C" pod_status pod_early_stop(const double* history, int32_t len, int32_t patience, int32_t* stop,
                                     int32_t* best) {
    if (!history || !stop || !best) return pod_fail(POD_ERR_ARG, "NULL argument");
    if (len < 1) return pod_fail(POD_ERR_ARG, "history is empty");
    if (patience < 0) return pod_fail(POD_ERR_ARG, "patience must be >= 0");
    int b = 0;
    for (int i = 1; i < len; ++i)
        if (history[i] > history[b]) b = i;   // strict: the earliest maximum wins
    *best = b;
    *stop = (len - 1 - b) >= patience ? 1 : 0;
    return POD_OK;
}

#include "pod_ppo.cuh"

#ifdef POD_EXP_GTIME
extern "C" int pod_debug_gtime(unsigned long long* host, int reset) {
    if (reset) {
        static unsigned long long init[1024][4];
        for (int i = 0; i < 1024; ++i) { init[i][0] = ~0ull; init[i][1] = 0; init[i][2] = ~0ull; init[i][3] = 0; }
        return cudaMemcpyToSymbol(pod::g_gtime, init, sizeof(init)) == cudaSuccess ? 0 : 1;
    }
    return cudaMemcpyFromSymbol(host, pod::g_gtime, sizeof(unsigned long long) * 1024 * 4) == cudaSuccess ? 0 : 1;
}
extern "C" int pod_debug_ftime(unsigned long long* host) {
    return cudaMemcpyFromSymbol(host, pod::g_ftime, sizeof(unsigned long long) * 1024 * 12) == cudaSuccess ? 0 : 1;
}
#endif
