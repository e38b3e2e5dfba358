// pod_elite.cpp — generational-evolution selector on the host
// plus its NCCL exchange: fitness all-gather and elite parameter-slab moves
// ("sending the network parameters rather than the gradients").
// libnccl.so.2 is dlopen'ed at pod_comm_init (the copy torch already loaded
// when present), so libpod.so itself loads on machines without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "pod.h"
#include "pod_internal.h"

extern "C" pod_status pod_elite_plan(const double* fitness, int32_t P, int32_t k, int32_t* plan) {
    if (!fitness || !plan) return pod_fail(POD_ERR_ARG, "fitness and plan must be non-NULL");
    if (P < 1) return pod_fail(POD_ERR_ARG, "empty population (S:L454)");
    if (k < 1 || k > P) return pod_fail(POD_ERR_ARG, "k=%d outside [1, %d]", k, P);
    for (int g = 0; g < P; ++g)
        if (!std::isfinite(fitness[g])) return pod_fail(POD_ERR_NONFINITE, "fitness of agent %d is not finite", g);
    std::vector<int32_t> order(static_cast<size_t>(P));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        if (fitness[x] != fitness[y]) return fitness[x] > fitness[y];
        return x < y;
    });
    std::vector<char> elite(static_cast<size_t>(P), 0);
    for (int r = 0; r < k; ++r) elite[static_cast<size_t>(order[r])] = 1;
    int next = 0;
    for (int g = 0; g < P; ++g) plan[g] = elite[static_cast<size_t>(g)] ? g : order[(next++) % k];
    return POD_OK;
}

extern "C" pod_status pod_elite_transfers(const int32_t* plan, int32_t P, int32_t P_local, int32_t rank,
                                          pod_transfer* ops, int32_t max_ops, int32_t* n_ops) {
    if (!plan || !n_ops || (max_ops > 0 && !ops)) return pod_fail(POD_ERR_ARG, "NULL argument");
    if (P < 1 || P_local < 1 || P % P_local != 0) return pod_fail(POD_ERR_ARG, "P_total must be a multiple of P_local");
    if (rank < 0 || rank >= P / P_local) return pod_fail(POD_ERR_ARG, "rank out of range");
    for (int g = 0; g < P; ++g) {
        const int s = plan[g];
        if (s < 0 || s >= P || plan[s] != s) return pod_fail(POD_ERR_ARG, "plan[%d]=%d is not an elite slot", g, s);
    }
    // An elite slab crosses to a remote rank at most once per (elite, destination rank): the first
    // eliminated slot of that rank which takes the elite (ascending slot order, the same walk on every
    // rank, so sends and receives pair up in order) receives it; the rank's later slots taking the same
    // elite are filled by a local copy from that slot once the exchange has landed (kind 3).
    int cnt = 0;
    auto emit = [&](pod_transfer op) -> bool {
        if (cnt >= max_ops) return false;
        ops[cnt++] = op;
        return true;
    };
    std::vector<int32_t> landed(static_cast<size_t>(P) * (P / P_local), -1);   // [src][dest rank] -> local slot
    // pass 0: local copies of local elites (kind 0)
    for (int g = rank * P_local; g < (rank + 1) * P_local; ++g) {
        const int src = plan[g];
        if (src != g && src / P_local == rank && !emit(pod_transfer{0, rank, src % P_local, g % P_local}))
            return pod_fail(POD_ERR_ARG, "max_ops %d too small", max_ops);
    }
    // pass 1: sends (1) and receives (2), ascending slot order over the whole population
    for (int g = 0; g < P; ++g) {
        const int src = plan[g];
        if (src == g) continue;
        const int dr = g / P_local, sr = src / P_local;
        if (dr == sr) continue;
        int32_t& first = landed[static_cast<size_t>(src) * (P / P_local) + dr];
        if (first >= 0) continue;   // this rank already receives the elite: fanned out in pass 2
        first = g % P_local;
        if (sr == rank && !emit(pod_transfer{1, dr, src % P_local, -1}))
            return pod_fail(POD_ERR_ARG, "max_ops %d too small", max_ops);
        if (dr == rank && !emit(pod_transfer{2, sr, -1, g % P_local}))
            return pod_fail(POD_ERR_ARG, "max_ops %d too small", max_ops);
    }
    // pass 2: local fan-out of received slabs (kind 3), after the exchange
    for (int g = rank * P_local; g < (rank + 1) * P_local; ++g) {
        const int src = plan[g];
        if (src == g || src / P_local == rank) continue;
        const int32_t first = landed[static_cast<size_t>(src) * (P / P_local) + rank];
        if (first != g % P_local && !emit(pod_transfer{3, src / P_local, first, g % P_local}))
            return pod_fail(POD_ERR_ARG, "max_ops %d too small", max_ops);
    }
    *n_ops = cnt;
    return POD_OK;
}

// ------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api.h ? &api : nullptr;
    tried = true;
    const char* env = getenv("POD_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
        if (!nm || !nm[0]) continue;
        api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
    }
    if (!api.h) return nullptr;
#define LOAD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
    LOAD(GetUniqueId);
    LOAD(CommInitRank);
    LOAD(CommDestroy);
    LOAD(AllGather);
    LOAD(Send);
    LOAD(Recv);
    LOAD(GroupStart);
    LOAD(GroupEnd);
    LOAD(GetErrorString);
#undef LOAD
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.Send || !api.Recv ||
        !api.GroupStart || !api.GroupEnd) {
        api.h = nullptr;
        return nullptr;
    }
    return &api;
}
}  // namespace

struct pod_comm {
    ncclComm_t comm;
    int nranks, rank, max_local;
    double* d_all;
    double* h_all;
    std::vector<pod_transfer> ops;
    // fused fusion (pod_comm_fuse_buffers): this rank's buffer and every rank's mapping of theirs
    void* fx_base = nullptr;
    size_t fx_bytes = 0, fx_stage = 0;
    std::vector<void*> fx_peer;   // [nranks], own entry = fx_base
    uint32_t fx_epoch = 0;
};

#define NCCL_TRY(call)                                                                                        \
    do {                                                                                                      \
        ncclResult_t _r = (call);                                                                             \
        if (_r != ncclSuccess)                                                                                \
            return pod_fail(POD_ERR_NCCL, "%s: %s", #call, api->GetErrorString ? api->GetErrorString(_r) : "?"); \
    } while (0)

extern "C" pod_status pod_comm_unique_id(uint8_t id[128]) {
    if (!id) return pod_fail(POD_ERR_ARG, "id is NULL");
    NcclApi* api = nccl();
    if (!api) return pod_fail(POD_ERR_NCCL, "libnccl.so.2 could not be loaded (set POD_NCCL_LIB)");
    ncclUniqueId u;
    NCCL_TRY(api->GetUniqueId(&u));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id, &u, 128);
    return POD_OK;
}

extern "C" pod_status pod_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t max_local,
                                    pod_comm_t** out) {
    if (!id || !out) return pod_fail(POD_ERR_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks || max_local < 1) return pod_fail(POD_ERR_ARG, "bad nranks/rank/max_local");
    pod_status st = pod_require_sm100();
    if (st) return st;
    NcclApi* api = nccl();
    if (!api) return pod_fail(POD_ERR_NCCL, "libnccl.so.2 could not be loaded (set POD_NCCL_LIB)");
    ncclUniqueId u;
    memcpy(&u, id, 128);
    pod_comm* c = new pod_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->max_local = max_local;
    ncclResult_t r = api->CommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return pod_fail(POD_ERR_NCCL, "ncclCommInitRank: %s", api->GetErrorString ? api->GetErrorString(r) : "?");
    }
    const size_t total = static_cast<size_t>(nranks) * max_local;
    if (cudaMalloc(&c->d_all, total * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&c->h_all, total * sizeof(double)) != cudaSuccess) {
        api->CommDestroy(c->comm);
        delete c;
        return pod_fail(POD_ERR_CUDA, "pod_comm_init: allocation failed");
    }
    c->ops.resize(2 * total + 2);
    *out = c;
    return POD_OK;
}

static void fx_release(pod_comm_t* c) {
    for (int q = 0; q < static_cast<int>(c->fx_peer.size()); ++q)
        if (q != c->rank && c->fx_peer[static_cast<size_t>(q)]) cudaIpcCloseMemHandle(c->fx_peer[static_cast<size_t>(q)]);
    c->fx_peer.clear();
    if (c->fx_base) cudaFree(c->fx_base);
    c->fx_base = nullptr;
    c->fx_bytes = c->fx_stage = 0;
}

extern "C" pod_status pod_comm_destroy(pod_comm_t* c) {
    if (!c) return POD_OK;
    fx_release(c);
    NcclApi* api = nccl();
    if (api && api->CommDestroy) api->CommDestroy(c->comm);
    cudaFree(c->d_all);
    cudaFreeHost(c->h_all);
    delete c;
    return POD_OK;
}

extern "C" pod_status pod_select_elite(pod_comm_t* c, const double* fitness_local, int32_t P_local, int32_t k,
                                       void* params, size_t param_bytes, int32_t* h_plan, void* stream) {
    if (!c || !fitness_local || !params || !h_plan) return pod_fail(POD_ERR_ARG, "NULL argument");
    if (P_local < 1 || P_local > c->max_local) return pod_fail(POD_ERR_ARG, "P_local must be in [1, %d]", c->max_local);
    if (param_bytes == 0) return pod_fail(POD_ERR_ARG, "param_bytes must be > 0");
    NcclApi* api = nccl();
    if (!api) return pod_fail(POD_ERR_NCCL, "NCCL not loaded");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int P = c->nranks * P_local;
    NCCL_TRY(api->AllGather(fitness_local, c->d_all, static_cast<size_t>(P_local), ncclFloat64, c->comm, s));
    if (cudaMemcpyAsync(c->h_all, c->d_all, sizeof(double) * P, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return pod_fail(POD_ERR_CUDA, "fitness D2H failed");
    pod_status st = pod_elite_plan(c->h_all, P, k, h_plan);
    if (st) return st;
    int32_t nops = 0;
    st = pod_elite_transfers(h_plan, P, P_local, c->rank, c->ops.data(), static_cast<int32_t>(c->ops.size()), &nops);
    if (st) return st;
    char* base = static_cast<char*>(params);
    for (int i = 0; i < nops; ++i) {
        const pod_transfer& op = c->ops[static_cast<size_t>(i)];
        if (op.kind == 0 &&
            cudaMemcpyAsync(base + op.dst_local * param_bytes, base + op.src_local * param_bytes, param_bytes,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return pod_fail(POD_ERR_CUDA, "local elite copy failed");
    }
    bool any_p2p = false;
    for (int i = 0; i < nops; ++i) any_p2p |= c->ops[static_cast<size_t>(i)].kind == 1 || c->ops[static_cast<size_t>(i)].kind == 2;
    if (any_p2p) {
        NCCL_TRY(api->GroupStart());
        for (int i = 0; i < nops; ++i) {
            const pod_transfer& op = c->ops[static_cast<size_t>(i)];
            if (op.kind == 1)
                NCCL_TRY(api->Send(base + op.src_local * param_bytes, param_bytes, ncclUint8, op.peer, c->comm, s));
            else if (op.kind == 2)
                NCCL_TRY(api->Recv(base + op.dst_local * param_bytes, param_bytes, ncclUint8, op.peer, c->comm, s));
        }
        NCCL_TRY(api->GroupEnd());
    }
    for (int i = 0; i < nops; ++i) {   // fan-out of received slabs, stream-ordered after the receives
        const pod_transfer& op = c->ops[static_cast<size_t>(i)];
        if (op.kind == 3 &&
            cudaMemcpyAsync(base + op.dst_local * param_bytes, base + op.src_local * param_bytes, param_bytes,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return pod_fail(POD_ERR_CUDA, "elite fan-out copy failed");
    }
    return POD_OK;
}

int pod_comm_size(const pod_comm_t* c) { return c ? c->nranks : 1; }
int pod_comm_rank(const pod_comm_t* c) { return c ? c->rank : 0; }

pod_status pod_comm_fuse_buffers(pod_comm_t* c, size_t stage_elems, size_t nflags, float** stage, uint32_t** flag,
                                 uint32_t** ack, uint32_t* epoch, cudaStream_t s) {
    NcclApi* api = nccl();
    if (!api) return pod_fail(POD_ERR_NCCL, "NCCL not loaded");
    const size_t stage_bytes = (stage_elems * sizeof(float) + 255) / 256 * 256;
    const size_t need = stage_bytes + 2 * nflags * sizeof(uint32_t);
    if (!c->fx_base || c->fx_bytes < need || c->fx_stage != stage_bytes) {
        // (re)build collectively: every rank reaches this with the same sizes (pod_fuse_pods is collective)
        fx_release(c);
        if (cudaMalloc(&c->fx_base, need) != cudaSuccess) return pod_fail(POD_ERR_CUDA, "fusion buffer allocation failed");
        if (cudaMemset(c->fx_base, 0, need) != cudaSuccess) return pod_fail(POD_ERR_CUDA, "fusion buffer clear failed");
        c->fx_bytes = need;
        c->fx_stage = stage_bytes;
        c->fx_epoch = 0;
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, c->fx_base) != cudaSuccess) return pod_fail(POD_ERR_CUDA, "cudaIpcGetMemHandle failed");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handles are 64 bytes");
        uint8_t* dh = nullptr;
        if (cudaMalloc(&dh, 64 * static_cast<size_t>(c->nranks + 1)) != cudaSuccess)
            return pod_fail(POD_ERR_CUDA, "handle exchange buffer allocation failed");
        std::vector<uint8_t> all(64 * static_cast<size_t>(c->nranks));
        cudaMemcpy(dh, &h, 64, cudaMemcpyHostToDevice);
        ncclResult_t r = api->AllGather(dh, dh + 64, 64, ncclUint8, c->comm, s);
        cudaError_t ce = r == ncclSuccess ? cudaStreamSynchronize(s) : cudaErrorUnknown;
        if (ce == cudaSuccess) ce = cudaMemcpy(all.data(), dh + 64, all.size(), cudaMemcpyDeviceToHost);
        cudaFree(dh);
        if (r != ncclSuccess) return pod_fail(POD_ERR_NCCL, "IPC handle all-gather failed");
        if (ce != cudaSuccess) return pod_fail(POD_ERR_CUDA, "IPC handle exchange: %s", cudaGetErrorString(ce));
        c->fx_peer.assign(static_cast<size_t>(c->nranks), nullptr);
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank) {
                c->fx_peer[static_cast<size_t>(q)] = c->fx_base;
                continue;
            }
            cudaIpcMemHandle_t hq;
            memcpy(&hq, all.data() + 64 * static_cast<size_t>(q), 64);
            if (cudaIpcOpenMemHandle(&c->fx_peer[static_cast<size_t>(q)], hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
                return pod_fail(POD_ERR_CUDA, "cudaIpcOpenMemHandle of rank %d failed (peer access over NVLink?)", q);
        }
    }
    for (int q = 0; q < c->nranks; ++q) {
        char* b = static_cast<char*>(c->fx_peer[static_cast<size_t>(q)]);
        stage[q] = reinterpret_cast<float*>(b);
        flag[q] = reinterpret_cast<uint32_t*>(b + stage_bytes);
        ack[q] = reinterpret_cast<uint32_t*>(b + stage_bytes + nflags * sizeof(uint32_t));
    }
    *epoch = ++c->fx_epoch;
    return POD_OK;
}

