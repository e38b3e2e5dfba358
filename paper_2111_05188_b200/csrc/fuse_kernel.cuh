// fuse_kernel.cuh — K-pod ensemble fusion of parameter slabs.
//
// Method ("fusing the trained models from K pods at each epoch"; P:L372 the pods exchange
// parameters, not gradients, "taking advantage of the soft update"; S:L302–310 soft_update,
// S:L364–372 fuse; reading R#24):
//   mean  = (1/K) sum over the K pods of the agent's parameters
//   fused = tau * mean + (1 - tau) * prev            (tau = 1: hard adoption of the mean)
//   every pod's parameters <- fused;  prev <- fused
// Slabs are the rollout's parameter format (pod_actor_layout: bf16 weight matrices, f32 biases and
// log-std).  Pods of one agent are K_local consecutive population slots on each of the
// communicator's ranks.  pod_fuse_pods runs fuse_x_kernel (end of this file): local sum, the exchange
// of the ranks' partial sums over peer memory, the rank-ordered global sum, the blend and the narrowing
// in one kernel per rank.  Arithmetic is float32 (sum in pod order on each rank, then in rank order,
// then the blend); the bf16 weights are rounded to nearest even once, at the end.  fuse_sum_kernel /
// fuse_blend_kernel are the single-rank pieces the PPO learner reuses (slab <-> float32 master).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace pod {

constexpr int FUSE_MAX_SEGS = 16;

struct FuseSeg {
    uint64_t slab_off;   // byte offset of the segment in a slab
    uint64_t flat_off;   // element offset in the float32 flat vector of one agent
    uint32_t count;      // elements
    uint32_t bf16;       // 1: bf16 elements, 0: f32
};

struct FuseArgs {
    FuseSeg seg[FUSE_MAX_SEGS];
    int32_t n_seg;
    int32_t K_local;           // pods of an agent on this rank (consecutive slots)
    int64_t n_elems;           // flat elements per agent
    uint64_t param_bytes;      // slab stride
    char* params;              // [A_local * K_local][param_bytes]
    float* work;               // [A_local][n_elems]
    float* prev;               // [A_local][n_elems] or null (tau == 1)
    float scale;               // 1 / K (all ranks)
    float tau;
};

__device__ __forceinline__ int fuse_find_seg(const FuseSeg* seg, int n_seg, int64_t idx, int64_t* off) {
    int s = 0;
    while (s + 1 < n_seg && static_cast<int64_t>(seg[s + 1].flat_off) <= idx) ++s;
    *off = idx - static_cast<int64_t>(seg[s].flat_off);
    return s;
}
__device__ __forceinline__ int fuse_find(const FuseArgs& a, int64_t idx, int64_t* off) {
    return fuse_find_seg(a.seg, a.n_seg, idx, off);
}

// 8 consecutive elements of a segment (every segment count and offset is a multiple of 8 elements,
// slab offsets are 128-B aligned): one 16-B load for bf16, two for f32
__device__ __forceinline__ void fuse_load8(const char* slab, const FuseSeg& sg, int64_t o, float (&x)[8]) {
    if (sg.bf16) {
        const uint4 v = *reinterpret_cast<const uint4*>(slab + sg.slab_off + 2 * o);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[2 * j] = __uint_as_float(w[j] << 16);
            x[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
    } else {
        const float4* p = reinterpret_cast<const float4*>(slab + sg.slab_off + 4 * o);
        const float4 a = p[0], b = p[1];
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
        x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
}

__device__ __forceinline__ void fuse_store8(char* slab, const FuseSeg& sg, int64_t o, const float (&x)[8]) {
    if (sg.bf16) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(x[2 * j]));
            const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(x[2 * j + 1]));
            w[j] = lo | (hi << 16);
        }
        *reinterpret_cast<uint4*>(slab + sg.slab_off + 2 * o) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
        float4* p = reinterpret_cast<float4*>(slab + sg.slab_off + 4 * o);
        p[0] = make_float4(x[0], x[1], x[2], x[3]);
        p[1] = make_float4(x[4], x[5], x[6], x[7]);
    }
}

// work[a][i] = sum_k params[a K_local + k][i] (widened), k ascending; 8 elements per thread
__global__ void fuse_sum_kernel(const __grid_constant__ FuseArgs a) {
    const int agent = blockIdx.y;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n8 = a.n_elems / 8;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n8; g += stride) {
        int64_t o;
        const FuseSeg& sg = a.seg[fuse_find(a, 8 * g, &o)];
        float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int k = 0; k < a.K_local; ++k) {
            float x[8];
            fuse_load8(a.params + (static_cast<int64_t>(agent) * a.K_local + k) * a.param_bytes, sg, o, x);
#pragma unroll
            for (int j = 0; j < 8; ++j) s[j] = __fadd_rn(s[j], x[j]);
        }
        float4* w = reinterpret_cast<float4*>(a.work + static_cast<int64_t>(agent) * a.n_elems + 8 * g);
        w[0] = make_float4(s[0], s[1], s[2], s[3]);
        w[1] = make_float4(s[4], s[5], s[6], s[7]);
    }
}

// fused = tau (work / K) + (1 - tau) prev -> prev and every pod's slab slot (bf16 RNE for weights)
__global__ void fuse_blend_kernel(const __grid_constant__ FuseArgs a) {
    const int agent = blockIdx.y;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n8 = a.n_elems / 8;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n8; g += stride) {
        int64_t o;
        const FuseSeg& sg = a.seg[fuse_find(a, 8 * g, &o)];
        const int64_t fi = static_cast<int64_t>(agent) * a.n_elems + 8 * g;
        const float4* w4 = reinterpret_cast<const float4*>(a.work + fi);
        const float4 w0 = w4[0], w1 = w4[1];
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __fmul_rn(wv[j], a.scale);
        if (a.prev) {
            float4* p4 = reinterpret_cast<float4*>(a.prev + fi);
            if (a.tau != 1.0f) {
                const float4 p0 = p4[0], p1 = p4[1];
                const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    f[j] = __fadd_rn(__fmul_rn(a.tau, f[j]), __fmul_rn(__fsub_rn(1.0f, a.tau), pv[j]));
            }
            p4[0] = make_float4(f[0], f[1], f[2], f[3]);
            p4[1] = make_float4(f[4], f[5], f[6], f[7]);
        }
        for (int k = 0; k < a.K_local; ++k)
            fuse_store8(a.params + (static_cast<int64_t>(agent) * a.K_local + k) * a.param_bytes, sg, o, f);
    }
}


// ---------------------------------------------------------------------------------------------------
// Fused cross-rank fusion: ONE kernel per rank does the local pod sum, the exchange with the other ranks
// over peer memory (NVLink: every rank's partial sums live in a buffer the others map), the rank-ordered
// global sum, the tau-blend and the narrowing into every local pod — no float32 work vector round trip
// through a collective library.  Per chunk of 2,048 elements of one agent (a grid-stride loop; the chunk
// sequence of block x is the same on every rank):
//   1. (epoch > 1) wait until every rank has acknowledged reading this chunk of my stage at epoch - 1;
//   2. partial = sum over my K_local pods (pod order) -> my stage; fence; flag[me][chunk] = epoch;
//   3. wait for flag[q][chunk] == epoch of every rank q, then total = sum over q = 0..R-1 (rank order) of
//      stage[q] — bit-identical on every rank;
//   4. fused = tau (total / K) + (1 - tau) prev -> prev and my pods; ack[me][chunk] = epoch.
// Every block signals before it waits, so a block waits only for blocks that have already been or will be
// scheduled (no deadlock).  The same kernel emulates R ranks on one device (gridDim.y = R, block row y
// plays rank y, all blocks resident): the single-process form of the fusion and the one-GPU check of the
// exchange protocol.
constexpr int FUSE_MAX_RANKS = 16;
constexpr int FUSE_CHUNK = 2048;   // elements per chunk: 256 threads x 8

struct FuseXArgs {
    FuseSeg seg[FUSE_MAX_SEGS];
    int32_t n_seg;
    int32_t K_local;
    int64_t n_elems;                 // flat elements per agent
    uint64_t param_bytes;
    float scale;                     // 1 / (K_local R)
    float tau;
    int32_t R;                       // ranks taking part
    int32_t my_rank;                 // >= 0: this process's rank (gridDim.y == 1); -1: rank = blockIdx.y
    int32_t A_local;                 // agents per rank
    uint32_t epoch;                  // > 0, increasing by one per call on a communicator
    int64_t nchunks;                 // chunks per agent
    char* params[FUSE_MAX_RANKS];    // [rank] -> [A_local K_local][param_bytes] (only this rank's when my_rank >= 0)
    float* prev[FUSE_MAX_RANKS];     // [rank] -> [A_local][n_elems] or null (tau == 1)
    float* stage[FUSE_MAX_RANKS];    // [rank] -> [A_local][n_elems] partial sums (peer pointers)
    uint32_t* flag[FUSE_MAX_RANKS];  // [rank] -> [A_local nchunks]
    uint32_t* ack[FUSE_MAX_RANKS];   // [rank] -> [A_local nchunks]
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) fuse_x_kernel(const __grid_constant__ FuseXArgs a) {
    const int r = a.my_rank >= 0 ? a.my_rank : static_cast<int>(blockIdx.y);
    const int64_t total_chunks = static_cast<int64_t>(a.A_local) * a.nchunks;
    for (int64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
        const int agent = static_cast<int>(c / a.nchunks);
        const int64_t e0 = (c % a.nchunks) * FUSE_CHUNK + 8 * static_cast<int64_t>(threadIdx.x);
        const bool live = e0 < a.n_elems;
        if (a.R > 1 && a.epoch > 1) {   // 1. my stage chunk is free: every rank has read epoch - 1
            if (threadIdx.x < a.R)
                while (ld_acquire_sys(a.ack[threadIdx.x] + c) < a.epoch - 1) {
                }
            __syncthreads();
        }
        // 2. the partial sum of my pods of this agent (pod order), 8 elements per thread
        int64_t o = 0;
        const FuseSeg* sg = nullptr;
        float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int64_t fi = static_cast<int64_t>(agent) * a.n_elems + e0;
        if (live) {
            sg = &a.seg[fuse_find_seg(a.seg, a.n_seg, e0, &o)];
            for (int k = 0; k < a.K_local; ++k) {
                float x[8];
                fuse_load8(a.params[r] + (static_cast<int64_t>(agent) * a.K_local + k) * a.param_bytes, *sg, o, x);
#pragma unroll
                for (int j = 0; j < 8; ++j) s[j] = __fadd_rn(s[j], x[j]);
            }
        }
        float tot[8];
        if (a.R > 1) {
            if (live) {
                float4* w = reinterpret_cast<float4*>(a.stage[r] + fi);
                w[0] = make_float4(s[0], s[1], s[2], s[3]);
                w[1] = make_float4(s[4], s[5], s[6], s[7]);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence_system();
                st_release_sys(a.flag[r] + c, a.epoch);
            }
            // 3. every rank's partial of this chunk has landed: rank-ordered sum (own values from registers)
            if (threadIdx.x < a.R && static_cast<int>(threadIdx.x) != r)
                while (ld_acquire_sys(a.flag[threadIdx.x] + c) != a.epoch) {
                }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 8; ++j) tot[j] = 0.0f;
            if (live)
                for (int q = 0; q < a.R; ++q) {
                    float v[8];
                    if (q == r) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] = s[j];
                    } else {
                        const float4* pq = reinterpret_cast<const float4*>(a.stage[q] + fi);
                        const float4 v0 = __ldcv(pq), v1 = __ldcv(pq + 1);   // peer memory: not through L1
                        v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w;
                        v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) tot[j] = __fadd_rn(tot[j], v[j]);
                }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) tot[j] = s[j];
        }
        // 4. blend and narrow into my pods
        if (live) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = __fmul_rn(tot[j], a.scale);
            if (a.prev[r]) {
                float4* p4 = reinterpret_cast<float4*>(a.prev[r] + fi);
                if (a.tau != 1.0f) {
                    const float4 p0 = p4[0], p1 = p4[1];
                    const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        f[j] = __fadd_rn(__fmul_rn(a.tau, f[j]), __fmul_rn(__fsub_rn(1.0f, a.tau), pv[j]));
                }
                p4[0] = make_float4(f[0], f[1], f[2], f[3]);
                p4[1] = make_float4(f[4], f[5], f[6], f[7]);
            }
            for (int k = 0; k < a.K_local; ++k)
                fuse_store8(a.params[r] + (static_cast<int64_t>(agent) * a.K_local + k) * a.param_bytes, *sg, o, f);
        }
        if (a.R > 1) {
            __syncthreads();   // every thread of the block is done reading the peers' stage chunk
            if (threadIdx.x == 0) st_release_sys(a.ack[r] + c, a.epoch);
        }
    }
}

}  // namespace pod
