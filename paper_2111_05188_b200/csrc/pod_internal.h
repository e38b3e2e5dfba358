// pod_internal.h — host-side helpers shared by the library's translation units.
#pragma once
#include "pod.h"

pod_status pod_fail(pod_status s, const char* fmt, ...);
pod_status pod_require_sm100();

#include <cstddef>
#include <cuda_runtime.h>
// communicator helpers for the fusion entry point (pod_elite.cpp)
int pod_comm_size(const pod_comm_t* c);
int pod_comm_rank(const pod_comm_t* c);
// the peer-mapped buffers of the fused cross-rank fusion (fuse_x_kernel): on first use, or when they must
// grow, every rank (collectively) allocates one zeroed buffer of stage_elems floats + 2 nflags words,
// exchanges its CUDA IPC handle over NCCL and maps the others'; returns every rank's stage / flag / ack
// pointers ([nranks] each, in this process's address space) and this call's epoch (1, 2, ... per buffer set)
pod_status pod_comm_fuse_buffers(pod_comm_t* c, size_t stage_elems, size_t nflags, float** stage, uint32_t** flag,
                                 uint32_t** ack, uint32_t* epoch, cudaStream_t stream);

// kernel-launch accounting (pod_kernel_launches): a launch made on stream s counts unless s is being
// captured (a captured graph counts its kernel nodes each time it is launched)
void pod_note_launch(cudaStream_t s, unsigned long long n = 1);
unsigned long long pod_graph_kernel_nodes(cudaGraph_t g);
void pod_note_graph_launch(unsigned long long kernel_nodes);
