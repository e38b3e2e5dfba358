// pod_internal.h — host-side helpers shared by the library's translation units.
#pragma once
#include "pod.h"

pod_status pod_fail(pod_status s, const char* fmt, ...);
pod_status pod_require_sm100();

#include <cstddef>
#include <cuda_runtime.h>
// communicator helpers for the fusion entry point (pod_elite.cpp)
int pod_comm_size(const pod_comm_t* c);
pod_status pod_comm_allreduce_sum_f32(pod_comm_t* c, float* buf, size_t count, cudaStream_t stream);
