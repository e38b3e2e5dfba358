// pod_internal.h — host-side helpers shared by the library's translation units.
#pragma once
#include "pod.h"

pod_status pod_fail(pod_status s, const char* fmt, ...);
pod_status pod_require_sm100();
