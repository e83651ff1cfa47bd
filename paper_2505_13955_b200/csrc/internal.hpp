// Host-side plumbing shared by the tomofuse-b200 translation units.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "../../include/tomofuse_b200.h"

namespace tf {

int set_error(int status, const char* fmt, ...);
// bp plan accessors for the fused filter -> staging path (backproject.cu)
const float* bp_plan_weights(const tf_bp_plan* p);  // device feather weights, nullptr if all ones
int bp_plan_n_chan(const tf_bp_plan* p);
int check_launch(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define TF_CUDA_TRY(expr)                                                                            \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess)                                                                       \
            return ::tf::set_error(TF_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));   \
    } while (0)

}  // namespace tf
