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
// K2-TC tap-plane workspace (bp_tc.cu), for K1 writing it directly (filter.cu)
int64_t bp_tc_header_bytes(const tf_bp_plan* p, int n_rows);
int tc_uniform_exponents(void* taps, int n_rows, double bound, cudaStream_t s);
int tc_row_exponents(void* taps, const float* lines, int rows_per_angle, int n_ang, int n_chan, const float* w,
                     double factor, cudaStream_t s);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define TF_CUDA_TRY(expr)                                                                            \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess)                                                                       \
            return ::tf::set_error(TF_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));   \
    } while (0)

}  // namespace tf
