// The back-projection plan shared by the CUDA-core K2 (backproject.cu) and
// the tensor-core K2 (bp_tc.cu): geometry constants in fp64 (the reference's
// arithmetic, geometry.py:27-153 / fbp.py:134-183), the per-angle cos/sin
// table and the per-tile-shape launch orders.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.hpp"

// tile shapes with a launch order: 0 = the CUDA-core kernels' 16 x 16,
// 1 = the tensor-core kernel's 11 x 11 (121 voxels in the MMA's M = 128 rows)
constexpr int kNumTileShapes = 2;
constexpr int kTileShape[kNumTileShapes][2] = {{16, 16}, {11, 11}};
constexpr int kShapeCuda = 0, kShapeTc = 1;

struct tf_bp_plan {
    tf_geometry g;
    int feather_band;
    double2* d_trig;  // (cos, sin) of k * (span / n_proj), fp64 libm, per angle
    float* d_w;       // feather weights (fp32, as numpy casts them)
    int* d_order[kNumTileShapes];  // tile launch order (Morton, FoV-active first) per tile shape
    int* h_order[kNumTileShapes];  // host copies (per-call tile lists of restricted tensor-core calls)
    int n_active[kNumTileShapes];
    int n_tiles[kNumTileShapes];
    double cx, cy, scale, axis, R2, sc2;
    float angle_wf;
};

namespace tf {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);
PFN_encodeTiled_t encode_fn();

}  // namespace tf
