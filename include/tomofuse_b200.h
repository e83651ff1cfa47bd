/*
 * tomofuse-b200 C ABI: the drop-in boundary for the reference's FBP hot path.
 *
 * The reference (`/root/reference/pkg/src/tomofuse/fbp.py`) is a pure-Python
 * package; its reconstruction "plugin surface" is the function set
 * preprocess / filter_multiplier / offset_weights / ramp_filter /
 * back_project / quantize / reconstruct.  Each entry point below replaces one
 * of them (cited per function).  The Python mirror
 * `paper_2505_13955_b200.fbp` binds this library with ctypes and keeps the
 * reference signatures, argument meaning and ValueError behaviour; see
 * INTEGRATION.md for the binding a tomofuse maintainer would add.
 *
 * Conventions
 *  - Plain pointers + sizes; no torch types.  Device pointers are caller-owned
 *    device memory; `stream` is a cudaStream_t passed as void*.
 *  - Work is stream-ordered and reentrant; plans are immutable after creation
 *    and may be shared by concurrent streams.  Hot calls never allocate.
 *  - Array order follows the reference: sinograms are angle-major
 *    (n_proj, n_rows, n_chan) (fbp.py:206), volumes are (z, y, x)
 *    (geometry.py:94-97).
 *  - Every call returns a tf_status; tf_error_string() gives the text the
 *    Python layer raises as ValueError / RuntimeError.
 */
#ifndef TOMOFUSE_B200_H
#define TOMOFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TF_API __attribute__((visibility("default")))
#else
#define TF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TF_OK = 0,
    TF_ERR_INVALID_ARGUMENT = 1, /* maps to ValueError */
    TF_ERR_CUDA = 2,             /* CUDA runtime/driver failure */
    TF_ERR_UNSUPPORTED = 3,      /* geometry outside the compiled kernels */
    TF_ERR_OUT_OF_MEMORY = 4
} tf_status;

/* Scan + grid description: AcquisitionParams (geometry.py:27-70) and
 * VolumeDims (geometry.py:73-97) flattened into one POD. */
typedef struct {
    int32_t n_proj, n_rows, n_chan;
    int32_t nx, ny;
    int32_t offset_chan; /* 0 for normal scans (ScanMode.NORMAL) */
    int32_t scan_mode;   /* 0 = NORMAL, 1 = OFFSET (geometry.py:22-24) */
    int32_t reserved;
    double angle_span;   /* radians */
    double pixel_pitch;  /* detector pitch, um */
    double voxel_pitch;  /* voxel pitch, um */
} tf_geometry;

typedef enum { TF_FILTER_RAMLAK = 0, TF_FILTER_SHEPPLOGAN = 1 } tf_filter_kind;

typedef enum { TF_F32 = 0, TF_F64 = 1 } tf_dtype;

typedef struct tf_filter_plan tf_filter_plan;
typedef struct tf_bp_plan tf_bp_plan;

TF_API const char* tf_error_string(int status);
/* Last error detail of the calling thread (messages match the reference's
 * ValueError texts where one exists). */
TF_API const char* tf_last_error(void);
TF_API int tf_version(void);

/* ---- host-side plan math (tiny tables; fp64, bit-for-bit the reference) -- */

/* Replaces fbp.filter_multiplier (fbp.py:105-116): Re(rfft(h))/pixel_pitch,
 * written to host_out[0 .. padded/2]. */
TF_API int tf_filter_multiplier(int kind, int64_t padded, double pixel_pitch, double* host_out);

/* Replaces fbp.offset_weights (fbp.py:147-183): n_chan fp64 weights. */
TF_API int tf_offset_weights(const tf_geometry* g, int feather_band, double* host_out);

/* ---- filtering: preprocess + blur + ramp (fbp.py:75-83, 119-131) -------- */

/* Plan for lines of n_chan channels. `padded` is the reference's FilterSpec
 * padding (0 = next pow2 >= 2n); it is validated (>= 2n) exactly like
 * FilterSpec.padded_length (fbp.py:48-60).  The filtered result is
 * independent of the pad length once pad >= 2n, so the kernel always
 * transforms at the internal length next_pow2(2n). */
TF_API int tf_filter_plan_create(int n_chan, int kind, int64_t padded, double pixel_pitch, double blur_sigma,
                          tf_filter_plan** plan);
TF_API int tf_filter_plan_destroy(tf_filter_plan* plan);

/* Filters n_lines lines.  in: n_lines x n_chan fp32 raw counts (i0 > 0:
 * Beer-Lambert -ln(max(raw,1)/i0) is fused in) or optical depth (i0 <= 0).
 * out: filtered fp32; line l goes to out + l_dst*n_chan where, for
 * n_slabs > 0, lines are (angle, row) pairs of an angle-major block with
 * `rows_per_angle` rows and rows are regrouped slab-major for a row-slab
 * all-to-all: row r in slab s = [slab_row0[s], slab_row0[s+1]) of angle a
 * goes to element offset slab_base[s] + (a*(slab_row0[s+1]-slab_row0[s]) +
 * r - slab_row0[s]) * n_chan.  n_slabs == 0 keeps the natural layout.
 * in == out (in-place) is allowed for the natural layout. */
TF_API int tf_filter(const tf_filter_plan* plan, const float* in, float* out, int64_t n_lines, float i0,
              int rows_per_angle, int n_slabs, const int32_t* slab_row0, const int64_t* slab_base,
              void* stream);

/* Same filter, written straight into K2's z-blocked staging layout (the
 * layout tf_bp_stage produces, feather weights of `bp` applied) -- the fused
 * reconstruction path, no intermediate filtered sinogram.  Lines are
 * (angle, row) of an angle-major block of `rows_per_angle` rows.  With
 * n_slabs > 0 the rows are split into slabs [slab_row0[s], slab_row0[s+1])
 * each staged as its own z-blocked array starting at element slab_base[s]
 * (the row-slab all-to-all send layout: it lands on the owner as its staging
 * buffer); n_slabs == 0 stages all rows as one slab at `stage`. */
TF_API int tf_filter_stage(const tf_filter_plan* plan, const tf_bp_plan* bp, const float* in, void* stage,
                           int64_t n_lines, float i0, int rows_per_angle, int n_slabs, const int32_t* slab_row0,
                           const int64_t* slab_base, void* stream);

/* Fused filter + exchange: like tf_filter_stage with n_slabs > 0, but slab s
 * is written straight to the device pointer slab_dst[s] -- typically the
 * owner GPU's staging buffer mapped over NVLink (CUDA IPC / symmetric
 * memory), already offset to this rank's first angle.  The K1 epilogue's
 * stores ARE the row-slab all-to-all; the caller orders them with a
 * cross-GPU barrier before the owners' back-projection. */
TF_API int tf_filter_stage_peers(const tf_filter_plan* plan, const tf_bp_plan* bp, const float* in, int64_t n_lines,
                                 float i0, int rows_per_angle, int n_slabs, const int32_t* slab_row0,
                                 void* const* slab_dst, void* stream);

/* Fused filter + exchange, natural rows: slab s's rows of every line
 * (angle-major, [angle][row - slab_row0[s]][chan], like tf_filter's slab map)
 * are written to the device pointer slab_dst[s], typically the owner GPU's
 * receive buffer over NVLink.  Each line is one contiguous run, so the remote
 * stores are fully coalesced; the owner stages its rows locally
 * (tf_bp_stage) after a cross-GPU barrier. */
TF_API int tf_filter_peers(const tf_filter_plan* plan, const float* in, int64_t n_lines, float i0, int rows_per_angle,
                           int n_slabs, const int32_t* slab_row0, void* const* slab_dst, void* stream);

/* K1 straight into K2-TC's tap planes (tf_bp_tc_taps_bytes): Beer-Lambert,
 * ramp filter, feather, x 2^e[r], fp16 hi/lo split in the epilogue -- no fp32
 * staging, no conversion pass.  Lines are (angle, row) of an angle-major
 * block of rows_per_angle rows; the workspace's angle 0 is the block's first.
 * i0 > 0 (raw counts): one exponent for every row from the analytic bound
 * |T| <= max|depth| * sum|h| / pitch with |depth| <= max(ln i0, ln FLT_MAX -
 * ln i0) (tf_filter_tap_bound), so the scale never depends on the data and
 * sub-slabs, chunks and GPUs see the same taps.  i0 <= 0 (optical depth):
 * per-row exponents from each row's max |depth| (one extra read pass). */
TF_API int tf_filter_taps(const tf_filter_plan* plan, const tf_bp_plan* bp, const float* in, void* taps,
                          int64_t taps_bytes, int64_t n_lines, float i0, int rows_per_angle, void* stream);
/* The bound on |T| that tf_filter_taps uses for raw counts with this i0. */
TF_API int tf_filter_tap_bound(const tf_filter_plan* plan, double i0, double* bound);

/* Beer-Lambert only (fbp.py:75-83): fp32 or fp64 counts -> fp64 depth
 * (the reference's output dtype), computed in fp64. */
TF_API int tf_preprocess(const void* raw, int raw_dtype, double* out, int64_t n, double i0, void* stream);

/* ---- back-projection (fbp.py:186-252) ---------------------------------- */

TF_API int tf_bp_plan_create(const tf_geometry* g, int feather_band, tf_bp_plan** plan);
TF_API int tf_bp_plan_destroy(tf_bp_plan* plan);

/* Bytes of the z-blocked staging buffer for `n_rows` rows. */
TF_API int64_t tf_bp_stage_bytes(const tf_bp_plan* plan, int n_rows);

/* Converts filtered rows [r0, r1) of an angle-major fp32 sinogram (row pitch
 * n_chan, angle pitch `rows_per_angle`*n_chan) into the z-blocked staging
 * layout, applying the offset-scan feather (fbp.py:242).  `stage` must hold
 * tf_bp_stage_bytes(plan, r1-r0) bytes. */
TF_API int tf_bp_stage(const tf_bp_plan* plan, const float* sino, int rows_per_angle, int r0, int r1, void* stage,
                void* stream);

enum {
    TF_BP_ACCUMULATE = 1, /* add to the unscaled partial sums already in vol */
    TF_BP_FINALIZE = 2,   /* apply FoV mask + angle_span/n_proj scale (fbp.py:246-251) */
    TF_BP_KERNEL_V1 = 4,  /* force the 1-voxel 2-tap kernel (default: x-pair
                             3-tap kernel when voxel/pixel pitch <= 1; both give
                             bit-identical volumes) */
    TF_BP_REDUCE = 8      /* internal: set by tf_backproject_reduce */
};

/* Back-projects angles [a0, a1) of a staged slab of `n_rows` rows into
 * vol (n_rows, ny, nx) fp32, restricted to tile [x0,x1) x [y0,y1)
 * (fbp.py:191-193).  Voxels outside the tile are not written.  With
 * flags = TF_BP_FINALIZE a single call reproduces back_project(); angle
 * chunks may be chained with TF_BP_ACCUMULATE (summation order stays
 * ascending in angle, fbp.py:198-201). */
TF_API int tf_backproject(const tf_bp_plan* plan, const void* stage, int n_rows, float* vol, int a0, int a1, int x0,
                   int x1, int y0, int y1, int flags, void* stream);

/* Angle-split back-projection with the reduction fused into K2's epilogue
 * (replaces the P_proj partials + Fabric.reduce_scatter_block of
 * pipeline.py:239-275 / fabric.py:67-101).  Back-projects angles [a0, a1) of
 * a staged full-height slab (rows [0, n_rows)) over the whole (ny, nx) plane
 * and ADDS the unscaled partial sums of volume row z into the slab that owns
 * it: slab_dst[s] + (z - slab_row0[s]) * ny * nx, for slab_row0[s] <= z <
 * slab_row0[s+1] (n_slabs <= 8; slab_row0[0] = 0, slab_row0[n_slabs] =
 * n_rows).  slab_dst may point into other GPUs' memory (NVLink peer
 * mappings); the adds are atomic, so concurrent ranks may target the same
 * slab.  Owners zero their slab first and call tf_bp_finalize after every
 * rank's adds have landed.  Summation order across ranks is not fixed.
 * `stage` holds only angles [a0, a1) (a rank's chunk, as tf_filter_stage
 * writes it), not all n_proj. */
TF_API int tf_backproject_reduce(const tf_bp_plan* plan, const void* stage, int n_rows, int a0, int a1, int n_slabs,
                                 const int32_t* slab_row0, void* const* slab_dst, int flags, void* stream);

/* FoV mask + angle_span/n_proj scale (fbp.py:246-251) applied to unscaled
 * partial sums vol (n_rows, ny, nx): the TF_BP_FINALIZE epilogue as a pass. */
TF_API int tf_bp_finalize(const tf_bp_plan* plan, float* vol, int n_rows, void* stream);

/* Shared-memory bytes the selected K2 variant gathers per voxel x projection
 * update for these flags (8 = 2-tap, 6 = x-pair 3-tap, 4 = 2x2 4-tap): the
 * algorithmic numerator of K2's roofline. */
TF_API int tf_bp_smem_bytes_per_update(const tf_bp_plan* plan, int flags, double* bytes);
/* Same, plus the voxel x projection updates K2 executes for a full-volume
 * call over n_rows rows and angles [a0, a1) (FoV-skipped tiles excluded,
 * rows padded to the 32-row z-block): the roofline's work count. */
TF_API int tf_bp_kernel_info(const tf_bp_plan* plan, int flags, int n_rows, int a0, int a1, double* bytes,
                             int64_t* executed_updates);

/* ---- tensor-core back-projection (K2-TC, the default; same contract as
 * tf_backproject) ------------------------------------------------------------
 * The same sum as tf_backproject (fbp.py:186-252) computed as per-angle GEMMs
 * D[voxel][row] += W[voxel][chan] * T[chan][row] on tcgen05: 11 x 11 voxel
 * tiles (121 of the MMA's M = 128 rows) x 256 (or 128) detector rows, exact
 * two-tap weights, fp16 hi/lo split operands, fp32 accumulation in TMEM over
 * blocks of 16 angles (blocks of the absolute angle index k / 16) re-added in
 * round-to-nearest fp32.  Not bitwise equal to the CUDA-core kernels
 * (different summation order); within the fp32 tolerance of the reference's
 * float64 output.  Angle chunks chained with TF_BP_ACCUMULATE at multiples of
 * 16 angles give the single-pass result bit for bit.
 *
 * Input: "tap planes", a workspace of tf_bp_tc_taps_bytes(plan, n_rows,
 * n_angles) bytes: a header of per-row exponents e[r], then per angle fp16
 * planes [hi, lo][row / 8][chan][row % 8] of the feathered filtered taps
 * scaled by 2^e[r].  Producers: tf_filter_taps (K1 straight from raw counts
 * or depth) and tf_bp_tc_stage (from filtered natural-layout rows).
 * Requires voxel_pitch / pixel_pitch <= 2.12 (tf_bp_tc_supported). */
TF_API int tf_bp_tc_supported(const tf_bp_plan* plan);
TF_API int64_t tf_bp_tc_taps_bytes(const tf_bp_plan* plan, int n_rows, int n_angles);
/* Filtered rows [r0, r1) of angles [a0, a1) of an angle-major fp32 sinogram
 * (row pitch n_chan, angle pitch rows_per_angle * n_chan) -> tap planes (the
 * workspace's angle 0 = a0).  t_bound > 0: a bound on |T| fixes one exponent
 * for every row (results independent of the data's range; an undersized
 * bound saturates the fp16 taps); t_bound <= 0: per-row exponents from the
 * rows' own max |T w| over [a0, a1). */
TF_API int tf_bp_tc_stage(const tf_bp_plan* plan, const float* sino, int rows_per_angle, int r0, int r1, int a0,
                          int a1, double t_bound, void* taps, int64_t taps_bytes, void* stream);
/* Sets every row's exponent of a tap workspace from the bound t_bound > 0. */
TF_API int tf_bp_tc_set_exponent(const tf_bp_plan* plan, void* taps, int n_rows, double t_bound, void* stream);
/* Back-projects angles [a0, a1) of tap planes holding [taps_a0, taps_a1) for
 * n_rows rows into vol (n_rows, ny, nx), tile and flags as tf_backproject. */
TF_API int tf_backproject_tc(const tf_bp_plan* plan, const void* taps, int64_t taps_bytes, int taps_a0, int taps_a1,
                             int n_rows, float* vol, int a0, int a1, int x0, int x1, int y0, int y1, int flags,
                             void* stream);
/* Work of one tf_backproject_tc call over n_rows rows and angles [a0, a1)
 * (host query, synchronous): MMA items (K-steps of 3 fp16 MMAs), voxel x
 * angle x row updates of the FoV-active tiles (the roofline's executed
 * updates), and tensor-pipe clocks of the MMAs (items x 3 x N/2). */
TF_API int tf_bp_tc_work(const tf_bp_plan* plan, int n_rows, int a0, int a1, int64_t* items,
                         int64_t* executed_updates, int64_t* mma_clocks);

/* ---- quantize (fbp.py:255-259) ------------------------------------------ */
/* vol is fp32 or fp64 (vol_dtype); arithmetic is fp64, round-half-even,
 * bit-identical to numpy for the same input values. */
TF_API int tf_quantize(const void* vol, int vol_dtype, uint16_t* out, int64_t n, double lo, double hi, void* stream);

/* ---- forward projection (phantom.py:199-255) ----------------------------- */
/* K5: the transpose of K2's interpolation (linear splat of each in-FoV voxel
 * onto its two channels), vol (n_rows, ny, nx) fp32 -> sino (n_proj, n_rows,
 * n_chan) fp32 scaled by voxel_pitch.  project_volume uses voxel_pitch =
 * pixel_pitch, as the reference does. */
TF_API int tf_forward_project(const tf_geometry* g, const float* vol, float* sino, void* stream);

/* ---- host <-> device slab streaming --------------------------------------- */
/* Strided 2-D async copy (cudaMemcpy2DAsync, direction inferred from UVA):
 * `height` rows of `width_bytes`, with the given pitches.  Used to move one
 * z-slab of an angle-major host sinogram (n_proj strided chunks) into HBM and
 * volume slabs back, overlapped with compute on other streams. */
TF_API int tf_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width_bytes,
                           size_t height, void* stream);

/* ---- synthetic input: analytic 3-D Shepp-Logan raw counts -------------- */
/* Writes raw counts i0*exp(-p) (fp32) for angles [a0,a1), rows [r0,r1) into
 * out (a1-a0, r1-r0, n_chan).  Attenuation max `mu_max` (1/um). */
TF_API int tf_phantom_sinogram(const tf_geometry* g, int a0, int a1, int r0, int r1, double i0, double mu_max,
                        float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TOMOFUSE_B200_H */
