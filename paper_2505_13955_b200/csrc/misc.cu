// K3 quantize, K4 analytic phantom, and the C-ABI error plumbing.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "internal.hpp"

namespace tf {

static thread_local char g_last_error[512] = "";

int set_error(int status, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
    return status;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(TF_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return TF_OK;
}

namespace {

// fbp.py:255-259: round(clip((v - lo) / (hi - lo), 0, 1) * 65535) in float64
// with round-half-even; bit-identical to numpy for the same float32 input.
template <typename T>
__device__ __forceinline__ uint16_t q1(T v, double lo, double den) {
    double s = __ddiv_rn(__dsub_rn((double)v, lo), den);
    s = fmin(fmax(s, 0.0), 1.0);
    return (uint16_t)rint(__dmul_rn(s, 65535.0));
}

__global__ void quantize_kernel(const float* __restrict__ v, uint16_t* __restrict__ q, long long n, double lo,
                                double den) {
    const long long n4 = n / 4;
    const long long step = (long long)gridDim.x * blockDim.x;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const float4* v4 = reinterpret_cast<const float4*>(v);
    uint2* q4 = reinterpret_cast<uint2*>(q);
    for (long long i = tid; i < n4; i += step) {
        float4 x = v4[i];
        uint32_t a = q1(x.x, lo, den) | ((uint32_t)q1(x.y, lo, den) << 16);
        uint32_t b = q1(x.z, lo, den) | ((uint32_t)q1(x.w, lo, den) << 16);
        q4[i] = make_uint2(a, b);
    }
    for (long long i = 4 * n4 + tid; i < n; i += step) q[i] = q1(v[i], lo, den);
}

template <typename T>
__global__ void quantize_kernel_scalar(const T* __restrict__ v, uint16_t* __restrict__ q, long long n, double lo,
                                       double den) {
    const long long step = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += step) q[i] = q1(v[i], lo, den);
}

// 3-D "modified Shepp-Logan" ellipsoids (Kak & Slaney, Toft contrasts), with
// rotation about z only so every slice is an ellipse and its parallel-beam
// projection is closed form.  {rho, a, b, c, x0, y0, z0, phi_deg}
__constant__ float kEllipsoids[10][8] = {
    {1.0f, 0.6900f, 0.920f, 0.810f, 0.00f, 0.0000f, 0.00f, 0.f},
    {-0.8f, 0.6624f, 0.874f, 0.780f, 0.00f, -0.0184f, 0.00f, 0.f},
    {-0.2f, 0.1100f, 0.310f, 0.220f, 0.22f, 0.0000f, 0.00f, -18.f},
    {-0.2f, 0.1600f, 0.410f, 0.280f, -0.22f, 0.0000f, 0.00f, 18.f},
    {0.1f, 0.2100f, 0.250f, 0.410f, 0.00f, 0.3500f, -0.15f, 0.f},
    {0.1f, 0.0460f, 0.046f, 0.050f, 0.00f, 0.1000f, 0.25f, 0.f},
    {0.1f, 0.0460f, 0.046f, 0.050f, 0.00f, -0.1000f, 0.25f, 0.f},
    {0.1f, 0.0460f, 0.023f, 0.050f, -0.08f, -0.6050f, 0.00f, 0.f},
    {0.1f, 0.0230f, 0.023f, 0.020f, 0.00f, -0.6060f, 0.00f, 0.f},
    {0.1f, 0.0230f, 0.046f, 0.020f, 0.06f, -0.6050f, 0.00f, 0.f},
};

struct PhantomArgs {
    float* out;
    int a0, a1, r0, r1, n_proj, n_rows, n_chan;
    double step;        // span / n_proj
    double axis, scale; // detector convention (geometry.py:142-153)
    double rph, rphz;   // phantom radius in voxels (xy, z)
    double len_um;      // voxels -> um for normalised lengths: rph * voxel_pitch
    double i0, mu;
};

__global__ void phantom_kernel(PhantomArgs p) {
    const int nr = p.r1 - p.r0, na = p.a1 - p.a0;
    const long long total = (long long)na * nr * p.n_chan;
    const long long step = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += step) {
        const int c = (int)(i % p.n_chan);
        const long long ar = i / p.n_chan;
        const int r = (int)(ar % nr) + p.r0;
        const int k = (int)(ar / nr) + p.a0;
        const double th = (double)k * p.step;
        float sn, cs;
        sincosf((float)th, &sn, &cs);
        const float u = (float)(((double)c - p.axis) / p.scale / p.rph);
        const float zn = (float)(((double)r - (p.n_rows - 1) / 2.0) / p.rphz);
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < 10; ++e) {
            const float* E = kEllipsoids[e];
            const float dz = (zn - E[6]) / E[3];
            const float kk = 1.f - dz * dz;
            if (kk <= 0.f) continue;
            const float sk = sqrtf(kk);
            const float A = E[1] * sk, B = E[2] * sk;
            float sp, cp;
            sincosf(th - E[7] * 0.017453292519943295f, &sp, &cp);
            const float a2 = A * A * cp * cp + B * B * sp * sp;
            const float up = u - (E[4] * cs + E[5] * sn);
            const float d = a2 - up * up;
            if (d > 0.f) acc += E[0] * 2.f * A * B * sqrtf(d) / a2;
        }
        const double depth = (double)acc * p.len_um * p.mu;
        p.out[i] = (float)(p.i0 * exp(-depth));
    }
}

}  // namespace
}  // namespace tf

using namespace tf;

extern "C" const char* tf_error_string(int status) {
    switch (status) {
        case TF_OK: return "ok";
        case TF_ERR_INVALID_ARGUMENT: return "invalid argument";
        case TF_ERR_CUDA: return "CUDA error";
        case TF_ERR_UNSUPPORTED: return "unsupported configuration";
        case TF_ERR_OUT_OF_MEMORY: return "out of memory";
        default: return "unknown status";
    }
}

extern "C" const char* tf_last_error(void) { return g_last_error; }

extern "C" int tf_version(void) { return 1; }

extern "C" int tf_quantize(const void* vol, int vol_dtype, uint16_t* out, int64_t n, double lo, double hi,
                           void* stream) {
    if (!(lo < hi)) return set_error(TF_ERR_INVALID_ARGUMENT, "window requires lo < hi, got [%g, %g]", lo, hi);
    if (n < 0) return set_error(TF_ERR_INVALID_ARGUMENT, "n must be >= 0");
    if (n == 0) return TF_OK;
    if (!vol || !out) return set_error(TF_ERR_INVALID_ARGUMENT, "null buffer");
    const double den = hi - lo;
    const int blocks = (int)std::min<long long>((n / 4 + 255) / 256 + 1, 148LL * 16);
    if (vol_dtype == TF_F64)
        quantize_kernel_scalar<double><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const double*>(vol), out, n,
                                                                              lo, den);
    else if (vol_dtype != TF_F32)
        return set_error(TF_ERR_INVALID_ARGUMENT, "unsupported volume dtype %d", vol_dtype);
    else if ((reinterpret_cast<uintptr_t>(vol) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 7) == 0)
        quantize_kernel<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const float*>(vol), out, n, lo, den);
    else
        quantize_kernel_scalar<float><<<blocks, 256, 0, as_stream(stream)>>>(static_cast<const float*>(vol), out, n,
                                                                             lo, den);
    return check_launch("quantize_kernel");
}

extern "C" int tf_phantom_sinogram(const tf_geometry* g, int a0, int a1, int r0, int r1, double i0, double mu_max,
                                   float* out, void* stream) {
    if (!g || !out) return set_error(TF_ERR_INVALID_ARGUMENT, "null argument");
    if (!(0 <= a0 && a0 <= a1 && a1 <= g->n_proj && 0 <= r0 && r0 <= r1 && r1 <= g->n_rows))
        return set_error(TF_ERR_INVALID_ARGUMENT, "phantom range out of bounds");
    const long long total = (long long)(a1 - a0) * (r1 - r0) * g->n_chan;
    if (total == 0) return TF_OK;
    PhantomArgs p{};
    p.out = out;
    p.a0 = a0;
    p.a1 = a1;
    p.r0 = r0;
    p.r1 = r1;
    p.n_proj = g->n_proj;
    p.n_rows = g->n_rows;
    p.n_chan = g->n_chan;
    p.step = g->angle_span / g->n_proj;
    p.axis = (g->n_chan - 1) / 2.0 - g->offset_chan;
    p.scale = g->voxel_pitch / g->pixel_pitch;
    p.rph = 0.48 * (double)std::min(g->nx, g->ny);
    p.rphz = 0.48 * (double)g->n_rows;
    p.len_um = p.rph * g->voxel_pitch;
    p.i0 = i0;
    p.mu = mu_max;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
    phantom_kernel<<<blocks, 256, 0, as_stream(stream)>>>(p);
    return check_launch("phantom_kernel");
}

extern "C" int tf_copy2d_async(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width_bytes,
                               size_t height, void* stream) {
    if (width_bytes == 0 || height == 0) return TF_OK;
    if (!dst || !src || dpitch < width_bytes || spitch < width_bytes)
        return set_error(TF_ERR_INVALID_ARGUMENT, "invalid 2-D copy");
    TF_CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, height, cudaMemcpyDefault,
                                  as_stream(stream)));
    return TF_OK;
}
