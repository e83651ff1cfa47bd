// Dev micro-benchmark: FP32 FFMA vs packed FFMA2 issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, float a, float b, int iters) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b, int iters) {
    float2 acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(acc[i], a2, b2);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fadd2(float* out, float a, float b, int iters) {
    float2 acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
    const float2 b2 = make_float2(b, -b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd2_rn(acc[i], b2);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* d;
    const int blocks = 148 * 8, threads = 256, iters = 20000;
    cudaMalloc(&d, sizeof(float) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int rep = 0; rep < 2; ++rep) {
        for (int kind = 0; kind < 3; ++kind) {
            cudaEventRecord(e0);
            if (kind == 0) k_ffma<<<blocks, threads>>>(d, 0.999f, 0.001f, iters);
            else if (kind == 1) k_ffma2<<<blocks, threads>>>(d, 0.999f, 0.001f, iters);
            else k_fadd2<<<blocks, threads>>>(d, 0.999f, 0.001f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double lane_ops = (double)blocks * threads * iters * 16;  // fp32 FMA/ADD lane-ops
            printf("%s: %.3f ms, %.1f Tlane-op/s, %.1f lane-op/clk/SM (clock attr %d kHz)\n",
                   kind == 0 ? "FFMA " : kind == 1 ? "FFMA2" : "FADD2", ms, lane_ops / ms / 1e9,
                   lane_ops / (ms * 1e-3) / 148 / (clk * 1e3), clk);
        }
    }
    return 0;
}
