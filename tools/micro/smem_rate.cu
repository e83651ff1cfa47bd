// Micro-benchmark: shared-memory load bandwidth per SM on sm_100a, the roof
// K2 (back-projection) is bound by.  Conflict-free LDS.128 (lane i reads the
// 16 B at i*16 of a rotating 512-B row), also LDS.64 and LDS.32, timed with
// the SM's own clock64 per CTA, so the result is bytes per SM clock
// independent of the clock the GPU runs at.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_rate smem_rate.cu && ./smem_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int W>  // words (4 B) per lane per load: 1, 2, 4
__global__ void __launch_bounds__(1024, 2) k_lds(unsigned* out, long long* cycles, int iters) {
    // cycles[3*cta + {0,1,2}] = start clock, end clock, SM id (clock64 is per SM)
    extern __shared__ unsigned sm[];
    const int n = 16384;  // 64 KB
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    long long t0 = clock64();
    int base = warp * 32 * W;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int off = ((base + u * 32 * W * 5) & (n - 1)) + lane * W;  // warp reads 32*W consecutive words
            if (W == 4) {
                uint4 v = *reinterpret_cast<const uint4*>(sm + off);
                acc0 ^= v.x; acc1 ^= v.y; acc2 ^= v.z; acc3 ^= v.w;
            } else if (W == 2) {
                uint2 v = *reinterpret_cast<const uint2*>(sm + off);
                acc0 ^= v.x; acc1 ^= v.y;
            } else {
                acc0 ^= sm[off];
            }
        }
        base += 32 * W * 3;
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        cycles[3 * blockIdx.x] = t0;
        cycles[3 * blockIdx.x + 1] = t1;
        cycles[3 * blockIdx.x + 2] = smid;
    }
}

template <int W>
void run(int nsm) {
    const int threads = 1024, ctas = nsm * 2, iters = 16384;
    unsigned* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(unsigned) * threads * ctas);
    cudaMalloc(&cyc, sizeof(long long) * 3 * ctas);
    cudaFuncSetAttribute(k_lds<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k_lds<W><<<ctas, threads, 65536>>>(out, cyc, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_lds<W><<<ctas, threads, 65536>>>(out, cyc, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long* h = new long long[3 * ctas];
    cudaMemcpy(h, cyc, sizeof(long long) * 3 * ctas, cudaMemcpyDeviceToHost);
    // per SM: bytes of its CTAs over [first start, last end] on that SM's clock
    const double bytes_per_cta = (double)threads * iters * 8 * W * 4;
    double sum_bpc = 0, min_bpc = 1e30;
    int sms = 0;
    for (int sm = 0; sm < 1024; ++sm) {
        long long lo = -1, hi = 0;
        int c = 0;
        for (int i = 0; i < ctas; ++i)
            if (h[3 * i + 2] == sm) {
                lo = (lo < 0 || h[3 * i] < lo) ? h[3 * i] : lo;
                hi = h[3 * i + 1] > hi ? h[3 * i + 1] : hi;
                ++c;
            }
        if (!c) continue;
        const double bpc = c * bytes_per_cta / (double)(hi - lo);
        sum_bpc += bpc;
        min_bpc = bpc < min_bpc ? bpc : min_bpc;
        ++sms;
    }
    const double total = bytes_per_cta * ctas;
    printf("{\"load\": \"LDS.%d\", \"bytes_per_clk_per_sm\": %.2f, \"bytes_per_clk_per_sm_min\": %.2f, "
           "\"tb_per_s\": %.2f, \"ms\": %.3f, \"sms\": %d, \"ctas\": %d}\n",
           32 * W, sum_bpc / sms, min_bpc, total / ms / 1e9, ms, sms, ctas);
    delete[] h;
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run<4>(nsm);
    run<2>(nsm);
    run<1>(nsm);
    return 0;
}
