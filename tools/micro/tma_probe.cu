// TMA throughput probe for K2-TC's tap boxes: one producer warp per CTA
// streams "items" of two boxes {8 x 16 channels (256 B rows), R8 row groups}
// (the T_hi / T_lo planes of one item) into an 8-slot ring; a consumer warp
// only waits and frees.  Reports clk per item per SM and B/clk/SM for:
//   mode 0: channel start c varies per item (K2's 16-B-granular window start)
//   mode 1: c rounded to even (32-B sector-aligned box rows)
//   mode 2: c rounded to a multiple of 8 (128-B aligned)
//   mode 3: like 0 but one 16 KB box per item (both planes as one 2-D box)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

constexpr int kS = 8;

template <int R8>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap map, int items, int n_chan, int n_ang,
                                               int mode, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int PLANE = R8 * 256;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kS * 2 * PLANE);
    uint64_t* empty = full + kS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int zg = (blockIdx.x % 8) * R8;
    if (warp == 0) {
        if (lane == 0) {
            for (int it = 0; it < items; ++it) {
                const int s = it % kS;
                if (it >= kS) mbar_wait(&empty[s], ((it / kS) - 1) & 1);
                int c = (int)((blockIdx.x * 131u + it * 37u) % (unsigned)(n_chan - 32));
                if (mode == 1) c &= ~1;
                if (mode == 2) c &= ~7;
                const int ka = 2 * ((it + blockIdx.x) % n_ang);
                uint8_t* st = smem + s * 2 * PLANE;
                mbar_expect(&full[s], 2 * PLANE);
                tma3(st, &map, &full[s], 8 * c, zg, ka);
                tma3(st + PLANE, &map, &full[s], 8 * c, zg, ka + 1);
            }
        }
    } else {
        long long t0 = clock64();
        for (int it = 0; it < items; ++it) {
            const int s = it % kS;
            mbar_wait(&full[s], (it / kS) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
    }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int n_chan = 2048, R8all = 256, n_ang = argc > 1 ? atoi(argv[1]) : 64, items = 4000;
    size_t bytes = (size_t)n_chan * 16 * R8all * 2 * n_ang;
    void* d;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(d, 0, bytes));
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    Enc enc = (Enc)fp;
    long long* out;
    CK(cudaMalloc(&out, 148 * 8));
    long long h[148];
    for (int mode = 0; mode < 3; ++mode) {
        CUtensorMap map;
        cuuint64_t dims[3] = {(cuuint64_t)8 * n_chan, (cuuint64_t)R8all, (cuuint64_t)(2 * n_ang)};
        cuuint64_t str[2] = {(cuuint64_t)n_chan * 16, (cuuint64_t)R8all * n_chan * 16};
        cuuint32_t box[3] = {128, 32, 1}, es[3] = {1, 1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        const int smem = kS * 2 * 32 * 256 + 2 * kS * 8;
        CK(cudaFuncSetAttribute(probe<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int rep = 0; rep < 2; ++rep) {
            probe<32><<<148, 64, smem>>>(map, items, n_chan, n_ang, mode, out);
            CK(cudaDeviceSynchronize());
        }
        CK(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
        double mean = 0;
        for (int i = 0; i < 148; ++i) mean += (double)h[i] / items;
        mean /= 148;
        printf("{\"mode\": %d, \"n_ang\": %d, \"working_set_MB\": %.0f, \"clk_per_item\": %.1f, \"B_per_clk_sm\": %.1f}\n", mode,
               n_ang, bytes / 1e6, mean, 16384.0 / mean);
    }
    return 0;
}
