// Probe: tcgen05.mma kind::f16 (fp16 in, fp32 accumulate in TMEM), M=128,
// N=256, K=16*KS, A K-major and B MN-major, both SWIZZLE_NONE canonical
// layouts written by threads; checks D against a CPU GEMM and times a long
// chain of MMAs (clk per instruction) -- the building block of a
// tensor-core back-projection variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu && ./umma_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#ifndef PN
#define PN 256
#endif
constexpr int M = 128, N = PN, KS = 2, K = 16 * KS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm_100)
    return d;                // layout type 0 = SWIZZLE_NONE, base offset 0
}

// A: M x K, K-major. B: K x N, MN-major.
__host__ __device__ constexpr uint32_t a_off(int m, int k) {
    return (m % 8) * 16 + (m / 8) * 128 + (k % 8) * 2 + (k / 8) * (M * 16);
}
__host__ __device__ constexpr uint32_t b_off(int n, int k) {
    return (n % 8) * 2 + (n / 8) * (K * 16) + (k % 8) * 16 + (k / 8) * 128;
}
constexpr uint32_t A_LBO = M * 16, A_SBO = 128, B_LBO = 128, B_SBO = K * 16;

constexpr uint32_t IDESC = (1u << 4)            // D = f32
                           | (0u << 7) | (0u << 10)  // A, B = f16
                           | (0u << 15)          // A K-major
                           | (1u << 16)          // B MN-major
                           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}

// -DATMEM: A from TMEM (columns [N, N + K/2), fp16 pairs, written with tcgen05.st), as the
// tensor-core back-projection does with its weight rows
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t ta, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(ta), "l"(db), "r"(IDESC), "r"(acc));
}

__global__ void __launch_bounds__(128, 1) k_probe(const __half* A, const __half* B, float* D, long long* clk, int reps) {
#ifndef NBUF
#define NBUF 1
#endif
    extern __shared__ __align__(1024) uint8_t dyn[];  // NBUF distinct copies of A and B
    uint8_t* sa = dyn;
    uint8_t* sb = dyn + NBUF * M * K * 2;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2[4];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int c = 0; c < NBUF; ++c) {
        for (int i = tid; i < M * K; i += 128) {
            int m = i / K, k = i % K;
            *reinterpret_cast<__half*>(sa + c * M * K * 2 + a_off(m, k)) = A[i];
        }
        for (int i = tid; i < N * K; i += 128) {
            int k = i / N, n = i % N;
            *reinterpret_cast<__half*>(sb + c * N * K * 2 + b_off(n, k)) = B[i];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        for (int c = 0; c < 4; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[c])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t td = tbase;
#ifdef ATMEM
    {
        uint32_t v[K / 2];
        for (int j = 0; j < K / 2; ++j) {
            __half2 h = __halves2half2(A[tid * K + 2 * j], A[tid * K + 2 * j + 1]);
            v[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        const uint32_t ta = td + ((uint32_t)(warp * 32) << 16) + N;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                     "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
#endif
    if (tid == 0) {
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int s = 0; s < KS; ++s)
#ifdef ATMEM
                mma_ts(td, td + N + s * 8, sdesc(smem_u32(sb) + (r % NBUF) * N * K * 2 + s * 256, B_LBO, B_SBO),
                       (r | s) ? 1u : 0u);
#else
                mma(td, sdesc(smem_u32(sa) + (r % NBUF) * M * K * 2 + s * 2 * A_LBO, A_LBO, A_SBO),
                    sdesc(smem_u32(sb) + (r % NBUF) * N * K * 2 + s * 256, B_LBO, B_SBO), (r | s) ? 1u : 0u);
#endif
#ifdef PCOMMIT  // a commit per KS-step group (as the back-projection kernel does per angle)
            for (int c = 0; c < PCOMMIT; ++c)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&bar2[c])));
#endif
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
        // wait for completion (phase 0)
        asm volatile(
            "{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}\n" ::"r"(
                smem_u32(&bar)));
        long long t1 = clock64();
        clk[0] = t1 - t0;
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred P;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W2;\n\t}\n" ::"r"(
            smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // lanes 32w..32w+31 = rows m; 256 columns = n
    for (int c = 0; c < N; c += 32) {
        uint32_t v[32];
        const uint32_t ta = td + ((uint32_t)(warp * 32) << 16) + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
            "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) D[(size_t)tid * N + c + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(td), "n"(512));
}

int main() {
    __half *hA = new __half[M * K], *hB = new __half[K * N];
    float* ref = new float[M * N];
    srand(1);
    float *fA = new float[M * K], *fB = new float[K * N];
    for (int i = 0; i < M * K; ++i) { fA[i] = (float)((rand() % 17) - 8) / 8.f; hA[i] = __float2half(fA[i]); }
    for (int i = 0; i < K * N; ++i) { fB[i] = (float)((rand() % 13) - 6) / 4.f; hB[i] = __float2half(fB[i]); }
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            float s = 0;
            for (int k = 0; k < K; ++k) s += fA[m * K + k] * fB[k * N + n];
            ref[m * N + n] = s;
        }
    __half *dA, *dB;
    float* dD;
    long long* dclk;
    cudaMalloc(&dA, M * K * 2);
    cudaMalloc(&dB, K * N * 2);
    cudaMalloc(&dD, M * N * 4);
    cudaMalloc(&dclk, 8);
    cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, K * N * 2, cudaMemcpyHostToDevice);
    for (int reps : {1, 3, 4096}) {
        cudaMemset(dD, 0, M * N * 4);
        const int dsm = NBUF * (M + N) * K * 2;
        cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);
        k_probe<<<1, 128, dsm>>>(dA, dB, dD, dclk, reps);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
        float* hD = new float[M * N];
        long long clk;
        cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&clk, dclk, 8, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        int bad = 0;
        for (int i = 0; i < M * N; ++i) {
            double d = hD[i] - reps * (double)ref[i];
            if (d < 0) d = -d;
            if (d > maxerr) maxerr = d;
            if (d > 1e-3 * reps) ++bad;
        }
        printf("{\"reps\": %d, \"ks\": %d, \"max_abs_err\": %.3e, \"bad\": %d, \"clk\": %lld, \"clk_per_mma\": %.1f, "
               "\"d00\": %.4f, \"ref00\": %.4f}\n",
               reps, KS, maxerr, bad, clk, (double)clk / (reps * KS), hD[0], reps * ref[0]);
        delete[] hD;
    }
    return 0;
}
